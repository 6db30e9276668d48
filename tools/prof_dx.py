"""One sdd dX launch and one transposed 2-CTA dX launch (kTuneDxt) for ncu (dev tool).
   python tools/prof_dx.py SIZE P"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
S, P = int(sys.argv[1]), float(sys.argv[2])
x, w, dy = (torch.randn(S, S, device="cuda").to(torch.bfloat16) for _ in range(3))
plan = sd.LayerPlan(x, w, dy, P, dy_ready=True)
plan.forward(0)
for tune in (0, 1048576, 0, 1048576):
    lib.sd_set_tuning(tune)
    plan.backward_dx()
lib.sd_set_tuning(0)
torch.cuda.synchronize()
print("done")
