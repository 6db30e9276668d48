"""e2e (host buffers, HostLayerPipeline) ms/step under several tuning values,
interleaved (dev tool).   python tools/e2e_ab.py [SIZE] [P] [tunings] [rounds]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402
from paper_2411_01238_b200.pipeline import HostLayerPipeline  # noqa: E402

lib = sd.load_library()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
P = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
tunings = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "0,384").split(",")]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 4
xh = torch.randn(S, S).to(torch.bfloat16).pin_memory()
wh = torch.randn(S, S).to(torch.bfloat16).pin_memory()
dyh = torch.randn(S, S).to(torch.bfloat16).pin_memory()
pipe = HostLayerPipeline(xh, wh, dyh, P)
res = {t: [] for t in tunings}
step = 0
for r in range(rounds):
    for t in tunings:
        lib.sd_set_tuning(t)
        for _ in range(3):
            pipe.step(step); step += 1
        pipe.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pipe.s_h2d)
        pipe.s_cmp.wait_stream(pipe.s_h2d)
        n = 10
        for _ in range(n):
            pipe.step(step); step += 1
        pipe.s_d2h.wait_stream(pipe.s_cmp)
        pipe.s_d2h.wait_stream(pipe.s_h2d)
        e1.record(pipe.s_d2h)
        pipe.synchronize()
        res[t].append(e0.elapsed_time(e1) / n)
lib.sd_set_tuning(0)
for t, v in res.items():
    v = sorted(v)
    print(f"tuning {t}: e2e {v[len(v) // 2]:.3f} ms/step (min {v[0]:.3f}, max {v[-1]:.3f}) "
          f"{(pipe.h2d_bytes + pipe.d2h_bytes) / (v[len(v) // 2] * 1e-3) / 1e9:.1f} GB/s")
