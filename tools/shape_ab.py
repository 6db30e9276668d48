"""Forward / backward of one SparseDrop layer at an arbitrary shape under several
tuning values, interleaved in one process (dev tool).
python tools/shape_ab.py M N K P tuningA,tuningB[,...] [rounds]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
M, N, K = (int(v) for v in sys.argv[1:4])
P = float(sys.argv[4])
tunings = [int(v) for v in sys.argv[5].split(",")]
rounds = int(sys.argv[6]) if len(sys.argv) > 6 else 8
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (torch.randn(K, N, device="cuda") * 0.03).to(torch.bfloat16)
dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
plan = sd.LayerPlan(x, w, dy, P)
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
res = {t: {"fwd": [], "bwd": []} for t in tunings}
t_end = time.time() + 1.0
while time.time() < t_end:
    plan.forward(1)
    plan.backward()
for r in range(rounds):
    for t in tunings:
        lib.sd_set_tuning(t)
        for k, fn in (("fwd", lambda: plan.forward(r)), ("bwd", plan.backward)):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            res[t][k].append(e0.elapsed_time(e1) * 1e3)
lib.sd_set_tuning(0)
for t in tunings:
    med = {k: sorted(v)[len(v) // 2] for k, v in res[t].items()}
    print(f"M={M} N={N} K={K} p={P} tuning={t}: fwd {med['fwd']:.1f} us  bwd {med['bwd']:.1f} us", flush=True)
