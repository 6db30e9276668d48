"""Interleaved A/B of tuning switches on BACK-TO-BACK layer steps (dev tool).

    python tools/ab_steps.py SIZE P flagsA,flagsB[,...] [rounds]

Like bench.py's headline: three plans over rotating input sets (> L2), K steps
(mask + forward + fused backward) enqueued back to back between one CUDA-event
pair, so launch overlap between steps and kernels (PDL) is what is measured.
Variants alternate every round after a sustained warm-up; prints the median
ms/step per variant."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
S = sys.argv[1]  # SIZE or M,N,K
M_, N_, K_ = (int(v) for v in S.split(",")) if "," in S else (int(S),) * 3
P = float(sys.argv[2])
variants = [int(v) for v in sys.argv[3].split(",")]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 10
K = 20
plans = []
for i in range(3):
    x = torch.randn(M_, K_, device="cuda").to(torch.bfloat16)
    w = torch.randn(K_, N_, device="cuda").to(torch.bfloat16)
    dy = torch.randn(M_, N_, device="cuda").to(torch.bfloat16)
    plans.append(sd.LayerPlan(x, w, dy, P, dy_ready=True))


DENSE = os.environ.get("DENSE") == "1"  # time the dense step (dense_forward + dense_backward) instead


def steps(n, seed0):
    for i in range(n):
        pl = plans[i % 3]
        if DENSE:
            pl.dense_forward()
            pl.dense_backward()
        else:
            pl.forward(seed0 + i)
            pl.backward()


t_end = time.time() + 1.5
while time.time() < t_end:
    for v in variants:
        lib.sd_set_tuning(v)
        steps(6, 0)
torch.cuda.synchronize()
res = {v: [] for v in variants}
for r in range(rounds):
    for v in variants:
        lib.sd_set_tuning(v)
        steps(3, 1000)  # settle the new mode
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        steps(K, 10 * r)
        b.record()
        torch.cuda.synchronize()
        res[v].append(a.elapsed_time(b) / K)
lib.sd_set_tuning(0)
for v in variants:
    xs = sorted(res[v])
    print(f"S={S} p={P} {'dense' if DENSE else 'sparse'} tuning {v:4d}: {xs[len(xs) // 2] * 1e3:7.1f} us/step (min {xs[0] * 1e3:6.1f})", flush=True)
