"""Interleaved sustained-load A/B of the dense fwd+bwd step: our 2-CTA kernel
with 256x256 pair tiles (tuning 4096), 256x512 pair tiles (8192), the default
choice (0), and cuBLAS (torch.matmul), at one size (dev tool, round 2).

    python tools/ab_dense.py SIZE [rounds]
Each number: the last 20 steps of ~0.25 s of the same variant with no idle gap."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
S = int(sys.argv[1])
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
K = 20
g = torch.Generator(device="cuda")
g.manual_seed(1)
sets = [tuple((torch.rand(S, S, generator=g, device="cuda") - 0.5).to(torch.bfloat16) for _ in range(3))
        for _ in range(3)]
plans = [sd.LayerPlan(*st, 0.5, dy_ready=True) for st in sets]


def ours(i):
    pl = plans[i % 3]
    pl.dense_forward()
    pl.dense_backward()


def cublas(i):
    x, w, dy = sets[i % 3]
    return x @ w, x.t() @ dy, dy @ w.t()


variants = {"2cta 256x256": (ours, 4096), "2cta 256x512": (ours, 8192), "default": (ours, 0),
            "cublas": (cublas, 0)}
res = {n: [] for n in variants}
for r in range(rounds):
    for name, (fn, tun) in variants.items():
        lib.sd_set_tuning(tun)
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < 0.25:
            fn(n)
            n += 1
            if n % 64 == 0:
                torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(K):
            fn(n + i)
        b.record()
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / K)
lib.sd_set_tuning(0)
fl = 3 * 2 * S ** 3
for name, v in res.items():
    v = sorted(v)
    m = v[len(v) // 2]
    print(f"S={S} {name:14s} median {m * 1e3:8.1f} us/step = {fl / (m * 1e-3) / 1e12:7.1f} TFLOP/s  (min {v[0] * 1e3:.1f}, "
          f"max {v[-1] * 1e3:.1f})", flush=True)
