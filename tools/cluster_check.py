"""Cluster-pair (A-multicast) GEMM path vs the 1-CTA path: bitwise parity of the
layer step + interleaved timing (dev tool).
python tools/cluster_check.py"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
BASE, CLU = 1, 1 | 32
cases = [(512, 384, 768, 0.5), (1024, 1024, 1024, 0.0), (1024, 1024, 1024, 0.3), (4096, 4096, 4096, 0.5),
         (4096, 4096, 4096, 0.9), (2048, 1152, 640, 0.7), (8192, 1024, 1024, 0.5)]
ok = True
for M, N, K, P in cases:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    plan = sd.LayerPlan(x, w, dy, P)
    outs = {}
    for t in (BASE, CLU):
        lib.sd_set_tuning(t)
        plan.y.zero_(); plan.dx.zero_(); plan.dw.zero_()
        plan.forward(7)
        plan.backward()
        torch.cuda.synchronize()
        outs[t] = (plan.y.float().clone(), plan.dx.float().clone(), plan.dw.float().clone())
    diffs = [(a - b).abs().max().item() for a, b in zip(outs[BASE], outs[CLU])]
    dwref = outs[BASE][2].abs().max().item()
    good = diffs[0] == 0 and diffs[1] == 0 and diffs[2] <= 1e-5 * max(dwref, 1)
    ok &= good
    # timing (interleaved)
    res = {BASE: [], CLU: []}
    for r in range(6):
        for t in (BASE, CLU):
            lib.sd_set_tuning(t)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e2 = torch.cuda.Event(enable_timing=True)
            for _ in range(2):
                plan.forward(r); plan.backward()
            e0.record()
            for i in range(10):
                plan.forward(i)
            e1.record()
            for i in range(10):
                plan.backward()
            e2.record()
            torch.cuda.synchronize()
            res[t].append((e0.elapsed_time(e1) * 100, e1.elapsed_time(e2) * 100))
    med = {t: [sorted(v[i] for v in res[t])[len(res[t]) // 2] for i in range(2)] for t in res}
    print(f"{M}x{N}x{K} p={P}: max|diff| y {diffs[0]:.2e} dx {diffs[1]:.2e} dw {diffs[2]:.2e} {'OK' if good else 'MISMATCH'}"
          f" | fwd {med[BASE][0]:.1f} -> {med[CLU][0]:.1f} us, bwd {med[BASE][1]:.1f} -> {med[CLU][1]:.1f} us", flush=True)
lib.sd_set_tuning(1)
print("ALL OK" if ok else "FAILURES")
