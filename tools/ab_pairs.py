"""Sustained-load interleaved A/B of the row-pair dX split (tuning 0) vs the
plain 1-CTA sdd dX (tuning 16384) on back-to-back layer steps (dev tool, r02).

    python tools/ab_pairs.py M N K p[,p...] [rounds]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
M, N, K = (int(v) for v in sys.argv[1:4])
ps = [float(v) for v in sys.argv[4].split(",")]
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 6
g = torch.Generator(device="cuda")
g.manual_seed(1)
nsets = 3 if M * K * 2 < (1 << 30) else 1
sets = [((torch.rand(M, K, generator=g, device="cuda") - 0.5).to(torch.bfloat16),
         (torch.rand(K, N, generator=g, device="cuda") - 0.5).to(torch.bfloat16),
         (torch.rand(M, N, generator=g, device="cuda") - 0.5).to(torch.bfloat16)) for _ in range(nsets)]
KS = 20 if M * N * K <= 4096 ** 3 else 5
for p in ps:
    plans = [sd.LayerPlan(*st, p, dy_ready=True) for st in sets]

    def step(i, what):
        pl = plans[i % nsets]
        if what == "step":
            pl.forward(seed=i)
            pl.backward()
        else:
            pl.backward_dx()

    res = {}
    for what in ("step", "dx"):
        for tun in (0, 16384):
            res[(what, tun)] = []
    for r in range(rounds):
        for what in ("step", "dx"):
            for tun in (0, 16384):
                lib.sd_set_tuning(tun)
                t0 = time.perf_counter()
                n = 0
                while time.perf_counter() - t0 < 0.2:
                    step(n, what)
                    n += 1
                    if n % 64 == 0:
                        torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for i in range(KS):
                    step(n + i, what)
                b.record()
                torch.cuda.synchronize()
                res[(what, tun)].append(a.elapsed_time(b) / KS)
    lib.sd_set_tuning(0)
    med = {k: sorted(v)[len(v) // 2] * 1e3 for k, v in res.items()}
    print(f"M={M} N={N} K={K} p={p}: step pairs {med[('step', 0)]:.1f} us vs sdd {med[('step', 16384)]:.1f} us "
          f"({med[('step', 0)] / med[('step', 16384)] - 1:+.1%}); dX alone pairs {med[('dx', 0)]:.1f} vs sdd "
          f"{med[('dx', 16384)]:.1f} us ({med[('dx', 0)] / med[('dx', 16384)] - 1:+.1%})", flush=True)
    del plans
