"""Dense/sparse step variants each timed in ITS OWN settled power-capped state
(bench.py's methodology: 1.5 s of the variant, then 20 timed steps), two rounds
alternating (dev tool, round 2).

    python tools/ab_settled.py SIZE p "name:tuning:kind" ...   kind in {dense, sparse, cublas}"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
S = int(sys.argv[1])
P = float(sys.argv[2])
variants = [v.split(":") for v in sys.argv[3:]]
g = torch.Generator(device="cuda")
g.manual_seed(1)


def rnd(r, c):
    return ((0.25 + torch.rand(r, c, generator=g, device="cuda")) *
            torch.where(torch.rand(r, c, generator=g, device="cuda") < 0.5, -1.0, 1.0)).to(torch.bfloat16)


sets = [(rnd(S, S), rnd(S, S), rnd(S, S)) for _ in range(3)]
plans = [sd.LayerPlan(*st, P, dy_ready=True) for st in sets]


def fn_of(kind):
    if kind == "dense":
        return lambda i: (plans[i % 3].dense_forward(), plans[i % 3].dense_backward())
    if kind == "sparse":
        return lambda i: (plans[i % 3].forward(seed=i), plans[i % 3].backward())
    return lambda i: (sets[i % 3][0] @ sets[i % 3][1], sets[i % 3][0].t() @ sets[i % 3][2],
                      sets[i % 3][2] @ sets[i % 3][1].t())


res = {v[0]: [] for v in variants}
for r in range(2):
    for name, tun, kind in variants:
        lib.sd_set_tuning(int(tun))
        fn = fn_of(kind)
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < 1.5:
            fn(n)
            n += 1
            if n % 64 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(20):
            fn(n + i)
        b.record()
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / 20 * 1e3)
lib.sd_set_tuning(0)
for name, v in res.items():
    print(f"S={S} p={P} {name:20s} " + " ".join(f"{x:8.1f}" for x in v) + " us/step", flush=True)
