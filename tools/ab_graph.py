"""Interleaved A/B under sustained load: eager launches vs CUDA-graph replay,
and 2-CTA tail halving on/off (dev tool, round 2).

    python tools/ab_graph.py SIZE P [rounds]

Every measurement is the LAST K steps of ~0.25 s of back-to-back work of the
same variant enqueued without a host sync in between (the GPU never idles
before the timed steps, so the power-capped clock is in its steady state for
that workload: an idle gap — e.g. while a graph is captured — lets the clock
rise and inflates a short timed burst). Variants alternate every round.
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
S = int(sys.argv[1])
P = float(sys.argv[2])
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 8
K = 20
g = torch.Generator(device="cuda")
g.manual_seed(1)


def rnd(r, c):
    return ((0.25 + torch.rand(r, c, generator=g, device="cuda")) *
            torch.where(torch.rand(r, c, generator=g, device="cuda") < 0.5, -1.0, 1.0)).to(torch.bfloat16)


plans = [sd.LayerPlan(rnd(S, S), rnd(S, S), rnd(S, S), P, dy_ready=True) for _ in range(3)]


def sparse(i):
    pl = plans[i % 3]
    pl.forward(seed=i)
    pl.backward()


def dense(i):
    pl = plans[i % 3]
    pl.dense_forward()
    pl.dense_backward()


def make(fn, graph, tuning):
    lib.sd_set_tuning(tuning)
    for i in range(6):
        fn(i)
    torch.cuda.synchronize()
    if not graph:
        return lambda i0: [fn(i0 + i) for i in range(K)]
    gr = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=cs):
        for i in range(K):
            fn(1000 + i)
    torch.cuda.synchronize()
    return lambda i0: gr.replay()


variants = {
    "sparse eager": (sparse, False, 0), "sparse graph": (sparse, True, 0),
    "dense eager": (dense, False, 0), "dense eager no-tail-halving": (dense, False, 4096),
    "dense graph": (dense, True, 0), "dense graph no-tail-halving": (dense, True, 4096),
}
runners = {}
for name, (fn, gph, tun) in variants.items():
    runners[name] = (make(fn, gph, tun), tun)
lib.sd_set_tuning(0)
res = {n: [] for n in variants}
for r in range(rounds):
    for name, (run, tun) in runners.items():
        lib.sd_set_tuning(tun)
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < 0.25:  # host enqueues; the GPU queue stays full
            run(n * K)
            n += 1
            if n % 50 == 0:
                torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(n * K)
        b.record()
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / K)
lib.sd_set_tuning(0)
for name, v in res.items():
    v = sorted(v)
    print(f"S={S} p={P} {name:32s} median {v[len(v) // 2] * 1e3:8.1f} us/step  (min {v[0] * 1e3:.1f}, max "
          f"{v[-1] * 1e3:.1f})", flush=True)
