"""Compute cost of issuing dW in row slabs (the data-parallel backward's
all-reduce overlap) on one rank's configs[4] shard at G = 8 (M = 65536 rows,
K = N = 8192), p = 0.5 — sustained, interleaved, device-timed (dev probe, r02).
The all-reduce itself needs several GPUs; here: fused backward vs dW + dX vs
dW in 2 / 4 slabs + dX, and the C-ABI path on a 1-rank communicator."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2411_01238_b200 as sd  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(5)
M, K, N, p = 65536, 8192, 8192, float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
x, w, dy = ((torch.rand(r, c, generator=g, device="cuda") - 0.5).to(torch.bfloat16) for r, c in ((M, K), (K, N), (M, N)))
plan = sd.LayerPlan(x, w, dy, p, dy_ready=True, row_block_offset=512)
comm = sd.Communicator(1, 0, sd.Communicator.new_unique_id())
side = torch.cuda.Stream()


def fused(i):
    plan.forward(i)
    plan.backward()


def split(i):
    plan.forward(i)
    plan.backward_dw()
    plan.backward_dx()


def slabs(n):
    def f(i):
        plan.forward(i)
        for k in range(n):
            plan.backward_dw_part(k, n)
        plan.backward_dx()
    return f


def cabi(n):
    def f(i):
        plan.forward(i)
        plan.backward_allreduce(comm, n, comm_stream=side)
    return f


variants = {"fused backward": fused, "dW + dX": split, "dW 2 slabs + dX": slabs(2), "dW 4 slabs + dX": slabs(4),
            "C-ABI allreduce 1 slab (1-rank NCCL)": cabi(1), "C-ABI allreduce 2 slabs (1-rank NCCL)": cabi(2)}
res = {k: [] for k in variants}
for r in range(3):
    for name, fn in variants.items():
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < 1.0:
            fn(n)
            n += 1
            if n % 8 == 0:
                torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(5):
            fn(1000 + i)
        b.record()
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / 5)
for name, v in res.items():
    v = sorted(v)
    print(f"M={M} K=N={K} p={p} {name:40s} median {v[1]:8.3f} ms/step (min {v[0]:.3f})", flush=True)
torch.cuda.synchronize()
comm.close()
