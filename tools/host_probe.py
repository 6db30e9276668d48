"""Host cost per layer step (dev tool): wall time of the enqueue calls only,
with the device held behind a long spin so the launch queue never drains.
   python tools/host_probe.py [SIZE] [P]"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
P = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
lib = sd.load_library()
x, w, dy = (torch.randn(S, S, device="cuda").to(torch.bfloat16) for _ in range(3))
plan = sd.LayerPlan(x, w, dy, P, dy_ready=True)
for i in range(20):
    plan.forward(i), plan.backward()
torch.cuda.synchronize()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
pl = plan._plan
N = 150


def timed(fn):
    torch.cuda.synchronize()
    torch.cuda._sleep(int(2e7))  # ~10 ms: the queue holds every launch below
    t0 = time.perf_counter()
    for i in range(N):
        fn(i)
    t = (time.perf_counter() - t0) / N * 1e6
    torch.cuda.synchronize()
    return t


def py_step(i):
    plan.forward(i)
    plan.backward()


def raw_step(i):
    lib.sd_layer_plan_forward(pl, ctypes.c_uint64(i), st)
    lib.sd_layer_plan_backward(pl, st)


def raw_fwd(i):
    lib.sd_layer_plan_forward(pl, ctypes.c_uint64(i), st)


def raw_dense(i):
    lib.sd_layer_plan_dense_forward(pl, st)
    lib.sd_layer_plan_dense_backward(pl, st)


def noop(i):
    lib.sd_abi_version()


for name, fn in (("python step", py_step), ("raw ctypes step", raw_step), ("raw forward only", raw_fwd),
                 ("raw dense step", raw_dense), ("ctypes no-op call", noop)):
    vals = sorted(timed(fn) for _ in range(5))
    print(f"S={S} p={P} {name:20s}: {vals[2]:6.2f} us per call", flush=True)
