"""Interleaved A/B of two builds of libsparsedrop_b200.so in ONE process (dev tool).

    python tools/ab_libs.py LIB_A[:tuning] LIB_B[:tuning] [SIZE|M,N,K] [P] [rounds]

Both libraries are loaded side by side (RTLD_LOCAL) and bound to the same
operand buffers through their own layer plans; each round times forward,
backward, standalone dW and dX of A then B with an L2 flush before every
kernel, after a sustained warm-up, so clocks, allocation and L2 state are
shared. Prints medians (us)."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_01238_b200._capi import SdBlockMask  # noqa: E402


_loaded = set()


def load(spec):
    path, _, tune = spec.partition(":")
    path = os.path.abspath(path)
    if path in _loaded:
        # dlopen of the same path returns the same instance (one tuning state):
        # A/B two tunings of one build through a private copy
        import shutil
        import tempfile
        copy = os.path.join(tempfile.mkdtemp(), os.path.basename(path))
        shutil.copy(path, copy)
        path = copy
    _loaded.add(path)
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
    lib.sd_mask_workspace_bytes.restype = ctypes.c_size_t
    lib.sd_set_tuning(int(tune or 0))
    return lib


S = sys.argv[3] if len(sys.argv) > 3 else "4096"  # SIZE or M,N,K
P = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 8
libs = [load(sys.argv[1]), load(sys.argv[2])]
M, N, K = (int(v) for v in S.split(",")) if "," in S else (int(S),) * 3
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
outs, plans, keep = [], [], []
for lib in libs:
    R, C = M // 128, K // 128
    nbytes = lib.sd_mask_workspace_bytes(R, C)
    ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device="cuda")
    mask = SdBlockMask()
    assert lib.sd_mask_bind(ctypes.byref(mask), ctypes.c_void_p((ws.data_ptr() + 255) & ~255), R, C, 128, 128, 0) == 0
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    dx = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
    dw = torch.empty(K, N, dtype=torch.float32, device="cuda")
    plan = ctypes.c_void_p()
    rc = lib.sd_layer_plan_create(ctypes.byref(plan), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                  ctypes.c_void_p(dy.data_ptr()), ctypes.c_void_p(y.data_ptr()), 1,
                                  ctypes.c_void_p(dx.data_ptr()), 1, ctypes.c_void_p(dw.data_ptr()), 0, M, N, K,
                                  ctypes.c_double(P), ctypes.byref(mask))
    assert rc == 0, rc
    plans.append(plan)
    keep.append((ws, mask))
    outs.append((y, dx, dw))
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
ops = {
    "fwd": lambda lib, pl: lib.sd_layer_plan_forward(pl, ctypes.c_uint64(5), st()),
    "bwd": lambda lib, pl: lib.sd_layer_plan_backward(pl, st()),
    "dw": lambda lib, pl: lib.sd_layer_plan_backward_dw(pl, st()),
    "dx": lambda lib, pl: lib.sd_layer_plan_backward_dx(pl, st()),
}
res = [{k: [] for k in ops} for _ in libs]
t_end = time.time() + 1.5
while time.time() < t_end:
    for lib, pl in zip(libs, plans):
        ops["fwd"](lib, pl)
        ops["bwd"](lib, pl)
torch.cuda.synchronize()
for _ in range(rounds):
    for i, (lib, pl) in enumerate(zip(libs, plans)):
        for name, fn in ops.items():
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            flush.fill_(1.0)
            ev[0].record()
            fn(lib, pl)
            ev[1].record()
            torch.cuda.synchronize()
            res[i][name].append(ev[0].elapsed_time(ev[1]) * 1e3)
same = [torch.equal(a, b) for a, b in zip(outs[0], outs[1])]
for i, spec in enumerate(sys.argv[1:3]):
    med = {k: sorted(v)[len(v) // 2] for k, v in res[i].items()}
    print(f"{spec:60s} S={S} p={P}: " + "  ".join(f"{k} {v:7.1f}" for k, v in med.items()), flush=True)
print("outputs (y, dx, dw) bitwise equal:", same)
