"""Interleaved A/B of library BUILDS on back-to-back layer steps (dev tool).

    python tools/ab_steps_libs.py SIZE|M,N,K P LIB_A[:tuning] LIB_B[:tuning] [...] [-r ROUNDS]

Every library is loaded side by side (RTLD_LOCAL) with its own three layer
plans over the same three rotating input sets (> L2). Each round runs, for each
library in turn, K = 20 steps (mask + forward + backward, dy_ready) enqueued
back to back between one CUDA-event pair, after a sustained warm-up of all
libraries; prints the median ms/step per library and whether the last step's
outputs are bitwise equal across libraries (same seed)."""
import ctypes
import os
import shutil
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_01238_b200._capi import SdBlockMask  # noqa: E402

args = [a for a in sys.argv[1:]]
rounds = 10
if "-r" in args:
    i = args.index("-r")
    rounds = int(args[i + 1])
    del args[i:i + 2]
S, P, specs = args[0], float(args[1]), args[2:]
M, N, K_ = (int(v) for v in S.split(",")) if "," in S else (int(S),) * 3
STEPS = 20
_seen = set()


def load(spec):
    path, _, tune = spec.partition(":")
    path = os.path.abspath(path)
    if path in _seen:  # same file twice (two tunings): a private copy, one dlopen instance each
        copy = os.path.join(tempfile.mkdtemp(), os.path.basename(path))
        shutil.copy(path, copy)
        path = copy
    _seen.add(path)
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
    lib.sd_mask_workspace_bytes.restype = ctypes.c_size_t
    lib.sd_set_tuning(int(tune or 0))
    return lib


libs = [load(s) for s in specs]
sets = []
for _ in range(3):
    x = torch.randn(M, K_, device="cuda").to(torch.bfloat16)
    w = torch.randn(K_, N, device="cuda").to(torch.bfloat16)
    dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    sets.append((x, w, dy))
keep = []
plans = []  # [lib][set]
outs = []   # [lib][set] = (y, dx, dw)
R, C = M // 128, K_ // 128
for lib in libs:
    pl_l, out_l = [], []
    for x, w, dy in sets:
        nbytes = lib.sd_mask_workspace_bytes(R, C)
        ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device="cuda")
        mask = SdBlockMask()
        assert lib.sd_mask_bind(ctypes.byref(mask), ctypes.c_void_p((ws.data_ptr() + 255) & ~255), R, C, 128, 128,
                                0) == 0
        y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        dx = torch.empty(M, K_, dtype=torch.bfloat16, device="cuda")
        dw = torch.empty(K_, N, dtype=torch.float32, device="cuda")
        plan = ctypes.c_void_p()
        rc = lib.sd_layer_plan_create(ctypes.byref(plan), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                      ctypes.c_void_p(dy.data_ptr()), ctypes.c_void_p(y.data_ptr()), 1,
                                      ctypes.c_void_p(dx.data_ptr()), 1, ctypes.c_void_p(dw.data_ptr()), 0, M, N, K_,
                                      ctypes.c_double(P), ctypes.byref(mask))
        assert rc == 0, rc
        assert lib.sd_layer_plan_set_options(plan, 1) == 0  # SD_PLAN_DY_READY, as bench.py
        keep.append((ws, mask))
        pl_l.append(plan)
        out_l.append((y, dx, dw))
    plans.append(pl_l)
    outs.append(out_l)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def steps(li, n, seed0):
    lib = libs[li]
    for i in range(n):
        pl = plans[li][i % 3]
        assert lib.sd_layer_plan_forward(pl, ctypes.c_uint64(seed0 + i), st) == 0
        assert lib.sd_layer_plan_backward(pl, st) == 0


t_end = time.time() + 2.0
while time.time() < t_end:
    for li in range(len(libs)):
        steps(li, STEPS, 1000)
    torch.cuda.synchronize()
res = [[] for _ in libs]
for r in range(rounds):
    order = list(range(len(libs)))
    if r % 2:
        order.reverse()
    for li in order:
        steps(li, 3, 7)  # queue ahead: the timed region starts under load
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        steps(li, STEPS, 100 + r * STEPS)
        b.record()
        torch.cuda.synchronize()
        res[li].append(a.elapsed_time(b) / STEPS)
# same seeds on every library: the outputs of the last step must match
for li in range(len(libs)):
    steps(li, 3, 424242)
torch.cuda.synchronize()
same = [all(torch.equal(a, b) for a, b in zip(outs[0][s], outs[li][s])) for li in range(len(libs)) for s in range(3)]
for li, spec in enumerate(specs):
    v = sorted(res[li])
    print(f"{os.path.basename(spec):28s} S={S} p={P}: {v[len(v) // 2] * 1e3:8.1f} us/step (min {v[0] * 1e3:8.1f})",
          flush=True)
print("outputs bitwise equal across libraries:", all(same))
