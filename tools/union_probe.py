"""Union-mode 2-CTA dsd vs the 1-CTA kernels (dev tool): pair lists built on the
host from the mask; checks bitwise equality with the 1-CTA forward/dW and times
both.  python tools/union_probe.py SIZE|M,N,K P..."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
lib.sd_dev_dsd_pairs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_void_p]
lib.sd_last_error.restype = ctypes.c_char_p
S = sys.argv[1]  # SIZE or M,N,K
M, N, K = (int(v) for v in S.split(",")) if "," in S else (int(S),) * 3
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731


def pair_lists(bits):
    """bits: (R, C) bool keep; pairs of rows (2p, 2p+1) -> (cnt[R/2], idx[R/2][C])."""
    R, C = bits.shape
    cnt = np.zeros(R // 2, np.int32)
    idx = np.zeros((R // 2, C), np.int32)
    for p in range(R // 2):
        own = bits[2 * p].astype(np.int32) | (bits[2 * p + 1].astype(np.int32) << 1)
        cols = np.nonzero(own)[0]
        cnt[p] = len(cols)
        idx[p, :len(cols)] = (cols << 2) | own[cols]
    return torch.from_numpy(cnt).cuda(), torch.from_numpy(idx).cuda()


def timeit(fn, n=10):
    ts = []
    for _ in range(n):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]


for P in [float(v) for v in sys.argv[2:]]:
    plan = sd.LayerPlan(x, w, dy, P)
    plan.forward(11)
    torch.cuda.synchronize()
    words = np.array(plan.mask.words(), dtype=np.uint64)
    R, C = M // 128, K // 128
    flat = np.unpackbits(words.view(np.uint8), bitorder="little")[: R * C].astype(bool)
    bits = flat.reshape(R, C)
    s = plan.scale
    # forward: rows = M blocks, reduction = K blocks
    fc, fi = pair_lists(bits)
    y1 = plan.y.clone()
    y2 = torch.empty_like(y1)
    fwd2 = lambda: lib.sd_dev_dsd_pairs(x.data_ptr(), w.data_ptr(), y2.data_ptr(), 1, M, N, K, 0, 128,  # noqa: E731
                                        fc.data_ptr(), fi.data_ptr(), C, ctypes.c_float(s), st())
    rc = fwd2()
    assert rc == 0, lib.sd_last_error()
    torch.cuda.synchronize()
    # dW: rows = K blocks (mask columns), reduction = M blocks
    dc, di = pair_lists(bits.T.copy())
    plan.backward_dw()
    torch.cuda.synchronize()
    dw1 = plan.dw.clone()
    dw2 = torch.empty_like(dw1)
    dw2f = lambda: lib.sd_dev_dsd_pairs(x.data_ptr(), dy.data_ptr(), dw2.data_ptr(), 0, K, N, M, 1, 128,  # noqa: E731
                                        dc.data_ptr(), di.data_ptr(), R, ctypes.c_float(s), st())
    rc = dw2f()
    assert rc == 0, lib.sd_last_error()
    torch.cuda.synchronize()
    union_f = float(fc.sum()) / (R // 2 * C)
    keep = bits.mean()
    t_f1 = timeit(lambda: lib.sd_linear_forward(x.data_ptr(), plan.mask.cptr(), w.data_ptr(), ctypes.c_float(s),
                                                  y1.data_ptr(), 1, M, N, K, st()))
    t_f2 = timeit(fwd2)
    t_w1 = timeit(plan.backward_dw)
    t_w2 = timeit(dw2f)
    t_x1 = timeit(plan.backward_dx)
    print(f"S={S} p={P} keep={keep:.3f} union={union_f:.3f}: fwd 1cta {t_f1:.1f} us / union-2cta {t_f2:.1f} us "
          f"(equal {torch.equal(y1, y2)}); dW 1cta {t_w1:.1f} / union-2cta {t_w2:.1f} (equal {torch.equal(dw1, dw2)}); "
          f"dX 1cta {t_x1:.1f}", flush=True)
