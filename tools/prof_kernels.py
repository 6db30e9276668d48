"""Launch a fixed set of kernels once each (after warm-up) for ncu capture (dev tool).
python tools/prof_kernels.py SIZE P [which...]   which in {fwd, dw, dx, dense_nn, dense_nt, dense_tn, mask, bwd,
cublas_nn}"""
import ctypes
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
P = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
which = sys.argv[3:] or ["fwd", "dw", "dx"]
M = N = K = S
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
dx = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
dw = torch.empty(K, N, device="cuda", dtype=torch.float32)
plan = sd.LayerPlan(x, w, dy, P, dy_ready=True)
plan.forward(0)
m = plan.mask
s = sd.dropout_scale(P)


def st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


fns = {
    "fwd": lambda: lib.sd_linear_forward(x.data_ptr(), m.cptr(), w.data_ptr(), s, y.data_ptr(), 1, M, N, K, st()),
    "dw": lambda: lib.sd_linear_backward_dw(x.data_ptr(), m.cptr(), dy.data_ptr(), s, dw.data_ptr(), 0, M, N, K, st()),
    "dx": lambda: lib.sd_linear_backward_dx(dy.data_ptr(), w.data_ptr(), m.cptr(), s, dx.data_ptr(), 1, M, N, K, st()),
    "dense_nn": lambda: lib.sd_dense_gemm(x.data_ptr(), w.data_ptr(), y.data_ptr(), 1, M, N, K, st()),
    "dense_nt": lambda: lib.sd_dense_gemm_nt(dy.data_ptr(), w.data_ptr(), dx.data_ptr(), 1, M, K, N, st()),
    "dense_tn": lambda: lib.sd_dense_gemm_tn(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, K, N, M, st()),
    "mask": lambda: sd.sample_mask(sd.DropoutSpec(P, 128, 128, 1), M, K, out=m),
    "bwd": lambda: plan.backward(),
    "cublas_nn": lambda: torch.matmul(x, w, out=y),
}
def run(k):
    r = fns[k]()
    if isinstance(r, int) and r != 0:
        raise RuntimeError(f"{k}: {sd.api.last_error() if hasattr(sd.api, 'last_error') else r}")


for _ in range(2):
    for k in which:
        run(k)
torch.cuda.synchronize()
for k in which:
    run(k)
torch.cuda.synchronize()
print("done", S, P, which)
