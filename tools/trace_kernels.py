"""Wait-cycle attribution for the GEMM kernel (dev tool; needs `make trace`).

  SPARSEDROP_B200_LIB=paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so \
      python tools/trace_kernels.py SIZE|M,N,K P
For each kernel: mean per-CTA cycles of the MMA thread's run, of its waits for
data (full), for TMEM (epilogue) and for the scheduler, the producer's waits for
free stages, and the epilogue's waits — as fractions of the MMA thread's run."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SPARSEDROP_B200_LIB", os.path.join(ROOT, "paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so"))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
lib.sd_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
S = sys.argv[1] if len(sys.argv) > 1 else "4096"
P = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
M, N, K = (int(v) for v in S.split(",")) if "," in S else (int(S),) * 3
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
plan = sd.LayerPlan(x, w, dy, P, dy_ready=True)
plan.forward(0)
torch.cuda.synchronize()
m = plan.mask
s = plan.scale
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
dx = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
dw = torch.empty(K, N, device="cuda", dtype=torch.float32)
st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
fns = {
    "dense_nn": lambda: lib.sd_dense_gemm(x.data_ptr(), w.data_ptr(), y.data_ptr(), 1, M, N, K, st()),
    "dense_nt": lambda: lib.sd_dense_gemm_nt(dy.data_ptr(), w.data_ptr(), dx.data_ptr(), 1, M, K, N, st()),
    "dense_tn": lambda: lib.sd_dense_gemm_tn(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, K, N, M, st()),
    "fwd": lambda: lib.sd_linear_forward(x.data_ptr(), m.cptr(), w.data_ptr(), s, y.data_ptr(), 1, M, N, K, st()),
    "dw": lambda: lib.sd_linear_backward_dw(x.data_ptr(), m.cptr(), dy.data_ptr(), s, dw.data_ptr(), 0, M, N, K, st()),
    "dx": lambda: lib.sd_linear_backward_dx(dy.data_ptr(), w.data_ptr(), m.cptr(), s, dx.data_ptr(), 1, M, N, K, st()),
    "bwd_fused": lambda: plan.backward(),
}
buf = np.zeros(1024 * 16, dtype=np.uint64)
names = ["prod_wait_empty", "prod_wait_sched", "mma_wait_full", "mma_wait_tmem", "mma_wait_sched", "epi_wait_tfull",
         "epi_wait_sched", "mma_run", "stages", "prod_run", "epi_run", "units"]
only = os.environ.get("ONLY", "").split(",") if os.environ.get("ONLY") else None
for name, fn in fns.items():
    if only and name not in only:
        continue
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    lib.sd_trace_read(buf.ctypes.data, buf.size)  # clear
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    lib.sd_trace_read(buf.ctypes.data, buf.size)
    t = buf.reshape(1024, 16)[:148].astype(np.float64)
    run = t[:, 7]
    active = run > 0
    r = {n: t[active, i].mean() for i, n in enumerate(names)}
    frac = lambda k: r[k] / r["mma_run"]  # noqa: E731
    mma_busy = 1 - frac("mma_wait_full") - frac("mma_wait_tmem") - frac("mma_wait_sched")
    if not active.any():
        print(f"{name:10s} {ms * 1e3:7.1f}us  (not on the traced 1-CTA kernel)")
        continue
    g_run = t[active, 12]; g_st = t[active, 13]; e_run = t[active, 14]
    ghz = (run[active] / np.maximum(g_run, 1)).mean()
    g0 = g_st.min()
    print(f"{name:10s} clock64 {ghz:.2f} GHz | CTA start spread {(g_st.max() - g0) / 1e3:.1f} us | "
          f"MMA run ns mean {g_run.mean() / 1e3:.1f} max {g_run.max() / 1e3:.1f} us | epi end max "
          f"{(e_run + g_st - g0).max() / 1e3:.1f} us after first start")
    print(f"{name:10s} {ms * 1e3:7.1f}us  mma_run={r['mma_run'] / 1e3:6.1f}kcyc (max {run.max() / 1e3:6.1f}, "
          f"min {run[active].min() / 1e3:6.1f})  wait_full={frac('mma_wait_full'):.2f} "
          f"wait_tmem={frac('mma_wait_tmem'):.2f} wait_sched={frac('mma_wait_sched'):.2f} -> issue-side busy {mma_busy:.2f} | "
          f"stages/CTA={r['stages']:.0f} ({r['stages'] * 512 / r['mma_run']:.2f} of run at 512cyc/stage) | "
          f"prod_wait_empty={r['prod_wait_empty'] / r['prod_run']:.2f} epi_wait_tfull={r['epi_wait_tfull'] / r['epi_run']:.2f} "
          f"units/CTA={r['units']:.1f}", flush=True)
