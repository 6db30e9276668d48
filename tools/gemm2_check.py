"""2-CTA (cta_group::2) GEMM path check + A/B timing against the 1-CTA kernel (dev tool).
python tools/gemm2_check.py [SIZES...]"""
import ctypes
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
sizes = [int(s) for s in sys.argv[1:]] or [512, 4096, 8192]


def st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ops(M, N, K):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    bt = b.t().contiguous()
    at = a.t().contiguous()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    y32 = torch.empty(M, N, device="cuda", dtype=torch.float32)
    ref = a.float() @ b.float()
    return {
        "nn_bf16": (lambda: lib.sd_dense_gemm(a.data_ptr(), b.data_ptr(), y.data_ptr(), 1, M, N, K, st()), y, ref),
        "nt_bf16": (lambda: lib.sd_dense_gemm_nt(a.data_ptr(), bt.data_ptr(), y.data_ptr(), 1, M, N, K, st()), y, ref),
        "tn_f32": (lambda: lib.sd_dense_gemm_tn(at.data_ptr(), b.data_ptr(), y32.data_ptr(), 0, M, N, K, st()), y32, ref),
    }


for S in sizes:
    M = N = K = S
    for name, (fn, out, ref) in ops(M, N, K).items():
        res = {}
        for tune in (17, 1):
            lib.sd_set_tuning(tune)
            out.zero_()
            fn()
            torch.cuda.synchronize()
            res[tune] = out.float().clone()
            err = ((res[tune] - ref).abs().max() / ref.abs().max()).item()
            # timing: back-to-back launches
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 20
            e0.record()
            for _ in range(n):
                fn()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / n
            tf = 2 * M * N * K / us / 1e6
            print(f"S={S} {name} tuning={tune}: rel_err {err:.2e}  {us:8.1f} us  {tf:7.1f} TF/s", flush=True)
        d = (res[17] - res[1]).abs().max().item()
        print(f"   max |1cta - 2cta| = {d:.3e}", flush=True)
lib.sd_set_tuning(0)
