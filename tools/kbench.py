"""Per-kernel microbenchmark (dev tool): each C-ABI GEMM back-to-back at a shape,
CUDA-event timed, reported as executed TFLOP/s.  python tools/kbench.py [size ...]"""
import ctypes
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()


def st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    sizes = [int(s) for s in sys.argv[1:]] or [4096, 8192]
    for S in sizes:
        M = N = K = S
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
        dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        dx = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
        dw = torch.empty(K, N, device="cuda", dtype=torch.float32)
        fl = 2 * M * N * K
        res = {}
        res["dense_nn(fwd)"] = timeit(lambda: lib.sd_dense_gemm(x.data_ptr(), w.data_ptr(), y.data_ptr(), 1, M, N, K, st()))
        res["dense_nt(dx)"] = timeit(lambda: lib.sd_dense_gemm_nt(dy.data_ptr(), w.data_ptr(), dx.data_ptr(), 1, M, K, N, st()))
        res["dense_tn(dw)"] = timeit(lambda: lib.sd_dense_gemm_tn(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, K, N, M, st()))
        res["torch_mm"] = timeit(lambda: torch.matmul(x, w))
        line = {k: f"{fl / v / 1e9:.0f}TF ({v * 1e3:.1f}us)" for k, v in res.items()}
        print(S, "dense", line, flush=True)
        for p in (0.0, 0.5):
            m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 0), M, K)
            keep = m.keep_count() / m.total_blocks()
            s = sd.dropout_scale(p)
            r = {}
            r["fwd"] = timeit(lambda: lib.sd_linear_forward(x.data_ptr(), m.cptr(), w.data_ptr(), s, y.data_ptr(), 1, M, N, K, st()))
            r["dw"] = timeit(lambda: lib.sd_linear_backward_dw(x.data_ptr(), m.cptr(), dy.data_ptr(), s, dw.data_ptr(), 0, M, N, K, st()))
            r["dx"] = timeit(lambda: lib.sd_linear_backward_dx(dy.data_ptr(), w.data_ptr(), m.cptr(), s, dx.data_ptr(), 1, M, N, K, st()))
            r["mask"] = timeit(lambda: sd.sample_mask(sd.DropoutSpec(p, 128, 128, 1), M, K, out=m))
            line = {k: f"{keep * fl / v / 1e9:.0f}TF ({v * 1e3:.1f}us)" for k, v in r.items()}
            print(S, f"p={p} keep={keep:.3f}", line, flush=True)
        del x, w, dy, y, dx, dw
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
