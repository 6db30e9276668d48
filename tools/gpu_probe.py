"""Quick GPU probe of each kernel family against torch / the oracle (dev tool).

Usage: python tools/gpu_probe.py [test ...]   (each test runs in a subprocess
with its own timeout so a hung kernel cannot take the others down)."""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TESTS = ["mask", "dense", "dense_nt", "dense_tn", "dsd", "dw", "dx", "sdd_ref", "layer"]


def run_one(name):
    import numpy as np
    import torch

    import paper_2411_01238_b200 as sd
    from oracle.oracle import Oracle

    o = Oracle()
    torch.manual_seed(0)
    dev = "cuda"

    def rnd(r, c, seed):
        return torch.from_numpy(o.random_matrix(r, c, seed)).to(dev).to(torch.bfloat16)

    def rel(a, b):
        a = a.double(); b = b.double()
        return ((a - b).norm() / max(b.norm().item(), 1e-30)).item()

    if name == "mask":
        for (rows, cols, p, seed) in [(1024, 1024, 0.5, 0), (4096, 4096, 0.3, 5), (65536, 8192, 0.5, 0),
                                      (65536, 768, 0.5, 0x238275bc38fcbe91), (128 * 37, 128 * 19, 0.9, 3)]:
            m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, seed), rows, cols)
            torch.cuda.synchronize()
            w, k = o.sample_mask(p, 128, 128, seed, rows, cols)
            got = np.array(m.words(), dtype=np.uint64)
            R, C = rows // 128, cols // 128
            ok_w = np.array_equal(got, w)
            ok_k = m.keep_count() == k
            rc = m.row_cnt_device().cpu().numpy(); ri = m.row_idx_device().cpu().numpy()
            ok_rows = all(ri[r, :rc[r]].tolist() == o.kept_blocks_in_row(w, R, C, r) for r in range(R))
            wt = o.transpose_mask(w, R, C)
            cc = m.col_cnt_device().cpu().numpy(); ci = m.col_idx_device().cpu().numpy()
            ok_cols = all(ci[c, :cc[c]].tolist() == o.kept_blocks_in_row(wt, C, R, c) for c in range(C))
            ro = sorted(m.row_order_device().cpu().tolist()) == list(range(R))
            print(f"mask {rows}x{cols} p={p}: words {ok_w} keep {ok_k} ({m.keep_count()}/{k}) rows {ok_rows} cols {ok_cols} order {ro}")
        return

    if name in ("dense", "dense_nt", "dense_tn"):
        for (M, N, K) in [(128, 256, 64), (256, 512, 256), (1024, 1024, 1024), (384, 640, 192)]:
            a = rnd(M, K, 1); b = rnd(K, N, 2)
            if name == "dense":
                c = sd.dense_gemm(a, b, out_dtype=torch.float32)
            elif name == "dense_nt":
                bt = b.t().contiguous()
                c = torch.empty(M, N, dtype=torch.float32, device=dev)
                sd.api.check(sd.api._lib().sd_dense_gemm_nt(a.data_ptr(), bt.data_ptr(), c.data_ptr(), 0, M, N, K,
                                                             sd.api.ctypes.c_void_p(sd.api._stream())))
            else:
                at = a.t().contiguous()
                c = torch.empty(M, N, dtype=torch.float32, device=dev)
                sd.api.check(sd.api._lib().sd_dense_gemm_tn(at.data_ptr(), b.data_ptr(), c.data_ptr(), 0, M, N, K,
                                                             sd.api.ctypes.c_void_p(sd.api._stream())))
            torch.cuda.synchronize()
            ref = a.float() @ b.float()
            print(f"{name} {M}x{N}x{K}: relF {rel(c, ref):.3e}  max|d| {(c - ref).abs().max().item():.3e}")
        return

    if name == "dsd":
        for (M, N, K, p) in [(1024, 1024, 1024, 0.5), (512, 768, 384, 0.3), (1024, 512, 1024, 0.9)]:
            a = rnd(M, K, 1); b = rnd(K, N, 2)
            m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 0), M, K)
            s = sd.dropout_scale(p)
            cnt = sd.KernelCounters()
            c = sd.dsd_matmul(a, m, b, s, counters=cnt, out_dtype=torch.float32)
            torch.cuda.synchronize()
            w = np.array(m.words(), dtype=np.uint64)
            ref = o.dsd_matmul(a.float().cpu().numpy(), w, b.float().cpu().numpy(), 128, 128, 128, s)
            print(f"dsd {M}x{N}x{K} p={p}: relF {rel(c.cpu(), torch.from_numpy(ref)):.3e} keep {m.keep_count()} counters {cnt.kblock_iterations}")
        return

    if name == "dw":
        for (M, N, K, p) in [(1024, 1024, 1024, 0.5), (512, 768, 384, 0.3), (1024, 512, 1024, 0.9)]:
            x = rnd(M, K, 1); dy = rnd(M, N, 3)
            m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 0), M, K)
            s = sd.dropout_scale(p)
            dw = torch.empty(K, N, dtype=torch.float32, device=dev)
            sd.api.check(sd.api._lib().sd_linear_backward_dw(x.data_ptr(), m.cptr(), dy.data_ptr(), s, dw.data_ptr(),
                                                             0, M, N, K, sd.api.ctypes.c_void_p(sd.api._stream())))
            torch.cuda.synchronize()
            w = np.array(m.words(), dtype=np.uint64)
            ref = o.layer_dw(x.float().cpu().numpy(), dy.float().cpu().numpy(), w, 128, 128, s)
            print(f"dw {M}x{N}x{K} p={p}: relF {rel(dw.cpu(), torch.from_numpy(ref)):.3e}")
        return

    if name == "dx":
        for (M, N, K, p) in [(1024, 1024, 1024, 0.5), (512, 768, 384, 0.3), (1024, 512, 1024, 0.9)]:
            dy = rnd(M, N, 3); wt = rnd(K, N, 2)
            m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 0), M, K)
            s = sd.dropout_scale(p)
            dx = torch.empty(M, K, dtype=torch.float32, device=dev)
            sd.api.check(sd.api._lib().sd_linear_backward_dx(dy.data_ptr(), wt.data_ptr(), m.cptr(), s, dx.data_ptr(),
                                                             0, M, N, K, sd.api.ctypes.c_void_p(sd.api._stream())))
            torch.cuda.synchronize()
            w = np.array(m.words(), dtype=np.uint64)
            ref = o.layer_dx(dy.float().cpu().numpy(), wt.float().cpu().numpy(), w, 128, 128, s)
            zeros_ok = bool(((torch.from_numpy(ref) == 0) == (dx.cpu() == 0)).all())
            print(f"dx {M}x{N}x{K} p={p}: relF {rel(dx.cpu(), torch.from_numpy(ref)):.3e} zero-pattern {zeros_ok}")
        return

    if name == "sdd_ref":
        for (M, N, K, p) in [(1024, 1024, 512, 0.5), (512, 768, 384, 0.3)]:
            a = rnd(M, K, 1); b = rnd(K, N, 2)
            m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 0), M, N)
            c = sd.sdd_matmul(a, b, m, 1.5, out_dtype=torch.float32)
            torch.cuda.synchronize()
            w = np.array(m.words(), dtype=np.uint64)
            ref = o.sdd_matmul(a.float().cpu().numpy(), b.float().cpu().numpy(), w, 128, 128, 1.5)
            print(f"sdd_ref {M}x{N}x{K} p={p}: relF {rel(c.cpu(), torch.from_numpy(ref)):.3e}")
        return

    if name == "layer":
        M, N, K = 4096, 4096, 4096
        x = rnd(M, K, 1); w = rnd(K, N, 2); dy = rnd(M, N, 3)
        layer = sd.LinearLayer(sd.LinearVariant.sparsedrop, w, sd.DropoutSpec(0.5, 128, 128, 0))
        for _ in range(3):
            y, ctx = sd.forward(layer, x, True, 0)
            g = sd.backward(layer, ctx, dy)
        torch.cuda.synchronize()
        t0 = time.time()
        ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(20):
            y, ctx = sd.forward(layer, x, True, 0)
            g = sd.backward(layer, ctx, dy)
        ev1.record(); torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / 20
        keep = ctx.block_mask.keep_count() / ctx.block_mask.total_blocks()
        print(f"layer 4096^3 p=0.5: {ms:.3f} ms/step, dense-equiv {3*2*M*N*K/ms/1e9:.1f} TFLOP/s, executed {keep*3*2*M*N*K/ms/1e9:.1f} TFLOP/s")
        for fn, nm in [(lambda: sd.dense_gemm(x, w), "dense fwd")]:
            for _ in range(3): fn()
            ev0.record()
            for _ in range(20): fn()
            ev1.record(); torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1) / 20
            print(f"{nm}: {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TFLOP/s")
        ev0.record()
        for _ in range(20): torch.matmul(x, w)
        ev1.record(); torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / 20
        print(f"torch.matmul: {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TFLOP/s")
        return


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        run_one(sys.argv[2])
        sys.exit(0)
    names = sys.argv[1:] or TESTS
    for n in names:
        t0 = time.time()
        try:
            r = subprocess.run([sys.executable, __file__, "--one", n], timeout=float(os.environ.get("PROBE_TIMEOUT", 90)),
                               capture_output=True, text=True)
            print(r.stdout, end="")
            if r.returncode != 0:
                print(f"[{n}] FAILED rc={r.returncode}\n{r.stderr[-3000:]}")
        except subprocess.TimeoutExpired:
            print(f"[{n}] TIMEOUT (hang?) after {time.time() - t0:.0f}s")
        sys.stdout.flush()
