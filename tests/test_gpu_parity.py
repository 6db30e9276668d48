"""GPU parity: the B200 CUDA path (through the C-ABI) against the oracle.

Bars (stated per test):
  * masks, keep counts, index lists, transposes, retiles: bit-exact;
  * GEMMs vs the double-precision oracle on the SAME bf16-rounded inputs:
      fp32 outputs  relative Frobenius < 1e-5 and |d| <= 1e-5 * (|A||B|)_ij
      bf16 outputs  relative Frobenius < 4e-3 and |d| <= 2^-7 |ref| + 1e-3 (|A||B|)_ij
  * structure: dropped output tiles (sdd) and fully dropped rows (dsd) are
    exactly +0.0; dsd at p=0 equals dense bitwise; dsd on X equals dense on
    mask_select(X) bitwise.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

F32_RELF = 1e-5
BF16_RELF = 4e-3


@pytest.fixture(scope="module")
def sd():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2411_01238_b200 as sd

    lib = sd.load_library()  # native code must be loaded; no fallback exists
    assert lib.sd_device_count() >= 1
    return sd


def _dev(o, r, c, seed):
    return torch.from_numpy(o.random_matrix(r, c, seed)).to(torch.bfloat16).cuda()


def _np(t):
    return t.double().cpu().numpy()


def _abs_prod(a, b):
    return np.abs(a) @ np.abs(b)


def check_f32(got, ref, bound):
    d = np.abs(got - ref)
    relf = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert relf < F32_RELF, relf
    assert (d <= 1e-5 * bound + 1e-30).all(), d.max()


def check_bf16(got, ref, bound):
    d = np.abs(got - ref)
    relf = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert relf < BF16_RELF, relf
    assert (d <= 2.0**-7 * np.abs(ref) + 1e-3 * bound).all(), d.max()


def words_np(mask):
    return np.array(mask.words(), dtype=np.uint64)


# --------------------------------------------------------------------------- masks

MASK_GEOMS = [
    (1024, 1024, 0), (4096, 4096, 0), (65536, 768, 0x238275BC38FCBE91), (65536, 3072, 5),
    (65536, 8192, 0), (8192, 8192, 0), (128 * 37, 128 * 19, 3), (128, 128, 1), (128 * 5, 128 * 70, 2),
    # > 32768 blocks or > 4096 rows: counts and orders from the ticketed last
    # block instead of the inline order block (sd_mask.cu)
    (524288, 8192, 0), (128 * 4100, 256, 7),
]


@pytest.mark.parametrize("rows,cols,seed", MASK_GEOMS)
@pytest.mark.parametrize("p", [0.0, 0.1, 0.5, 0.9])
def test_mask_bit_exact(sd, oracle, rows, cols, seed, p):
    m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, seed), rows, cols)
    w, keep = oracle.sample_mask(p, 128, 128, seed, rows, cols)
    R, C = rows // 128, cols // 128
    assert np.array_equal(words_np(m), w)
    assert m.keep_count() == keep
    rc = m.row_cnt_device().cpu().numpy()
    ri = m.row_idx_device().cpu().numpy()
    for r in range(R):
        assert ri[r, : rc[r]].tolist() == oracle.kept_blocks_in_row(w, R, C, r)
    wt = oracle.transpose_mask(w, R, C)
    cc = m.col_cnt_device().cpu().numpy()
    ci = m.col_idx_device().cpu().numpy()
    for c in range(C):
        assert ci[c, : cc[c]].tolist() == oracle.kept_blocks_in_row(wt, C, R, c)
    ro = m.row_order_device().cpu().numpy()
    assert sorted(ro.tolist()) == list(range(R))
    assert all(rc[ro[i]] >= rc[ro[i + 1]] for i in range(R - 1))  # heaviest first
    co = m.col_order_device().cpu().numpy()
    assert sorted(co.tolist()) == list(range(C))
    assert all(cc[co[i]] >= cc[co[i + 1]] for i in range(C - 1))


def test_mask_golden(sd, golden):
    for c in golden["masks"]["cases"]:
        if c["m_blk"] < 64 or c["rows"] * c["cols"] // (c["m_blk"] * c["k_blk"]) > 2**20:
            continue
        m = sd.sample_mask(sd.DropoutSpec(c["p"], c["m_blk"], c["k_blk"], c["seed"]), c["rows"], c["cols"])
        assert m.keep_count() == c["keep_count"], c["name"]
        if "words" in c:
            assert [hex(x) for x in m.words()] == c["words"], c["name"]
        if "row_lists" in c:
            for r in range(c["block_rows"]):
                assert sd.kept_blocks_in_row(m, r) == c["row_lists"][r]


def test_cfg1_word(sd):
    m = sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, 0), 1024, 1024)
    assert m.words() == [0xE43D829A90C95084] and m.keep_count() == 25


@pytest.mark.parametrize("offset,nrows", [(0, 64), (64, 64), (448, 64), (7, 13)])
def test_mask_shard_offsets(sd, oracle, offset, nrows):
    """A row shard's locally generated mask equals the global mask's rows."""
    m = sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, 0), nrows * 128, 8192, row_block_offset=offset)
    gw, _ = oracle.sample_mask(0.5, 128, 128, 0, 512 * 128, 8192)
    sw, keep = oracle.sample_mask(0.5, 128, 128, 0, nrows * 128, 8192, row_block_offset=offset)
    assert np.array_equal(words_np(m), sw) and m.keep_count() == keep
    assert np.array_equal(sw, gw[offset: offset + nrows])  # C = 64: one word per block row


def test_transpose_and_retile(sd, oracle, golden):
    m = sd.sample_mask(sd.DropoutSpec(0.45, 128, 256, 13), 128 * 12, 256 * 9)
    w = words_np(m)
    t = sd.transpose_mask(m)
    assert np.array_equal(words_np(t), oracle.transpose_mask(w, 12, 9))
    assert (t.block_rows(), t.block_cols(), t.m_blk(), t.k_blk()) == (9, 12, 256, 128)
    assert np.array_equal(words_np(sd.transpose_mask(t)), w)  # involution
    r = sd.retile(m, 1, 2)
    assert np.array_equal(words_np(r), oracle.retile(w, 12, 9, 128, 256, 1, 2))
    assert r.keep_count() == 2 * m.keep_count()
    with pytest.raises(ValueError):
        sd.retile(m, 3, 1)
    for c in golden["masks"]["retile"]:
        base = sd.sample_mask(sd.DropoutSpec(c["p"], c["m_blk"], c["k_blk"], c["seed"]), c["rows"], c["cols"])
        got = sd.retile(base, c["split_m"], c["split_k"])
        assert [hex(x) for x in got.words()] == c["words"]


def test_mask_from_words_roundtrip(sd, oracle):
    w, keep = oracle.sample_mask(0.3, 128, 128, 21, 128 * 9, 128 * 7)
    m = sd.mask_from_words(9, 7, 128, 128, w.tolist())
    assert m.keep_count() == keep and np.array_equal(words_np(m), w)
    for r in range(9):
        assert sd.kept_blocks_in_row(m, r) == oracle.kept_blocks_in_row(w, 9, 7, r)
    with pytest.raises(ValueError, match="padding|past the block grid"):
        sd.mask_from_words(3, 3, 128, 128, [2**64 - 1])
    with pytest.raises(IndexError):
        sd.kept_blocks_in_row(m, 9)


def test_mask_validation(sd):
    with pytest.raises(ValueError, match="m_blk"):
        sd.sample_mask(sd.DropoutSpec(0.5, 100, 128, 0), 1024, 1024)
    with pytest.raises(ValueError, match="k_blk"):
        sd.sample_mask(sd.DropoutSpec(0.5, 128, 100, 0), 1024, 1024)
    with pytest.raises(ValueError):
        sd.sample_mask(sd.DropoutSpec(1.0, 128, 128, 0), 1024, 1024)


# --------------------------------------------------------------------------- dense

# (2560, 2048, 512) and (2304, 2304, 320) have >= 74 256x256 pair tiles and run
# on the 2-CTA (cta_group::2) kernel; the others on the 1-CTA kernel
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 512, 256), (1024, 1024, 1024), (384, 640, 192),
                                   (512, 384, 4096), (2560, 2048, 512), (2304, 2304, 320)])
@pytest.mark.parametrize("layout", ["nn", "nt", "tn"])
def test_dense_gemm(sd, oracle, M, N, K, layout):
    a = _dev(oracle, M, K, 1)
    b = _dev(oracle, K, N, 2)
    an, bn = _np(a), _np(b)
    ref = oracle.dense_gemm(an, bn)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    lib = sd.load_library()
    for dt, code in [(torch.float32, 0), (torch.bfloat16, 1)]:
        c = torch.empty(M, N, dtype=dt, device="cuda")
        if layout == "nn":
            sd.dense_gemm(a, b, out=c)
        elif layout == "nt":
            bt = b.t().contiguous()
            sd.api.check(lib.sd_dense_gemm_nt(a.data_ptr(), bt.data_ptr(), c.data_ptr(), code, M, N, K, st))
        else:
            at = a.t().contiguous()
            sd.api.check(lib.sd_dense_gemm_tn(at.data_ptr(), b.data_ptr(), c.data_ptr(), code, M, N, K, st))
        torch.cuda.synchronize()
        (check_f32 if dt == torch.float32 else check_bf16)(_np(c), ref, _abs_prod(an, bn))


@pytest.mark.parametrize("layout", ["nn", "nt", "tn"])
def test_dense_2cta_equals_1cta_bitwise(sd, oracle, layout):
    """The 2-CTA kernel accumulates every output element over the same K16
    steps in the same order as the 1-CTA kernel: results are bit-identical."""
    M, N, K = 4096, 2048, 768
    a = _dev(oracle, M, K, 1)
    b = _dev(oracle, K, N, 2)
    lib = sd.load_library()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    outs = {}
    try:
        for tune in (1 | 16, 1):
            lib.sd_set_tuning(tune)
            for dt, code in [(torch.float32, 0), (torch.bfloat16, 1)]:
                c = torch.empty(M, N, dtype=dt, device="cuda")
                if layout == "nn":
                    sd.dense_gemm(a, b, out=c)
                elif layout == "nt":
                    bt = b.t().contiguous()
                    sd.api.check(lib.sd_dense_gemm_nt(a.data_ptr(), bt.data_ptr(), c.data_ptr(), code, M, N, K, st))
                else:
                    at = a.t().contiguous()
                    sd.api.check(lib.sd_dense_gemm_tn(at.data_ptr(), b.data_ptr(), c.data_ptr(), code, M, N, K, st))
                outs[(tune, code)] = c
        torch.cuda.synchronize()
    finally:
        lib.sd_set_tuning(0)
    for code in (0, 1):
        assert torch.equal(outs[(1 | 16, code)], outs[(1, code)])


# --------------------------------------------------------------------------- dsd forward

DSD_CASES = [(1024, 1024, 1024, 0.5), (512, 768, 384, 0.3), (1024, 512, 1024, 0.9), (256, 384, 2048, 0.1),
             (2048, 256, 512, 0.7)]


@pytest.mark.parametrize("M,N,K,p", DSD_CASES)
def test_dsd_matmul(sd, oracle, M, N, K, p):
    a, b = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2)
    m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 4), M, K)
    s = sd.dropout_scale(p)
    w = words_np(m)
    an, bn = _np(a), _np(b)
    ref = oracle.dsd_matmul(an, w, bn, 128, 128, 128, s)
    masked = oracle.dsd_matmul(an, w, np.abs(bn), 128, 128, 128, 1.0)  # noqa: F841 (bound below)
    bound = s * _abs_prod(np.abs(an), np.abs(bn))
    cnt = sd.KernelCounters()
    c32 = sd.dsd_matmul(a, m, b, s, counters=cnt, out_dtype=torch.float32)
    c16 = sd.dsd_matmul(a, m, b, s, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    check_f32(_np(c32), ref, bound)
    check_bf16(_np(c16), ref, bound)
    # KernelCounters (gemm.hpp:31-37) with n_blk = 128: kept_in_row * N/128
    rc = m.row_cnt_device().cpu().numpy()
    assert cnt.kblock_per_tile_row == [int(v) * (N // 128) for v in rc]
    # fully dropped rows are exactly +0.0
    for r in np.where(rc == 0)[0]:
        blk = c32[r * 128:(r + 1) * 128]
        assert bool((blk == 0).all()) and not bool(torch.signbit(blk).any())


def test_dsd_equals_dense_on_masked_input_bitwise(sd, oracle):
    """gemm.hpp:14-22 contract on device: skipping a block == multiplying zeros."""
    M, N, K = 1024, 512, 1024
    a, b = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2)
    m = sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, 9), M, K)
    w = words_np(m)
    am = a.clone()
    for r in range(M // 128):
        for c in range(K // 128):
            b_ = r * (K // 128) + c
            if not (int(w[b_ >> 6]) >> (b_ & 63)) & 1:
                am[r * 128:(r + 1) * 128, c * 128:(c + 1) * 128] = 0
    c_sparse = sd.dsd_matmul(a, m, b, 1.0, out_dtype=torch.float32)
    c_dense = sd.dense_gemm(am, b, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(c_sparse, c_dense)


def test_dsd_p0_equals_dense_bitwise(sd, oracle):
    M, N, K = 512, 768, 1024
    a, b = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2)
    m = sd.sample_mask(sd.DropoutSpec(0.0, 128, 128, 9), M, K)
    assert m.keep_count() == m.total_blocks()
    torch.cuda.synchronize()
    assert torch.equal(sd.dsd_matmul(a, m, b, 1.0, out_dtype=torch.float32),
                       sd.dense_gemm(a, b, out_dtype=torch.float32))


def test_dsd_empty_rows_vit_fc1(sd, oracle):
    """ViT fc1 at p=0.5 has fully dropped M-block rows."""
    M, K, N = 65536, 768, 3072
    seed = sd.effective_seed(0, 0, 0)
    m = sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, seed), M, K)
    rc = m.row_cnt_device().cpu().numpy()
    empty = np.where(rc == 0)[0]
    assert len(empty) == 8
    x, w = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2)
    y = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    sd.dsd_matmul(x, m, w, 2.0, out=y)
    torch.cuda.synchronize()
    for r in empty:
        blk = y[r * 128:(r + 1) * 128]
        assert bool((blk == 0).all()) and not bool(torch.signbit(blk).any())
    # spot rows vs oracle
    words = words_np(m)
    xn, wn = _np(x), _np(w)
    for r in [int(empty[0]), 0, 17, 511]:
        ref = oracle.dsd_matmul(xn, words, wn, 128, 128, 128, 2.0, row_lo=r * 128, row_hi=(r + 1) * 128)
        check_bf16(_np(y[r * 128:(r + 1) * 128]), ref, 2.0 * _abs_prod(np.abs(xn[r * 128:(r + 1) * 128]), np.abs(wn)))


# --------------------------------------------------------------------------- backward

@pytest.mark.parametrize("M,N,K,p", DSD_CASES)
def test_layer_dw(sd, oracle, M, N, K, p):
    x, dy = _dev(oracle, M, K, 1), _dev(oracle, M, N, 3)
    m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 6), M, K)
    s = sd.dropout_scale(p)
    dw = torch.full((K, N), float("nan"), dtype=torch.float32, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    sd.api.check(sd.load_library().sd_linear_backward_dw(x.data_ptr(), m.cptr(), dy.data_ptr(), s, dw.data_ptr(),
                                                         0, M, N, K, st))
    torch.cuda.synchronize()
    w = words_np(m)
    xn, dyn = _np(x), _np(dy)
    ref = oracle.layer_dw(xn, dyn, w, 128, 128, s)
    check_f32(_np(dw), ref, s * _abs_prod(np.abs(xn).T, np.abs(dyn)))
    cc = m.col_cnt_device().cpu().numpy()
    for c in np.where(cc == 0)[0]:  # all-dropped mask columns: dW rows exactly zero
        assert bool((dw[c * 128:(c + 1) * 128] == 0).all())


@pytest.mark.parametrize("M,N,K,p", DSD_CASES)
def test_layer_dx(sd, oracle, M, N, K, p):
    dy, wt = _dev(oracle, M, N, 3), _dev(oracle, K, N, 2)
    m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 8), M, K)
    s = sd.dropout_scale(p)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for dt, code in [(torch.float32, 0), (torch.bfloat16, 1)]:
        dx = torch.full((M, K), float("nan"), dtype=dt, device="cuda")
        sd.api.check(sd.load_library().sd_linear_backward_dx(dy.data_ptr(), wt.data_ptr(), m.cptr(), s,
                                                             dx.data_ptr(), code, M, N, K, st))
        torch.cuda.synchronize()
        w = words_np(m)
        dyn, wn = _np(dy), _np(wt)
        ref = oracle.layer_dx(dyn, wn, w, 128, 128, s)
        bound = s * _abs_prod(np.abs(dyn), np.abs(wn).T)
        got = _np(dx)
        (check_f32 if dt == torch.float32 else check_bf16)(got, ref, bound)
        # dropped tiles: exactly +0.0 (sign bit clear), kept tiles never zero here
        zero = ref == 0
        assert np.array_equal(got == 0, zero)
        assert not bool(torch.signbit(dx.float()[torch.from_numpy(zero).cuda()]).any())


@pytest.mark.parametrize("n_blk", [128, 256])
def test_sdd_reference_form(sd, oracle, n_blk):
    """sdd_matmul(a, b, mask) exactly as gemm.hpp:176-213 (b row-major)."""
    M, N, K = 1024, 1024, 512
    a, b = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2)
    m = sd.sample_mask(sd.DropoutSpec(0.5, 128, n_blk, 3), M, N)
    cnt = sd.KernelCounters()
    c = sd.sdd_matmul(a, b, m, 1.5, counters=cnt, out_dtype=torch.float32)
    torch.cuda.synchronize()
    an, bn = _np(a), _np(b)
    ref = oracle.sdd_matmul(an, bn, words_np(m), 128, n_blk, 1.5)
    check_f32(_np(c), ref, 1.5 * _abs_prod(np.abs(an), np.abs(bn)))
    assert np.array_equal(_np(c) == 0, ref == 0)
    rc = m.row_cnt_device().cpu().numpy()
    assert cnt.kblock_per_tile_row == [int(v) * (n_blk // 128) * (K // 128) for v in rc]


def test_layer_golden_256(sd, oracle, golden):
    """Device layer fwd+bwd vs the reference's own forward/backward (double)."""
    g = golden["layer_256"]
    M, N, K, mb, kb, seed, step, li = [int(v) for v in g["meta"]]
    p = float(g["p"][0])
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    layer = sd.LinearLayer(sd.LinearVariant.sparsedrop, w, sd.DropoutSpec(p, mb, kb, seed), layer_index=li)
    y, ctx = sd.forward(layer, x, True, step, out_dtype=torch.float32)
    gr = sd.backward(layer, ctx, dy, dx_dtype=torch.float32)
    torch.cuda.synchronize()
    assert np.array_equal(words_np(ctx.block_mask), g["words"])
    s = sd.dropout_scale(p)
    xn, wn, dyn = _np(x), _np(w), _np(dy)
    check_f32(_np(y), g["y"].astype(np.float64), s * _abs_prod(np.abs(xn), np.abs(wn)))
    check_f32(_np(gr.dx), g["dx"].astype(np.float64), s * _abs_prod(np.abs(dyn), np.abs(wn).T))
    check_f32(_np(gr.dw), g["dw"].astype(np.float64), s * _abs_prod(np.abs(xn).T, np.abs(dyn)))


def test_layer_plan_matches_api(sd, oracle):
    M, N, K, p = 1024, 768, 1024, 0.4
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    plan = sd.LayerPlan(x, w, dy, p)
    seed = sd.effective_seed(0, 5, 0)
    plan.forward(seed)
    plan.backward()
    layer = sd.LinearLayer(sd.LinearVariant.sparsedrop, w, sd.DropoutSpec(p, 128, 128, 0))
    y, ctx = sd.forward(layer, x, True, 5)
    gr = sd.backward(layer, ctx, dy)
    torch.cuda.synchronize()
    assert torch.equal(plan.y, y) and torch.equal(plan.dx, gr.dx) and torch.equal(plan.dw, gr.dw)
    # dense baseline of the plan
    plan.dense_forward()
    plan.dense_backward()
    torch.cuda.synchronize()
    assert torch.equal(plan.y, sd.dense_gemm(x, w))


def test_inference_and_dense_variant(sd, oracle):
    M, N, K = 256, 256, 384
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    layer = sd.LinearLayer(sd.LinearVariant.sparsedrop, w, sd.DropoutSpec(0.5, 128, 128, 0))
    y, ctx = sd.forward(layer, x, False, 0, out_dtype=torch.float32)  # inference: dense
    gr = sd.backward(layer, ctx, dy, dx_dtype=torch.float32)
    torch.cuda.synchronize()
    xn, wn, dyn = _np(x), _np(w), _np(dy)
    check_f32(_np(y), oracle.dense_gemm(xn, wn), _abs_prod(np.abs(xn), np.abs(wn)))
    check_f32(_np(gr.dx), oracle.dense_gemm(dyn, wn.T), _abs_prod(np.abs(dyn), np.abs(wn).T))
    check_f32(_np(gr.dw), oracle.dense_gemm(xn.T, dyn), _abs_prod(np.abs(xn).T, np.abs(dyn)))


# --------------------------------------------------------------------------- full-size properties

def test_cfg2_4096_sampled_rows(sd, oracle):
    """configs[1] size: sampled output row blocks vs the oracle, plus structure."""
    M = N = K = 4096
    p = 0.5
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    plan = sd.LayerPlan(x, w, dy, p)
    plan.forward(seed=0)
    plan.backward()
    torch.cuda.synchronize()
    words = words_np(plan.mask)
    wo, keep = oracle.sample_mask(p, 128, 128, 0, M, K)
    assert np.array_equal(words, wo) and plan.mask.keep_count() == keep == 496
    s = sd.dropout_scale(p)
    xn, wn, dyn = _np(x), _np(w), _np(dy)
    for r in [0, 13, 31]:
        lo, hi = r * 128, (r + 1) * 128
        ref_y = oracle.dsd_matmul(xn, words, wn, 128, 128, 128, s, row_lo=lo, row_hi=hi)
        check_bf16(_np(plan.y[lo:hi]), ref_y, s * _abs_prod(np.abs(xn[lo:hi]), np.abs(wn)))
        ref_dx = oracle.layer_dx(dyn, wn, words, 128, 128, s, row_lo=lo, row_hi=hi)
        check_bf16(_np(plan.dx[lo:hi]), ref_dx, s * _abs_prod(np.abs(dyn[lo:hi]), np.abs(wn).T))
        assert np.array_equal(_np(plan.dx[lo:hi]) == 0, ref_dx == 0)
    for c in [0, 21]:
        lo, hi = c * 128, (c + 1) * 128
        ref_dw = oracle.layer_dw(xn, dyn, words, 128, 128, s, krow_lo=lo, krow_hi=hi)
        check_f32(_np(plan.dw[lo:hi]), ref_dw, s * _abs_prod(np.abs(xn[:, lo:hi]).T, np.abs(dyn)))


def test_dw_linearity_in_row_shards(sd, oracle):
    """Row-sharded dW: the sum of shard-local partial dWs (each with its own
    locally generated mask rows) equals the single-GPU dW (fp32 tolerance)."""
    M, N, K, p, G = 2048, 512, 1024, 0.5, 4
    x, dy = _dev(oracle, M, K, 1), _dev(oracle, M, N, 3)
    w = _dev(oracle, K, N, 2)
    full = sd.LayerPlan(x, w, dy, p)
    full.forward(seed=11)
    full.backward()
    parts = torch.zeros(K, N, dtype=torch.float64, device="cuda")
    rows = M // G
    ys = []
    for g in range(G):
        xs, dys = x[g * rows:(g + 1) * rows].contiguous(), dy[g * rows:(g + 1) * rows].contiguous()
        sp = sd.LayerPlan(xs, w, dys, p, row_block_offset=g * rows // 128)
        sp.forward(seed=11)
        sp.backward()
        parts += sp.dw.double()
        ys.append((sp.y.clone(), sp.dx.clone()))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([a for a, _ in ys]), full.y)
    assert torch.equal(torch.cat([b for _, b in ys]), full.dx)
    relf = ((parts - full.dw.double()).norm() / full.dw.double().norm()).item()
    assert relf < 1e-6


def test_api_errors_through_cabi(sd, oracle):
    a = _dev(oracle, 256, 256, 1)
    b = _dev(oracle, 384, 256, 2)
    with pytest.raises(ValueError, match="gemm shape mismatch"):
        sd.dense_gemm(a, b)
    m = sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, 0), 512, 256)
    with pytest.raises(ValueError, match="mask geometry"):
        sd.dsd_matmul(a, m, _dev(oracle, 256, 256, 2), 2.0)
    bad = torch.empty(100, 256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="m_blk"):
        sd.dense_gemm(bad, _dev(oracle, 256, 256, 2))


def test_native_library_loaded(sd):
    """The compute ran in libsparsedrop_b200.so (launch counter advanced)."""
    import os

    n0 = sd.launch_count()
    sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, 0), 1024, 1024)
    assert sd.launch_count() == n0 + 1
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert "libsparsedrop_b200.so" in maps


def test_mlp_block_composition(sd, oracle):
    """ViT-style MLP block (cfg3 shape family): each stage vs the oracle on the
    same bf16 intermediates, masks from effective_seed(seed, step, layer)."""
    from paper_2411_01238_b200.mlp import SparseDropMLP, gelu_grad, gelu_grad_reference, gelu_reference

    M, D, H, p = 1024, 256, 768, 0.5
    x, w1, w2, dy = _dev(oracle, M, D, 1), _dev(oracle, D, H, 2), _dev(oracle, H, D, 3), _dev(oracle, M, D, 4)
    mlp = SparseDropMLP(x, w1, w2, dy, p, seed=5)
    y, dx, dw1, dw2 = mlp.step(step_seed=9)
    torch.cuda.synchronize()
    s = sd.dropout_scale(p)
    w0, _ = oracle.sample_mask(p, 128, 128, oracle.effective_seed(5, 9, 0), M, D)
    w1m, _ = oracle.sample_mask(p, 128, 128, oracle.effective_seed(5, 9, 1), M, H)
    assert np.array_equal(words_np(mlp.fc1.mask), w0) and np.array_equal(words_np(mlp.fc2.mask), w1m)
    xn, w1n, w2n, dyn = _np(x), _np(w1), _np(w2), _np(dy)
    h = mlp.fc1.y
    check_bf16(_np(h), oracle.dsd_matmul(xn, w0, w1n, 128, 128, 128, s), s * _abs_prod(np.abs(xn), np.abs(w1n)))
    act = _np(mlp.act)
    # the fused activation kernels vs the torch fp32 reference (bf16 outputs: 1 ulp)
    assert (mlp.act.float() - gelu_reference(h).float()).abs().max().item() <= 2**-7 * (
        gelu_reference(h).float().abs().max().item())
    gref = gelu_grad_reference(h, mlp.fc2.dx).float()
    assert ((mlp.dact.float() - gref).abs() <= 2**-7 * gref.abs() + 1e-6).all()
    check_bf16(_np(y), oracle.dsd_matmul(act, w1m, w2n, 128, 128, 128, s), s * _abs_prod(np.abs(act), np.abs(w2n)))
    check_f32(_np(dw2), oracle.layer_dw(act, dyn, w1m, 128, 128, s), s * _abs_prod(np.abs(act).T, np.abs(dyn)))
    da_ref = oracle.layer_dx(dyn, w2n, w1m, 128, 128, s)
    check_bf16(_np(mlp.fc2.dx), da_ref, s * _abs_prod(np.abs(dyn), np.abs(w2n).T))
    dact = _np(mlp.dact)
    assert torch.equal(mlp.dact, gelu_grad(h, mlp.fc2.dx))
    check_f32(_np(dw1), oracle.layer_dw(xn, dact, w0, 128, 128, s), s * _abs_prod(np.abs(xn).T, np.abs(dact)))
    check_bf16(_np(dx), oracle.layer_dx(dact, w1n, w0, 128, 128, s), s * _abs_prod(np.abs(dact), np.abs(w1n).T))


def test_cfg4_sampled_rows(sd, oracle):
    """configs[3] size (M=65536, K=N=8192, p=0.3): sampled row blocks of Y and dX."""
    M, N, K, p = 65536, 8192, 8192, 0.3
    x, w, dy = _dev(oracle, 1024, K, 1), _dev(oracle, K, N, 2), _dev(oracle, 1024, N, 3)
    # tile the 1024-row generated blocks to full size (the oracle only needs the sampled rows)
    x = x.repeat(M // 1024, 1)
    dy = dy.repeat(M // 1024, 1)
    plan = sd.LayerPlan(x, w, dy, p)
    plan.forward(seed=0)
    plan.backward()
    torch.cuda.synchronize()
    words = words_np(plan.mask)
    wo, keep = oracle.sample_mask(p, 128, 128, 0, M, K)
    assert np.array_equal(words, wo) and plan.mask.keep_count() == keep == 22942
    s = sd.dropout_scale(p)
    wn = _np(w)
    for r in [0, 301]:
        lo, hi = r * 128, (r + 1) * 128
        xs, dys = _np(x[lo:hi]), _np(dy[lo:hi])
        # the oracle wants full matrices; pass the slab with a slab-local mask row
        rw, _ = oracle.sample_mask(p, 128, 128, 0, 128, K, row_block_offset=r)
        ref_y = oracle.dsd_matmul(xs, rw, wn, 128, 128, 128, s)
        check_bf16(_np(plan.y[lo:hi]), ref_y, s * _abs_prod(np.abs(xs), np.abs(wn)))
        ref_dx = oracle.layer_dx(dys, wn, rw, 128, 128, s)
        check_bf16(_np(plan.dx[lo:hi]), ref_dx, s * _abs_prod(np.abs(dys), np.abs(wn).T))
        assert np.array_equal(_np(plan.dx[lo:hi]) == 0, ref_dx == 0)


@pytest.mark.parametrize("p", [0.0, 0.5])
def test_layer_dw_split_k(sd, oracle, p):
    """Few output tiles over a long reduction: split-K with TMA reduce-add (fp32)."""
    M, N, K = 16384, 512, 256
    x, dy = _dev(oracle, M, K, 1), _dev(oracle, M, N, 3)
    m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 6), M, K)
    s = sd.dropout_scale(p)
    dw = torch.full((K, N), float("nan"), dtype=torch.float32, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    sd.api.check(sd.load_library().sd_linear_backward_dw(x.data_ptr(), m.cptr(), dy.data_ptr(), s, dw.data_ptr(),
                                                         0, M, N, K, st))
    dwt = torch.empty(K, N, dtype=torch.float32, device="cuda")
    sd.api.check(sd.load_library().sd_dense_gemm_tn(x.data_ptr(), dy.data_ptr(), dwt.data_ptr(), 0, K, N, M, st))
    torch.cuda.synchronize()
    xn, dyn = _np(x), _np(dy)
    bound = s * _abs_prod(np.abs(xn).T, np.abs(dyn))
    check_f32(_np(dw), oracle.layer_dw(xn, dyn, words_np(m), 128, 128, s), bound)
    check_f32(_np(dwt), oracle.dense_gemm(xn.T, dyn), _abs_prod(np.abs(xn).T, np.abs(dyn)))
