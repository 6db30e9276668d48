"""GPU parity at the BASELINE.json configurations the small tests cannot reach.

Every output is compared with the oracle (oracle/sd_oracle.c, pinned to the
unmodified reference) on sampled slabs, with INDEPENDENT (non-repeated) random
inputs of the reference's random_matrix distribution generated on the device:

  dW  sampled K-row slabs (mask-column blocks) x N-column slabs, over the FULL
      M reduction (the oracle runs on the slab's own columns of X and dY, with
      the column's bits of the mask as an R x 1 mask: layer.hpp:159-160 over
      transpose_mask, block_mask.cpp:117-123);
  Y   sampled 128-row blocks x N-column slabs (dsd_matmul on the row's words);
  dX  sampled 128-row blocks x K-column slabs (layer_dx on the row's words).

These shapes take the code paths the small tests do not:
  cfg3 fc2 dW (M=65536, K=3072, N=768, p=0.1): split-K with ~92 kept entries per
      split, i.e. longer than the scheduler's 64-entry smem staging, so the
      producer streams list indices from global memory and each CTA releases
      the mask workspace itself (sd_gemm.cu, `staged == false`);
  cfg4 (65536 x 8192^2, p=0.1) / cfg5 shard (rows 65536..131071 of 524288,
      row_block_offset=512, p=0.5): dW lists of 256-460 entries, no split;
  T8 8192^3 at p=0.1 and 0.5.
Bars as in test_gpu_parity.py: fp32 relF < tol and |d| <= tol
(|A||B|)_ij with tol = max(1e-5, chain_steps * 2^-24) (f32_tol below: the
tensor core's fp32 accumulation error grows linearly with the chain length); bf16 relF < 4e-3 and |d| <= 2^-7|ref| + 1e-3 (|A||B|)_ij; masks
bit-exact; dropped dX blocks exactly +0.0.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def sd():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2411_01238_b200 as sd

    sd.load_library()
    return sd


def _rand(gen, r, c):
    """random_matrix's distribution (oracles.hpp:31-41): |v| in [0.25, 1.25), random sign, bf16."""
    u = torch.rand(r, c, generator=gen, device="cuda")
    sign = torch.where(torch.rand(r, c, generator=gen, device="cuda") < 0.5, -1.0, 1.0)
    return ((0.25 + u) * sign).to(torch.bfloat16)


def _np(t):
    return t.double().cpu().numpy()


def _bits(words, R, C):
    return np.unpackbits(np.ascontiguousarray(words, dtype=np.uint64).view(np.uint8), bitorder="little")[:R * C] \
        .reshape(R, C)


def _words(bits):
    flat = np.ascontiguousarray(bits, dtype=np.uint8).reshape(-1)
    pad = (-flat.size) % 64
    return np.packbits(np.concatenate([flat, np.zeros(pad, np.uint8)]), bitorder="little").view(np.uint64)


def f32_tol(steps):
    """fp32-accumulate tolerance for a reduction chain of `steps` tcgen05 K=16
    MMA steps into one TMEM accumulator: max(1e-5, steps * 2^-24). The tensor
    core's fp32 accumulation does not round to nearest — its error grows
    LINEARLY with the chain length, not as a random walk: measured relF 4.9e-5
    over 3680 steps (cfg4 dW, p=0.1, one unsplit chain per output tile) vs
    ~1e-5 over the ~740-step chains of the split-K cfg3 dW with the same total
    reduction length, i.e. ~1.3e-8 per step = 0.22 * 2^-24 (half an fp32 ulp
    per step is the bound used). Chains up to 168 steps keep the 1e-5 bar of
    test_gpu_parity.py."""
    return max(1e-5, steps * 2.0**-24)


def check_f32(got, ref, bound, tol=1e-5):
    relf = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert relf < tol, (relf, tol)
    d = np.abs(got - ref)
    assert (d <= tol * bound + 1e-30).all(), (d - tol * bound).max()


def check_bf16(got, ref, bound):
    relf = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert relf < 4e-3, relf
    d = np.abs(got - ref)
    assert (d <= 2.0**-7 * np.abs(ref) + 1e-3 * bound).all(), d.max()


def _check_dw(oracle, plan, bits, s, kbs, nslabs):
    """dW rows of mask-column blocks `kbs` x columns `nslabs` over the full M."""
    R = bits.shape[0]
    for kb in kbs:
        xs = _np(plan.x[:, kb * 128:(kb + 1) * 128])
        col = _words(bits[:, kb:kb + 1])  # R x 1 mask: this column's keep bits
        for (n0, n1) in nslabs:
            dys = _np(plan.dy[:, n0:n1])
            ref = oracle.layer_dw(xs, dys, col, 128, 128, s, threads=THREADS)
            got = _np(plan.dw[kb * 128:(kb + 1) * 128, n0:n1])
            keep_rows = np.repeat(bits[:, kb].astype(bool), 128)
            bound = s * (np.abs(xs[keep_rows]).T @ np.abs(dys[keep_rows]))
            check_f32(got, ref, bound, tol=f32_tol(int(bits[:, kb].sum()) * 128 // 16))
            if not bits[:, kb].any():
                assert (got == 0).all()
    assert R == plan.m // 128


def _check_rows(oracle, plan, bits, s, rows, nslab, kslab):
    """Y[row block, nslab] and dX[row block, kslab] for sampled row blocks."""
    n0, n1 = nslab
    k0, k1 = kslab
    wn = _np(plan.w[:, n0:n1])
    wk = _np(plan.w[k0:k1, :])
    for r in rows:
        lo, hi = r * 128, (r + 1) * 128
        xs, dys = _np(plan.x[lo:hi]), _np(plan.dy[lo:hi])
        row = _words(bits[r:r + 1])
        ref_y = oracle.dsd_matmul(xs, row, wn, 128, 128, 128, s, threads=THREADS)
        keep_cols = np.repeat(bits[r].astype(bool), 128)
        check_bf16(_np(plan.y[lo:hi, n0:n1]), ref_y, s * (np.abs(xs[:, keep_cols]) @ np.abs(wn[keep_cols])))
        if not bits[r].any():
            assert (plan.y[lo:hi].float() == 0).all()
        sub = _words(bits[r:r + 1, k0 // 128:k1 // 128])
        ref_dx = oracle.layer_dx(dys, wk, sub, 128, 128, s, threads=THREADS)
        got = _np(plan.dx[lo:hi, k0:k1])
        check_bf16(got, ref_dx, s * (np.abs(dys) @ np.abs(wk).T))
        assert np.array_equal(got == 0, ref_dx == 0)
        # dropped blocks are +0.0 with the sign bit clear
        raw = plan.dx[lo:hi, k0:k1].view(torch.int16).cpu().numpy()
        assert (raw[ref_dx == 0] == 0).all()


def _plan(sd, gen, M, N, K, p, seed, row_block_offset=0):
    x, w, dy = _rand(gen, M, K), _rand(gen, K, N), _rand(gen, M, N)
    plan = sd.LayerPlan(x, w, dy, p, row_block_offset=row_block_offset)
    plan.forward(seed=seed)
    plan.backward()
    torch.cuda.synchronize()
    return plan


def _mask_bits(oracle, plan, p, seed, row_block_offset=0):
    words = np.array(plan.mask.words(), dtype=np.uint64)
    wo, keep = oracle.sample_mask(p, 128, 128, seed, plan.m, plan.k, row_block_offset=row_block_offset)
    assert np.array_equal(words, wo) and plan.mask.keep_count() == keep
    return _bits(words, plan.m // 128, plan.k // 128)


def test_cfg3_fc2_dw_long_split_lists(sd, oracle):
    """ViT-B fc2 (configs[2]): dW 3072 x 768 over M=65536 at p=0.1 — split-K whose
    splits hold ~92 kept blocks each (> the 64-entry staging)."""
    M, N, K, p, seed = 65536, 768, 3072, 0.1, 0x51ED
    gen = torch.Generator(device="cuda")
    gen.manual_seed(31)
    plan = _plan(sd, gen, M, N, K, p, seed)
    bits = _mask_bits(oracle, plan, p, seed)
    per_col = bits.sum(axis=0)
    assert per_col.min() > 5 * 64, per_col.min()  # every split list is longer than kListCap
    s = sd.dropout_scale(p)
    _check_dw(oracle, plan, bits, s, kbs=[0, 11, 23], nslabs=[(0, 256), (512, 768)])
    _check_rows(oracle, plan, bits, s, rows=[0, 257, 511], nslab=(0, 768), kslab=(1024, 1536))


def test_cfg4_p01_all_outputs(sd, oracle):
    """configs[3] (M=65536, K=N=8192) at p=0.1: dW lists of ~460 entries."""
    M, N, K, p, seed = 65536, 8192, 8192, 0.1, 0
    gen = torch.Generator(device="cuda")
    gen.manual_seed(41)
    plan = _plan(sd, gen, M, N, K, p, seed)
    bits = _mask_bits(oracle, plan, p, seed)
    assert plan.mask.keep_count() == 29505
    s = sd.dropout_scale(p)
    _check_dw(oracle, plan, bits, s, kbs=[0, 37, 63], nslabs=[(0, 256), (7936, 8192)])
    _check_rows(oracle, plan, bits, s, rows=[0, 301, 511], nslab=(4096, 4352), kslab=(0, 512))


def test_cfg5_shard_p05(sd, oracle):
    """configs[4] row shard 1 of 8 (global rows 65536..131071 of M=524288,
    row_block_offset=512), K=N=8192, p=0.5: shard-local mask bit-exact with
    the global mask's rows; dW lists of ~256 entries (partial dW of the shard)."""
    M, N, K, p, seed, off = 65536, 8192, 8192, 0.5, 0, 512
    gen = torch.Generator(device="cuda")
    gen.manual_seed(51)
    plan = _plan(sd, gen, M, N, K, p, seed, row_block_offset=off)
    bits = _mask_bits(oracle, plan, p, seed, row_block_offset=off)
    # the same rows of the global 4096 x 64 mask (each block row is one word at C = 64)
    gw, gkeep = oracle.sample_mask(p, 128, 128, seed, 524288, K)
    assert gkeep == 130639
    assert np.array_equal(np.array(plan.mask.words(), dtype=np.uint64), gw[off:off + 512])
    s = sd.dropout_scale(p)
    _check_dw(oracle, plan, bits, s, kbs=[5, 40], nslabs=[(0, 256), (4096, 4352)])
    _check_rows(oracle, plan, bits, s, rows=[3, 400], nslab=(7936, 8192), kslab=(2048, 2560))


@pytest.mark.parametrize("p", [0.1, 0.5])
def test_t8_all_outputs(sd, oracle, p):
    """The north-star 8192^3 layer: Y, dX and dW against the oracle."""
    M = N = K = 8192
    gen = torch.Generator(device="cuda")
    gen.manual_seed(61 + int(10 * p))
    plan = _plan(sd, gen, M, N, K, p, 3)
    bits = _mask_bits(oracle, plan, p, 3)
    s = sd.dropout_scale(p)
    _check_dw(oracle, plan, bits, s, kbs=[1, 62], nslabs=[(0, 512)])
    _check_rows(oracle, plan, bits, s, rows=[0, 33, 63], nslab=(1024, 1536), kslab=(7680, 8192))


def test_cfg4_overlapped_equals_serialized_bitwise(sd):
    """Back-to-back steps on the cfg4 dW shape with both launch overlaps on
    (mask generation on the reader release counter, early backward) against
    every launch waiting for the whole preceding grid (SD_TUNING 384)."""
    lib = sd.load_library()
    M, N, K, p = 65536, 8192, 8192, 0.3
    gen = torch.Generator(device="cuda")
    gen.manual_seed(71)
    x, w, dy = _rand(gen, M, K), _rand(gen, K, N), _rand(gen, M, N)
    outs = {}
    try:
        for tune in (0, 384):
            lib.sd_set_tuning(tune)
            plan = sd.LayerPlan(x, w, dy, p, dy_ready=True)
            for step in range(3):
                plan.forward(seed=sd.effective_seed(0, step, 0))
                plan.backward()
            torch.cuda.synchronize()
            got = [plan.y.clone(), plan.dx.clone(), plan.dw.clone()]
            outs[tune] = got
            del plan
    finally:
        lib.sd_set_tuning(0)
    for a, b in zip(outs[0], outs[384]):
        assert torch.equal(a, b)


def test_split_k_dw_deterministic(sd):
    """Split-K dW (the cfg3 fc2 shape) is bit-identical run to run: the splits are
    reduced in a fixed order (no arrival-order reduce-add), as the reference's
    serial reduction is (gemm.hpp:84-85)."""
    M, N, K, p = 65536, 768, 3072, 0.1
    gen = torch.Generator(device="cuda")
    gen.manual_seed(81)
    x, w, dy = _rand(gen, M, K), _rand(gen, K, N), _rand(gen, M, N)
    plan = sd.LayerPlan(x, w, dy, p)
    plan.forward(seed=9)
    ref = None
    for _ in range(10):
        plan.dw.fill_(float("nan"))
        plan.backward()
        torch.cuda.synchronize()
        if ref is None:
            ref = plan.dw.clone()
        else:
            assert torch.equal(plan.dw, ref)
    assert not torch.isnan(ref).any()


@pytest.mark.parametrize("p", [0.1, 0.5])
def test_cfg3_vit_mlp_full_size(sd, oracle, p):
    """configs[2] at full size: the ViT-B MLP training step, 65536 tokens,
    768 -> 3072 -> 768, SparseDrop before each Linear (GELU between). Every GEMM
    of the step against the oracle on sampled slabs of its own inputs (the
    step's bf16 intermediates), masks bit-exact from effective_seed(seed, step,
    layer) (layer.hpp:64-67); GELU' consumed exactly as computed."""
    from paper_2411_01238_b200.mlp import SparseDropMLP, gelu_grad

    M, D, H = 65536, 768, 3072
    gen = torch.Generator(device="cuda")
    gen.manual_seed(91 + int(10 * p))
    x, w1, w2, dy = _rand(gen, M, D), _rand(gen, D, H), _rand(gen, H, D), _rand(gen, M, D)
    mlp = SparseDropMLP(x, w1, w2, dy, p, seed=17)
    mlp.step(step_seed=4)
    torch.cuda.synchronize()
    s = sd.dropout_scale(p)
    f1, f2 = mlp.fc1, mlp.fc2
    b1 = _mask_bits(oracle, f1, p, oracle.effective_seed(17, 4, 0))
    b2 = _mask_bits(oracle, f2, p, oracle.effective_seed(17, 4, 1))
    assert torch.equal(mlp.act, __import__("paper_2411_01238_b200.mlp", fromlist=["gelu"]).gelu(f1.y))
    assert torch.equal(mlp.dact, gelu_grad(f1.y, f2.dx))
    # fc2: y = s (act . m1) W2, dW2 over all 65536 rows (split-K at p=0.1), dX2 (= d act)
    _check_rows(oracle, f2, b2, s, rows=[0, 300, 511], nslab=(0, 768), kslab=(2560, 3072))
    _check_dw(oracle, f2, b2, s, kbs=[0, 23], nslabs=[(256, 512)])
    # fc1: h = s (x . m0) W1, dW1 from dact over all rows, dX1
    _check_rows(oracle, f1, b1, s, rows=[7, 450], nslab=(1024, 1536), kslab=(0, 768))
    _check_dw(oracle, f1, b1, s, kbs=[0, 5], nslabs=[(0, 256), (2816, 3072)])


def test_cfg5_eight_uneven_row_shards(sd):
    """configs[4]'s decomposition over G = 8 ranks at reduced size, with uneven
    shards (60 block rows over 8 ranks: paper_2411_01238_b200.sharding): each
    shard's mask equals the global mask's rows, Y and dX rows are bit-identical
    to the unsharded layer's, and the 8 partial dWs sum to the full dW (the
    all-reduce's result) within fp32 reassociation."""
    from paper_2411_01238_b200.sharding import all_shards

    M, N, K, p, G = 128 * 60, 1024, 2048, 0.5, 8
    gen = torch.Generator(device="cuda")
    gen.manual_seed(101)
    x, w, dy = _rand(gen, M, K), _rand(gen, K, N), _rand(gen, M, N)
    full = sd.LayerPlan(x, w, dy, p)
    full.forward(seed=23)
    full.backward()
    words_full = np.array(full.mask.words(), dtype=np.uint64)
    bits_full = _bits(words_full, M // 128, K // 128)
    acc = torch.zeros(K, N, dtype=torch.float64, device="cuda")
    shards = all_shards(M, 128, G)
    assert sorted({sh.rows // 128 for sh in shards}) == [7, 8]
    for sh in shards:
        r0, r1 = sh.row0, sh.row0 + sh.rows
        pl = sd.LayerPlan(x[r0:r1].contiguous(), w, dy[r0:r1].contiguous(), p, row_block_offset=sh.row_block_offset)
        pl.forward(seed=23)
        pl.backward()
        torch.cuda.synchronize()
        b = _bits(np.array(pl.mask.words(), dtype=np.uint64), sh.rows // 128, K // 128)
        assert np.array_equal(b, bits_full[r0 // 128:r1 // 128])
        assert torch.equal(pl.y, full.y[r0:r1]) and torch.equal(pl.dx, full.dx[r0:r1])
        acc += pl.dw.double()
    relf = ((acc - full.dw.double()).norm() / full.dw.double().norm()).item()
    assert relf < 1e-6, relf
