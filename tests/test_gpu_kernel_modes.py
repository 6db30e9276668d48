"""Kernel-mode parity (GPU): every unit kind / kernel instantiation of the GEMM
path must produce BIT-IDENTICAL outputs — they reduce each output element over
the same 16-deep MMA steps in the same order and differ only in tiling:

  narrow  sd_gemm_kernel<false>: 128 x 256 units, double-buffered TMEM
  wide    sd_gemm_kernel<true>:  128 x 512 units (two N=256 MMAs per A tile)
  union   sd_gemm2_kernel union mode: 2-CTA pairs over the union of two rows'
          kept lists, a dropped A half loaded as an out-of-bounds (zero) box

plus one oracle check of the wide path (gemm.hpp:133-213 semantics)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

NARROW, WIDE = 1 | 64, 1 | 32  # sd_set_tuning bits (include/sparsedrop_b200.h)


@pytest.fixture(scope="module")
def sd():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2411_01238_b200 as sd

    sd.load_library()
    return sd


def _dev(o, r, c, seed):
    return torch.from_numpy(o.random_matrix(r, c, seed)).to(torch.bfloat16).cuda()


def _layer_outputs(sd, x, w, dy, p, seed, fused=True):
    plan = sd.LayerPlan(x, w, dy, p)
    plan.forward(seed)
    if fused:
        plan.backward()
    else:
        plan.backward_dw()
        plan.backward_dx()
    torch.cuda.synchronize()
    return [plan.y.clone(), plan.dx.clone(), plan.dw.clone()]


# (M, N, K, p): square, ragged N (640 = 512 + 128), narrow N (<= 256 -> narrow
# even when wide is forced), MLP-like small dW outputs (split-K), p = 0.9 with
# fully dropped rows, p = 0
LAYER_CASES = [(1024, 1024, 1024, 0.5), (1024, 640, 1152, 0.3), (512, 256, 768, 0.5), (4096, 768, 384, 0.1),
               (2048, 3072, 768, 0.9), (1024, 1536, 512, 0.0)]


@pytest.mark.parametrize("M,N,K,p", LAYER_CASES)
@pytest.mark.parametrize("fused", [True, False])
def test_layer_wide_equals_narrow_bitwise(sd, oracle, M, N, K, p, fused):
    lib = sd.load_library()
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    try:
        lib.sd_set_tuning(NARROW)
        ref = _layer_outputs(sd, x, w, dy, p, 21, fused)
        lib.sd_set_tuning(WIDE)
        got = _layer_outputs(sd, x, w, dy, p, 21, fused)
    finally:
        lib.sd_set_tuning(0)
    # split-K dW included: its splits are reduced in a fixed order (split 0
    # stores, split j adds after split j-1), so wide and narrow agree bitwise
    for name, a, b in zip(("y", "dx", "dw"), ref, got):
        assert torch.equal(a, b), name


@pytest.mark.parametrize("n_blk", [128, 256])
def test_generic_sdd_and_dsd_wide_equals_narrow(sd, oracle, n_blk):
    """The generic C-ABI dsd / sdd entry points (reference TileConfig forms)."""
    lib = sd.load_library()
    M, N, K = 1024, 1024, 768
    a, b = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2)
    m_dsd = sd.sample_mask(sd.DropoutSpec(0.4, 128, 128, 5), M, K)
    m_sdd = sd.sample_mask(sd.DropoutSpec(0.4, 128, n_blk, 6), M, N)
    outs = {}
    try:
        for tune in (NARROW, WIDE):
            lib.sd_set_tuning(tune)
            outs[tune] = (sd.dsd_matmul(a, m_dsd, b, 1.5, out_dtype=torch.float32),
                          sd.sdd_matmul(a, b, m_sdd, 1.5, out_dtype=torch.bfloat16))
        torch.cuda.synchronize()
    finally:
        lib.sd_set_tuning(0)
    for u, v in zip(outs[NARROW], outs[WIDE]):
        assert torch.equal(u, v)


def test_wide_forward_matches_oracle(sd, oracle):
    lib = sd.load_library()
    M, N, K, p = 512, 1280, 640, 0.5
    x, w = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2)
    m = sd.sample_mask(sd.DropoutSpec(p, 128, 128, 3), M, K)
    s = sd.dropout_scale(p)
    try:
        lib.sd_set_tuning(WIDE)
        y = sd.dsd_matmul(x, m, w, s, out_dtype=torch.float32)
        torch.cuda.synchronize()
    finally:
        lib.sd_set_tuning(0)
    words = np.array(m.words(), dtype=np.uint64)
    xn, wn = x.double().cpu().numpy(), w.double().cpu().numpy()
    ref = oracle.dsd_matmul(xn, words, wn, 128, 128, 128, s)
    bound = s * (np.abs(xn) @ np.abs(wn))
    got = y.double().cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5
    assert (np.abs(got - ref) <= 1e-5 * bound + 1e-30).all()


def _pair_lists(bits):
    """Pairs of rows (2p, 2p+1) of a (R, C) keep matrix -> union lists of
    (block << 2) | owner bits, the 2-CTA kernel's union-mode format."""
    R, C = bits.shape
    cnt = np.zeros(R // 2, np.int32)
    idx = np.zeros((R // 2, C), np.int32)
    for q in range(R // 2):
        own = bits[2 * q].astype(np.int32) | (bits[2 * q + 1].astype(np.int32) << 1)
        cols = np.nonzero(own)[0]
        cnt[q] = len(cols)
        idx[q, :len(cols)] = (cols << 2) | own[cols]
    return torch.from_numpy(cnt).cuda(), torch.from_numpy(idx).cuda()


@pytest.mark.parametrize("p", [0.3, 0.8])
def test_union_2cta_dsd_bitwise(sd, oracle, p):
    """2-CTA union mode (dev entry sd_dev_dsd_pairs): a CTA whose row dropped a
    block multiplies an all-zero (out-of-bounds) A box, so every output equals
    the 1-CTA dsd bit for bit — forward (row pairs) and dW (mask-column pairs)."""
    lib = sd.load_library()
    lib.sd_dev_dsd_pairs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                     ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_void_p]
    M, N, K = 2048, 1024, 1536
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    plan = sd.LayerPlan(x, w, dy, p)
    plan.forward(77)
    plan.backward_dw()
    torch.cuda.synchronize()
    R, C = M // 128, K // 128
    words = np.array(plan.mask.words(), dtype=np.uint64)
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[: R * C].astype(bool).reshape(R, C)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    fc, fi = _pair_lists(bits)
    y2 = torch.empty_like(plan.y)
    assert lib.sd_dev_dsd_pairs(x.data_ptr(), w.data_ptr(), y2.data_ptr(), 1, M, N, K, 0, 128, fc.data_ptr(),
                                fi.data_ptr(), C, plan.scale, st) == 0
    dc, di = _pair_lists(bits.T.copy())
    dw2 = torch.empty_like(plan.dw)
    assert lib.sd_dev_dsd_pairs(x.data_ptr(), dy.data_ptr(), dw2.data_ptr(), 0, K, N, M, 1, 128, dc.data_ptr(),
                                di.data_ptr(), R, plan.scale, st) == 0
    torch.cuda.synchronize()
    assert torch.equal(y2, plan.y)
    assert torch.equal(dw2, plan.dw)


@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
def test_dw_parts_equal_full_dw_bitwise(sd, oracle, nparts):
    """sd_layer_plan_backward_dw_part: dW row slabs (mask-column blocks) for the
    data-parallel all-reduce overlap reproduce backward_dw bit for bit."""
    M, N, K, p = 2048, 1024, 1024, 0.5
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    plan = sd.LayerPlan(x, w, dy, p)
    plan.forward(31)
    plan.backward_dw()
    torch.cuda.synchronize()
    full = plan.dw.clone()
    plan.dw.fill_(float("nan"))
    slabs = [plan.backward_dw_part(i, nparts) for i in range(nparts)]
    torch.cuda.synchronize()
    assert sum(s.shape[0] for s in slabs) == K
    assert torch.equal(plan.dw, full)
    with pytest.raises(IndexError):
        plan.backward_dw_part(nparts, nparts)


@pytest.mark.parametrize("M,N,K", [(1024, 1024, 1024), (2048, 768, 3072), (512, 1536, 640)])
def test_p0_plan_equals_sparse_kernels(sd, oracle, M, N, K):
    """A p = 0 layer plan runs the dense kernels (nothing to skip); its outputs
    equal the masked kernels' bit for bit (generic C-ABI dsd / sdd entries)."""
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    plan = sd.LayerPlan(x, w, dy, 0.0)
    plan.forward(5)
    plan.backward()
    torch.cuda.synchronize()
    m = plan.mask
    assert m.keep_count() == m.total_blocks()
    lib = sd.load_library()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    y = torch.empty_like(plan.y)
    dx = torch.empty_like(plan.dx)
    dw = torch.empty_like(plan.dw)
    sd.api.check(lib.sd_linear_forward(x.data_ptr(), m.cptr(), w.data_ptr(), 1.0, y.data_ptr(), 1, M, N, K, st))
    sd.api.check(lib.sd_linear_backward_dx(dy.data_ptr(), w.data_ptr(), m.cptr(), 1.0, dx.data_ptr(), 1, M, N, K, st))
    sd.api.check(lib.sd_linear_backward_dw(x.data_ptr(), m.cptr(), dy.data_ptr(), 1.0, dw.data_ptr(), 0, M, N, K, st))
    torch.cuda.synchronize()
    assert torch.equal(plan.y, y)
    assert torch.equal(plan.dx, dx)
    if not torch.equal(plan.dw, dw):  # split-K (small dW outputs) reduces in arrival order
        assert torch.allclose(plan.dw, dw, rtol=1e-5, atol=1e-5 * float(dw.abs().max()))


def test_gelu_table_equals_direct_all_bf16(sd):
    """sd_gelu_forward on large activations reads a 64 K-entry table built with
    the direct kernel's math: every bf16 bit pattern (NaN/Inf included) must map
    to the same output bits as the direct evaluation (used below 512 K elements)."""
    from paper_2411_01238_b200.mlp import gelu

    pats = torch.arange(65536, dtype=torch.int32, device="cuda").to(torch.int16).view(torch.bfloat16)
    big = pats.repeat(16)                         # 1 M elements: table path
    small = pats[: 65536 // 2].clone(), pats[65536 // 2:].clone()  # 32 K each: direct path
    out_big = gelu(big)
    out_small = torch.cat([gelu(small[0]), gelu(small[1])])
    torch.cuda.synchronize()
    ref = out_small.view(torch.int16)
    assert torch.equal(out_big.view(torch.int16)[:65536], ref)
    assert torch.equal(out_big.view(torch.int16).view(16, 65536), ref.expand(16, 65536))


def test_gelu_grad_table_equals_direct_all_bf16(sd):
    """sd_gelu_backward on large activations reads d GELU/dh from a 16 K-entry
    table (2^-31 <= |h| < 2^33) and evaluates the rest directly: every bf16
    h pattern (NaN/Inf included), with random upstream gradients, must give the
    same output bits as the direct kernel (used below 512 K elements)."""
    from paper_2411_01238_b200.mlp import gelu_grad

    pats = torch.arange(65536, dtype=torch.int32, device="cuda").to(torch.int16).view(torch.bfloat16)
    h = pats.repeat(16)                            # 1 M elements: table path
    g = torch.randn(h.numel(), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)).to(
        torch.bfloat16)
    out_big = gelu_grad(h, g)
    parts = [gelu_grad(h[i:i + 32768].clone(), g[i:i + 32768].clone()) for i in range(0, h.numel(), 32768)]
    torch.cuda.synchronize()
    assert torch.equal(out_big.view(torch.int16), torch.cat(parts).view(torch.int16))


@pytest.mark.parametrize("p", [0.1, 0.2, 0.3])
@pytest.mark.parametrize("entry", ["fused", "dx_only", "own_bits_fallback"])
def test_masked_dense_dx_equals_sdd_bitwise(sd, oracle, p, entry):
    """At low p the plan computes dX as the 2-CTA dense GEMM with dropped output
    blocks written as +0.0 (tuning bit 1024 keeps the sdd kernel): same bits,
    dropped blocks exactly +0.0."""
    lib = sd.load_library()
    M = N = K = 4096
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    outs = []
    # own_bits_fallback: tuning bit 2048 forces the masked 2-CTA dX's path for
    # CTAs with more than kMaxOwnUnits units (keep bits read per output chunk,
    # workspace released at exit) — the path the cfg5 single-GPU shard takes
    first = 2048 if entry == "own_bits_fallback" else 0
    try:
        for bits in (first, 1024):
            lib.sd_set_tuning(bits)
            plan = sd.LayerPlan(x, w, dy, p)
            plan.forward(11)
            if entry in ("fused", "own_bits_fallback"):
                plan.backward()
            else:
                plan.backward_dx()
                plan.backward_dw()
            torch.cuda.synchronize()
            outs.append((plan.dx.clone(), plan.dw.clone(), plan.mask.words()))
    finally:
        lib.sd_set_tuning(0)
    (dx0, dw0, m0), (dx1, dw1, m1) = outs
    assert m0 == m1
    assert torch.equal(dx0.view(torch.int16), dx1.view(torch.int16))
    assert torch.equal(dw0, dw1)
    kept = np.array(m0, dtype=np.uint64)
    bits = np.unpackbits(kept.view(np.uint8), bitorder="little")[: 32 * 32].reshape(32, 32)
    blocks = dx0.view(32, 128, 32, 128).permute(0, 2, 1, 3).reshape(32, 32, -1)
    dropped = torch.from_numpy(bits == 0).cuda()
    assert (blocks[dropped].view(torch.int16) == 0).all()


def test_backward_waits_for_caller_pdl_kernel(sd, oracle):
    """a caller kernel between forward and backward that writes dY and
    triggers its dependents early (PDL, as CUTLASS / cuBLASLt kernels may) must
    be waited for. Without SD_PLAN_DY_READY (the default) every backward runs
    griddepcontrol.wait, so dX / dW see the caller's dY."""
    lib = sd.load_library()
    M = N = K = 2048
    x, w, dy0 = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    dy = torch.empty_like(dy0)
    plan = sd.LayerPlan(x, w, dy, 0.5)  # dy_ready=False (default)
    dy.copy_(dy0 * 2)                   # exact in bf16
    plan.forward(7)
    plan.backward()
    torch.cuda.synchronize()
    ref = (plan.dx.clone(), plan.dw.clone())
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for it in range(5):
        dy.zero_()
        plan.dx.fill_(float("nan"))
        plan.dw.fill_(float("nan"))
        torch.cuda.synchronize()
        plan.forward(7)
        assert lib.sd_dev_pdl_early_writer(ctypes.c_void_p(dy0.data_ptr()), ctypes.c_void_p(dy.data_ptr()),
                                           ctypes.c_int64(dy.numel()), 200000, st) == 0
        plan.backward()
        torch.cuda.synchronize()
        assert torch.equal(plan.dx, ref[0]), it
        assert torch.equal(plan.dw, ref[1]), it


@pytest.mark.parametrize("p", [0.0, 0.1, 0.5, 0.9])
def test_graph_replay_equals_eager(sd, oracle, p):
    """Layer steps captured into a CUDA graph (bench.py's timed region) and
    replayed give the eager steps' outputs bit for bit: captured GEMM launches
    get dedicated scheduler slots, the mask generation falls back to
    griddepcontrol.wait under capture, split-K turnstiles reset themselves."""
    M, N, K = 2048, 1536, 1024
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    plan = sd.LayerPlan(x, w, dy, p, dy_ready=True)
    seeds = [3, 4, 5]
    for sd_ in seeds:
        plan.forward(sd_)
        plan.backward()
    torch.cuda.synchronize()
    ref = [plan.y.clone(), plan.dx.clone(), plan.dw.clone(), plan.mask.words()]
    gr = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=cs):
        for sd_ in seeds:
            plan.forward(sd_)
            plan.backward()
    for _ in range(3):
        for t in (plan.y, plan.dx, plan.dw):
            t.fill_(float("nan"))
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(plan.y, ref[0]) and torch.equal(plan.dx, ref[1]) and torch.equal(plan.dw, ref[2])
        assert plan.mask.words() == ref[3]


@pytest.mark.parametrize("M,N,K", [(1024, 2048, 768), (2048, 1024, 1536)])
@pytest.mark.parametrize("layout", ["nn", "nt", "tn"])
@pytest.mark.parametrize("out_f32", [True, False])
def test_gemm2_wide_equals_narrow_bitwise(sd, oracle, M, N, K, layout, out_f32):
    """2-CTA pair tiles 256 x 512 (two N=256 MMAs per A tile, tuning 8192) vs
    256 x 256 (tuning 4096): same bits for every layout of the dense GEMMs
    (forward nn, dX nt, dW tn) — each element reduced over the same K=16 steps."""
    lib = sd.load_library()
    a_mn, b_mn = {"nn": (0, 1), "nt": (0, 0), "tn": (1, 1)}[layout]
    a = _dev(oracle, K, M, 1) if a_mn else _dev(oracle, M, K, 1)
    b = _dev(oracle, K, N, 2) if b_mn else _dev(oracle, N, K, 2)
    dt, tdt = (0, torch.float32) if out_f32 else (1, torch.bfloat16)
    outs = []
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    try:
        for bits in (4096, 8192, 16):
            lib.sd_set_tuning(bits)
            c = torch.full((M, N), float("nan"), dtype=tdt, device="cuda")
            sd.api.check(lib.sd_gemm_ex(a.data_ptr(), a_mn, b.data_ptr(), b_mn, c.data_ptr(), dt, M, N, K, 1.5, st))
            torch.cuda.synchronize()
            outs.append(c)
    finally:
        lib.sd_set_tuning(0)
    assert torch.equal(outs[0], outs[1])  # 2-CTA narrow == wide
    assert torch.equal(outs[0], outs[2])  # == the 1-CTA kernel
    assert not torch.isnan(outs[0].float()).any()


@pytest.mark.parametrize("p", [0.1, 0.3])
def test_masked_dense_dx_wide_pairs_bitwise(sd, oracle, p):
    """The masked 2-CTA dX on 256 x 512 pair tiles (four 128-column keep bits per
    unit) equals the sdd kernel bit for bit; also with per-chunk bit reads."""
    lib = sd.load_library()
    M, N, K = 2048, 1024, 2048
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    outs = []
    try:
        for bits in (8192, 8192 | 2048, 1024):
            lib.sd_set_tuning(bits)
            plan = sd.LayerPlan(x, w, dy, p)
            plan.forward(11)
            plan.backward_dx()
            torch.cuda.synchronize()
            outs.append(plan.dx.clone())
    finally:
        lib.sd_set_tuning(0)
    assert torch.equal(outs[0].view(torch.int16), outs[2].view(torch.int16))
    assert torch.equal(outs[1].view(torch.int16), outs[2].view(torch.int16))


PAIR_CASES = [(4096, 4096, 4096, 0.5), (4096, 4096, 4096, 0.3), (2048, 2048, 8192, 0.7), (1024, 1536, 3072, 0.4),
              (2048, 3072, 768, 0.5), (512, 640, 1152, 0.5)]


@pytest.mark.parametrize("M,N,K,p", PAIR_CASES)
@pytest.mark.parametrize("entry", ["fused", "dx_only"])
def test_row_pair_dx_equals_sdd_bitwise(sd, oracle, M, N, K, p, entry):
    """Mid-p dX split by mask-row pairs (kept blocks common to rows 2i and 2i+1,
    in ascending pairs, on the 2-CTA kernel; the remainder + zero fill on the
    1-CTA sdd kernel; tuning bit 16384) equals the plain sdd dX bit for bit,
    dropped blocks exactly +0.0. Column counts C = K/128 of 32, 64, 24 (rows
    straddling mask words), 6 and 9 (odd)."""
    lib = sd.load_library()
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    outs = []
    try:
        for bits in (0, 16384):
            lib.sd_set_tuning(bits)
            plan = sd.LayerPlan(x, w, dy, p)
            plan.forward(13)
            plan.dx.fill_(float("nan"))
            if entry == "fused":
                plan.backward()
            else:
                plan.backward_dx()
            torch.cuda.synchronize()
            outs.append((plan.dx.clone(), plan.dw.clone() if entry == "fused" else None, plan.mask.words()))
    finally:
        lib.sd_set_tuning(0)
    (dx0, dw0, m0), (dx1, dw1, m1) = outs
    assert m0 == m1
    assert torch.equal(dx0.view(torch.int16), dx1.view(torch.int16))
    if dw0 is not None:
        assert torch.equal(dw0, dw1)
    R, C = M // 128, K // 128
    bits = np.unpackbits(np.array(m0, dtype=np.uint64).view(np.uint8), bitorder="little")[: R * C].reshape(R, C)
    blocks = dx0.view(R, 128, C, 128).permute(0, 2, 1, 3).reshape(R, C, -1)
    assert (blocks[torch.from_numpy(bits == 0).cuda()].view(torch.int16) == 0).all()


@pytest.mark.parametrize("p", [0.0, 0.1, 0.5, 0.9])
def test_plan_graph_step_equals_eager(sd, oracle, p):
    """sd_layer_plan_graph_step: the step captured once into a CUDA graph, the
    mask seed patched per launch — every replay equals the eager step with the
    same seed (new seeds give new, oracle-exact masks), and eager steps after
    graph replays are unaffected."""
    M, N, K = 2048, 1024, 1536
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    ref_plan = sd.LayerPlan(x, w, dy, p, dy_ready=True)
    plan = sd.LayerPlan(x, w, dy, p, dy_ready=True)
    for seed in (5, 6, 7, 1 << 40):
        ref_plan.forward(seed)
        ref_plan.backward()
        plan.graph_step(seed)
        torch.cuda.synchronize()
        for a, b in ((plan.y, ref_plan.y), (plan.dx, ref_plan.dx), (plan.dw, ref_plan.dw)):
            assert torch.equal(a, b), seed
        words, _ = oracle.sample_mask(p, 128, 128, seed, M, K)
        assert np.array_equal(np.array(plan.mask.words(), dtype=np.uint64), words)
    # forward-only graph, then an eager backward on the user stream
    plan.graph_step(11, backward=False)
    plan.backward()
    ref_plan.forward(11)
    ref_plan.backward()
    # and plain eager steps after replays
    plan.forward(12)
    plan.backward()
    ref_plan.forward(12)
    ref_plan.backward()
    torch.cuda.synchronize()
    for a, b in ((plan.y, ref_plan.y), (plan.dx, ref_plan.dx), (plan.dw, ref_plan.dw)):
        assert torch.equal(a, b)


# Launch sizes around one wave of 128 x 256 units (148 SMs): tail halving is on
# only from one full wave up (sd_gemm.cu launch_gemms). Fused backward unit
# counts here (dX 4 per block row + dW 32): 144, 148 and 152.
WAVE_CASES = [(3584, 1024, 1024), (3712, 1024, 1024), (3840, 1024, 1024)]


@pytest.mark.parametrize("M,N,K", WAVE_CASES)
@pytest.mark.parametrize("p", [0.3, 0.5, 0.9])
def test_one_wave_boundary_tail_halving_bitwise(sd, oracle, M, N, K, p):
    """Around the one-wave threshold the default (halving on from one wave),
    halving forced off (tuning 1) and narrow units give identical bits, and
    the default matches the oracle on sampled row blocks."""
    x, w, dy = _dev(oracle, M, K, 31), _dev(oracle, K, N, 32), _dev(oracle, M, N, 33)
    lib = sd.load_library()
    outs = {}
    try:
        for t in (0, 1, 64):
            lib.sd_set_tuning(t)
            outs[t] = _layer_outputs(sd, x, w, dy, p, 77)
    finally:
        lib.sd_set_tuning(0)
    for t in (1, 64):
        for a, b in zip(outs[0], outs[t]):
            assert torch.equal(a, b), t
    y, dx, dw = outs[0]
    words, _ = oracle.sample_mask(p, 128, 128, 77, M, K)
    s = sd.dropout_scale(p)
    xn, wn, dyn = (t.double().cpu().numpy() for t in (x, w, dy))
    for lo in (0, M - 128):
        hi = lo + 128
        ref_y = oracle.dsd_matmul(xn, words, wn, 128, 128, 128, s, row_lo=lo, row_hi=hi)
        g = y[lo:hi].double().cpu().numpy()
        assert np.linalg.norm(g - ref_y) <= 4e-3 * max(np.linalg.norm(ref_y), 1e-30)
    ref_dw = oracle.layer_dw(xn, dyn, words, 128, 128, s, krow_lo=0, krow_hi=128)
    g = dw[:128].double().cpu().numpy()
    assert np.linalg.norm(g - ref_dw) <= 1e-5 * max(np.linalg.norm(ref_dw), 1e-30)



DXT = 1048576  # sd_set_tuning bit kTuneDxt: a plan's dX on the transposed 2-CTA kernel (sd_dxt.cu)


@pytest.mark.parametrize("M,N,K,p", [(1024, 1024, 1024, 0.5), (2048, 768, 3072, 0.9), (4096, 2048, 4096, 0.5),
                                     (1536, 1024, 2560, 0.3), (2048, 4096, 1024, 0.7)])
def test_transposed_2cta_dx_matches_sdd(sd, oracle, M, N, K, p):
    """dX^T = W dY^T on 2-CTA pairs (two kept blocks of one mask row per MMA):
    bit-identical to the 1-CTA sdd dX (the same 16-deep MMA chains over n in the
    same order), dropped blocks exact +0.0, and dW unchanged."""
    x, w, dy = _dev(oracle, M, K, 41), _dev(oracle, K, N, 42), _dev(oracle, M, N, 43)
    lib = sd.load_library()
    ref = _layer_outputs(sd, x, w, dy, p, 91)
    try:
        lib.sd_set_tuning(DXT)
        got = _layer_outputs(sd, x, w, dy, p, 91)
    finally:
        lib.sd_set_tuning(0)
    words, _ = oracle.sample_mask(p, 128, 128, 91, M, K)
    s = sd.dropout_scale(p)
    dyn, wn = dy.double().cpu().numpy(), w.double().cpu().numpy()
    for lo in (0, M - 128):
        ref_dx = oracle.layer_dx(dyn, wn, words, 128, 128, s, row_lo=lo, row_hi=lo + 128)
        g = got[1][lo:lo + 128].double().cpu().numpy()
        assert np.linalg.norm(g - ref_dx) <= 4e-3 * max(np.linalg.norm(ref_dx), 1e-30)
        assert (got[1][lo:lo + 128].view(torch.int16).cpu().numpy()[ref_dx == 0] == 0).all()
    assert torch.equal(got[2], ref[2]) and torch.equal(got[0], ref[0])
    assert torch.equal(got[1], ref[1])


NO_SMALL_HASH = 2097152  # sd_set_tuning bit kTuneNoSmallHash


@pytest.mark.parametrize("M,N,K,p", [(1024, 1024, 1024, 0.5), (1024, 1024, 1024, 0.1), (1024, 1024, 1024, 0.9),
                                     (512, 768, 1536, 0.3), (768, 256, 8192, 0.5), (1024, 512, 1024, 0.95)])
def test_small_plan_hash_mode_equals_list_mode(sd, oracle, M, N, K, p):
    """Small plans (the whole step fits on the SMs at once) run their GEMMs in
    hash mode — kept lists from the counter hash, the forward ahead of the mask
    generation — and must give the bits of the list-reading path
    (kTuneNoSmallHash), repeatedly, with the plan's mask equal to the oracle's."""
    x, w, dy = _dev(oracle, M, K, 51), _dev(oracle, K, N, 52), _dev(oracle, M, N, 53)
    lib = sd.load_library()
    plan = sd.LayerPlan(x, w, dy, p, dy_ready=True)
    outs = []
    for tune in (0, NO_SMALL_HASH, 0):
        lib.sd_set_tuning(tune)
        try:
            res = []
            for step in range(3):
                plan.forward(100 + step)
                plan.backward()
                torch.cuda.synchronize()
                res.append([plan.y.clone(), plan.dx.clone(), plan.dw.clone(),
                            np.array(plan.mask.words(), dtype=np.uint64)])
            outs.append(res)
        finally:
            lib.sd_set_tuning(0)
    for step in range(3):
        words, keep = oracle.sample_mask(p, 128, 128, 100 + step, M, K)
        for run in outs:
            assert np.array_equal(run[step][3], words)
            for a, b in zip(run[step][:3], outs[0][step][:3]):
                assert torch.equal(a, b)
