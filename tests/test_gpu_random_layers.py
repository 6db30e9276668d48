"""GPU: randomized layer geometries against the oracle (seeded, bounded sizes).

Each case draws M, N, K (multiples of 128), p in [0, 0.95) and mask blocks of
128 or 256 rows/columns, runs one layer step through LayerPlan (forward:
sample_mask + dsd; backward: dW + dX) and checks every output against the
oracle on the same bf16 inputs: masks bit-exact, Y / dX within the bf16 bar,
dW within the fp32 bar, dropped dX blocks exactly +0.0. Then the same step
under every unit shape (narrow / wide units, fused / split backward) must give
the same bits — split-K included — and a second run must repeat them."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

rng = np.random.default_rng(20261017)
CASES = []
for _ in range(16):
    mb = int(rng.choice([128, 128, 256]))
    kb = int(rng.choice([128, 128, 256]))
    M = mb * int(rng.integers(1, 9)) * (2 if mb == 128 else 1)
    K = kb * int(rng.integers(1, 9))
    N = 128 * int(rng.integers(1, 13))
    p = float(rng.choice([0.0, 0.05, 0.1, 0.2, 0.35, 0.5, 0.65, 0.8, 0.95]))
    CASES.append((M, N, K, mb, kb, p, int(rng.integers(0, 2**31))))


@pytest.fixture(scope="module")
def sd():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2411_01238_b200 as sd

    sd.load_library()
    return sd


def _dev(o, r, c, seed):
    return torch.from_numpy(o.random_matrix(r, c, seed)).to(torch.bfloat16).cuda()


def _step(sd, x, w, dy, p, mb, kb, seed):
    plan = sd.LayerPlan(x, w, dy, p, m_blk=mb, k_blk=kb)
    plan.forward(seed)
    plan.backward()
    torch.cuda.synchronize()
    return plan, [plan.y.clone(), plan.dx.clone(), plan.dw.clone()]


@pytest.mark.parametrize("M,N,K,mb,kb,p,seed", CASES)
def test_random_layer_against_oracle(sd, oracle, M, N, K, mb, kb, p, seed):
    x, w, dy = _dev(oracle, M, K, seed % 1000 + 1), _dev(oracle, K, N, seed % 1000 + 2), _dev(oracle, M, N, seed % 1000 + 3)
    plan, outs = _step(sd, x, w, dy, p, mb, kb, seed)
    words = np.array(plan.mask.words(), dtype=np.uint64)
    wo, keep = oracle.sample_mask(p, mb, kb, seed, M, K)
    assert np.array_equal(words, wo) and plan.mask.keep_count() == keep
    s = sd.dropout_scale(p)
    xn, wn, dyn = (t.double().cpu().numpy() for t in (x, w, dy))
    ref_y = oracle.dsd_matmul(xn, wo, wn, mb, 128, kb, s)
    ref_dx = oracle.layer_dx(dyn, wn, wo, mb, kb, s)
    ref_dw = oracle.layer_dw(xn, dyn, wo, mb, kb, s)
    R, C = M // mb, K // kb
    bits = np.unpackbits(wo.view(np.uint8), bitorder="little")[:R * C].reshape(R, C).astype(bool)
    xm = xn * np.kron(bits, np.ones((mb, kb)))
    for got, ref, bound, f32 in (
            (outs[0], ref_y, s * (np.abs(xm) @ np.abs(wn)), False),
            (outs[1], ref_dx, s * (np.abs(dyn) @ np.abs(wn).T), False),
            (outs[2], ref_dw, s * (np.abs(xm).T @ np.abs(dyn)), True)):
        g = got.double().cpu().numpy()
        d = np.abs(g - ref)
        relf = np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)
        if f32:
            assert relf < 1e-5 and (d <= 1e-5 * bound + 1e-30).all(), relf
        else:
            assert relf < 4e-3 and (d <= 2.0**-7 * np.abs(ref) + 1e-3 * bound).all(), relf
    dx_raw = outs[1].view(torch.int16).cpu().numpy()
    assert (dx_raw[ref_dx == 0] == 0).all()
    # every unit shape (narrow / wide units, fused / split backward) gives the
    # same bits, and a repeat gives the same bits. (p = 0 plans run the dense
    # kernels, which tuning 64 would swap for the masked ones: skipped there.)
    lib = sd.load_library()
    try:
        for tune in ((1 | 64, 1 | 32, 8) if p > 0 else (8,)):
            lib.sd_set_tuning(tune)
            _, o2 = _step(sd, x, w, dy, p, mb, kb, seed)
            for a, b in zip(outs, o2):
                assert torch.equal(a, b), tune
    finally:
        lib.sd_set_tuning(0)
    _, o3 = _step(sd, x, w, dy, p, mb, kb, seed)
    for a, b in zip(outs, o3):
        assert torch.equal(a, b)


# Larger random geometries: multi-wave launches, tail halving, split-K dW, dsd
# lists longer than the 64-entry staging, the two-launch backward. Checked on
# sampled row slabs of Y / dX and K-row slabs of dW (full M reduction) against
# the oracle, plus bitwise across unit modes and repeats.
rng_l = np.random.default_rng(20261018)
LARGE = []
for _ in range(8):
    mb = int(rng_l.choice([128, 128, 256]))
    kb = int(rng_l.choice([128, 128, 256]))
    M = 256 * int(rng_l.integers(8, 65))      # 2048 .. 16384 rows
    K = kb * int(rng_l.integers(4, 8192 // kb + 1))
    N = 256 * int(rng_l.integers(1, 17))      # 256 .. 4096
    p = float(rng_l.choice([0.1, 0.3, 0.5, 0.7, 0.9]))
    LARGE.append((M, N, K, mb, kb, p, int(rng_l.integers(0, 2**31))))


def _slab_check(got, ref, bound, f32):
    g = got.double().cpu().numpy()
    d = np.abs(g - ref)
    relf = np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)
    if f32:
        assert relf < 1e-5 and (d <= 1e-5 * bound + 1e-30).all(), relf
    else:
        assert relf < 4e-3 and (d <= 2.0**-7 * np.abs(ref) + 1e-3 * bound).all(), relf


@pytest.mark.parametrize("M,N,K,mb,kb,p,seed", LARGE)
def test_large_random_layer_slabs(sd, oracle, M, N, K, mb, kb, p, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)

    def rnd(r, c):
        u = torch.rand(r, c, generator=gen, device="cuda")
        return ((0.25 + u) * torch.where(torch.rand(r, c, generator=gen, device="cuda") < 0.5, -1.0, 1.0)).to(
            torch.bfloat16)

    x, w, dy = rnd(M, K), rnd(K, N), rnd(M, N)
    plan, outs = _step(sd, x, w, dy, p, mb, kb, seed)
    wo, keep = oracle.sample_mask(p, mb, kb, seed, M, K)
    assert np.array_equal(np.array(plan.mask.words(), dtype=np.uint64), wo) and plan.mask.keep_count() == keep
    s = sd.dropout_scale(p)
    xn, wn, dyn = (t.double().cpu().numpy() for t in (x, w, dy))
    R, C = M // mb, K // kb
    bits = np.unpackbits(wo.view(np.uint8), bitorder="little")[:R * C].reshape(R, C).astype(bool)
    for lo in sorted({0, (M // 2) // mb * mb, M - mb}):
        hi = lo + mb
        xm = xn[lo:hi] * np.kron(bits[lo // mb:lo // mb + 1], np.ones((mb, kb)))
        _slab_check(outs[0][lo:hi], oracle.dsd_matmul(xn, wo, wn, mb, 128, kb, s, row_lo=lo, row_hi=hi),
                    s * (np.abs(xm) @ np.abs(wn)), False)
        ref_dx = oracle.layer_dx(dyn, wn, wo, mb, kb, s, row_lo=lo, row_hi=hi)
        _slab_check(outs[1][lo:hi], ref_dx, s * (np.abs(dyn[lo:hi]) @ np.abs(wn).T), False)
        assert (outs[1][lo:hi].view(torch.int16).cpu().numpy()[ref_dx == 0] == 0).all()
    xm = xn * np.kron(bits, np.ones((mb, kb)))
    for klo in sorted({0, K - kb}):
        khi = klo + kb
        _slab_check(outs[2][klo:khi], oracle.layer_dw(xn, dyn, wo, mb, kb, s, krow_lo=klo, krow_hi=khi),
                    s * (np.abs(xm[:, klo:khi]).T @ np.abs(dyn)), True)
    lib = sd.load_library()
    try:
        for tune in (1 | 64, 1 | 32, 8, 65536):
            lib.sd_set_tuning(tune)
            _, o2 = _step(sd, x, w, dy, p, mb, kb, seed)
            for a, b in zip(outs, o2):
                assert torch.equal(a, b), tune
    finally:
        lib.sd_set_tuning(0)
    _, o3 = _step(sd, x, w, dy, p, mb, kb, seed)
    for a, b in zip(outs, o3):
        assert torch.equal(a, b)
