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
