"""GPU: the §8f rows — BMSK save/load/replay of device masks (f3) and the
paper's Dropout+Dense / Block-dropout+Dense baselines (f2) vs the reference."""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def sd():
    import paper_2411_01238_b200 as sd

    sd.load_library()
    return sd


def _dev(o, r, c, seed):
    return torch.from_numpy(o.random_matrix(r, c, seed)).to(torch.bfloat16).cuda()


def test_bmsk_device_roundtrip_matches_reference_bytes(sd, tmp_path):
    from paper_2411_01238_b200 import bmsk

    cases = json.loads((GOLDEN / "bmsk.json").read_text())
    # a mask sampled ON THE DEVICE serialises to exactly the reference's bytes
    m = sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, 0), 1024, 1024)
    assert bmsk.to_bytes(m).hex() == cases[0]["bytes"]
    for c in cases:
        back = bmsk.from_bytes(bytes.fromhex(c["bytes"]))
        assert [hex(w) for w in back.words()] == c["words"]
        assert [back.block_rows(), back.block_cols(), back.m_blk(), back.k_blk()] == c["geom"]
        assert bmsk.to_bytes(back).hex() == c["bytes"]
    path = str(tmp_path / "mask.bmsk")
    m = sd.sample_mask(sd.DropoutSpec(0.25, 128, 128, 321), 128 * 8, 128 * 16)
    sd.save_mask(m, path)
    back = sd.load_mask(path)
    assert back.words() == m.words() and back.keep_count() == m.keep_count()
    with pytest.raises(RuntimeError):
        sd.load_mask(str(tmp_path / "missing.bmsk"))
    bad = bytearray.fromhex(cases[1]["bytes"])
    bad[-1] |= 0x80  # a padding bit past the 4x4 grid
    with pytest.raises(RuntimeError, match="nonzero bits"):
        bmsk.from_bytes(bytes(bad), "pad")


def test_replayed_mask_drives_the_gemm(sd, oracle):
    """A BMSK-loaded mask is re-compacted on the device and used by dsd directly."""
    from paper_2411_01238_b200 import bmsk

    M, N, K = 512, 256, 768
    m = sd.sample_mask(sd.DropoutSpec(0.4, 128, 128, 5), M, K)
    back = bmsk.from_bytes(bmsk.to_bytes(m))
    a, b = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2)
    torch.cuda.synchronize()
    assert torch.equal(sd.dsd_matmul(a, m, b, 1.5), sd.dsd_matmul(a, back, b, 1.5))


def test_dropout_dense_matches_reference(sd, oracle):
    from paper_2411_01238_b200.baselines import BaselineLayer

    g = dict(np.load(GOLDEN / "dropout_dense_256.npz"))
    M, N, K, seed, step, li = [int(v) for v in g["meta"]]
    p = float(g["p"][0])
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    lay = BaselineLayer("dropout_dense", x, w, dy, p, seed=seed, layer_index=li)
    lay.forward(step)
    lay.backward()
    torch.cuda.synchronize()
    # the element mask is the reference's sample_element_mask, bit for bit
    em = oracle.element_mask(oracle.effective_seed(seed, step, li), p, M, K)
    xm_ref = x.float().cpu().numpy() * em
    assert np.array_equal(lay.xm.float().cpu().numpy(), xm_ref)
    for got, want in ((lay.y, g["y"]), (lay.dx, g["dx"]), (lay.dw, g["dw"])):
        got = got.double().cpu().numpy()
        want = want.astype(np.float64)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 4e-3
    assert np.array_equal(lay.dx.float().cpu().numpy() == 0, g["dx"] == 0)


def test_block_dropout_dense_equals_sparsedrop(sd, oracle):
    """Naive block dropout + dense GEMM computes the same values as the fused
    SparseDrop path (the paper's comparison is about time, not results)."""
    from paper_2411_01238_b200.baselines import BaselineLayer

    M, N, K, p = 1024, 512, 768, 0.5
    x, w, dy = _dev(oracle, M, K, 1), _dev(oracle, K, N, 2), _dev(oracle, M, N, 3)
    base = BaselineLayer("block_dropout_dense", x, w, dy, p, seed=0)
    base.forward(4)
    base.backward()
    plan = sd.LayerPlan(x, w, dy, p)
    plan.forward(sd.effective_seed(0, 4, 0))
    plan.backward()
    torch.cuda.synchronize()
    assert base.mask.words() == plan.mask.words()
    assert torch.equal(base.y, plan.y)
    assert torch.equal(base.dx, plan.dx)
    assert (base.dw - plan.dw).abs().max().item() <= 1e-4 * plan.dw.abs().max().item()
    dense = BaselineLayer("dense", x, w, dy, 0.0)
    dense.forward(0)
    dense.backward()
    torch.cuda.synchronize()
    assert torch.equal(dense.y, sd.dense_gemm(x, w))
