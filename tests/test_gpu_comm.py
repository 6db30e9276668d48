"""GPU: the data-parallel backward behind the C-ABI (sd_comm_*,
sd_layer_plan_backward_allreduce) on a 1-rank NCCL communicator — the only
NCCL world a one-GPU box can form (NCCL refuses two ranks on one device; the
2-rank logic is covered over gloo in test_sharding_gloo.py / test_dp_bench.py).

With one rank the all-reduce is the identity, so the sharded step must give
exactly the outputs of the plain backward: dW slabs bit-identical to the full
dW (same tiles and reduction order), dX unchanged, for every slab count."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sd():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2411_01238_b200 as sd

    sd.load_library()
    return sd


@pytest.fixture(scope="module")
def comm(sd):
    c = sd.Communicator(1, 0, sd.Communicator.new_unique_id())
    yield c
    torch.cuda.synchronize()
    c.close()


def _rand(gen, r, c):
    u = torch.rand(r, c, generator=gen, device="cuda")
    return ((0.25 + u) * torch.where(torch.rand(r, c, generator=gen, device="cuda") < 0.5, -1.0, 1.0)).to(
        torch.bfloat16)


@pytest.mark.parametrize("p,nparts", [(0.5, 1), (0.5, 2), (0.5, 4), (0.1, 2), (0.0, 3)])
def test_backward_allreduce_one_rank_equals_backward(sd, comm, p, nparts):
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    M, N, K = 4096, 2048, 1024
    x, w, dy = _rand(gen, M, K), _rand(gen, K, N), _rand(gen, M, N)
    plan = sd.LayerPlan(x, w, dy, p, row_block_offset=96)
    plan.forward(seed=5)
    plan.backward()
    torch.cuda.synchronize()
    ref_dx, ref_dw = plan.dx.clone(), plan.dw.clone()
    side = torch.cuda.Stream()
    for use_side in (True, False):
        plan.dx.fill_(float("nan"))
        plan.dw.fill_(float("nan"))
        plan.forward(seed=5)
        plan.backward_allreduce(comm, nparts, comm_stream=side if use_side else None)
        torch.cuda.synchronize()
        assert torch.equal(plan.dx, ref_dx)
        assert torch.equal(plan.dw, ref_dw)


def test_comm_allreduce_sum_identity(sd, comm):
    t = torch.randn(1 << 20, device="cuda")
    ref = t.clone()
    comm.allreduce_sum(t)
    torch.cuda.synchronize()
    assert torch.equal(t, ref)
    assert sd.Communicator.nccl_version() >= 22700


def test_backward_allreduce_validation(sd, comm):
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    x, w, dy = _rand(gen, 256, 256), _rand(gen, 256, 256), _rand(gen, 256, 256)
    plan = sd.LayerPlan(x, w, dy, 0.5)
    plan.forward(seed=1)
    with pytest.raises(IndexError):
        plan.backward_allreduce(comm, 3)  # 2 mask columns
    with pytest.raises(IndexError):
        plan.backward_allreduce(comm, 0)
