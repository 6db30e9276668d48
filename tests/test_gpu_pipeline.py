"""HostLayerPipeline (bench.py's e2e path): host buffers in, host outputs out,
steps rotating over buffer sets on three streams. Every step's host outputs
must equal a device-resident LayerPlan's outputs for the same step seed."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sd():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2411_01238_b200 as sd

    sd.load_library()
    return sd


@pytest.mark.parametrize("nslots", [2, 3])
def test_pipeline_steps_equal_device_plan(sd, nslots):
    from paper_2411_01238_b200.pipeline import HostLayerPipeline

    M, N, K, p = 1024, 768, 512, 0.5
    g = torch.Generator().manual_seed(5)
    xh, wh, dyh = (torch.randn(r, c, generator=g).to(torch.bfloat16).pin_memory()
                   for r, c in ((M, K), (K, N), (M, N)))
    pipe = HostLayerPipeline(xh, wh, dyh, p, nslots=nslots)
    outs = []
    for i in range(7):
        o = pipe.step(i)
        pipe.synchronize()  # the slot's host outputs are rewritten nslots steps later
        outs.append(tuple(t.clone() for t in o))
    plan = sd.LayerPlan(xh.cuda(), wh.cuda(), dyh.cuda(), p)
    for i, (y, dx, dw) in enumerate(outs):
        plan.forward(sd.effective_seed(0, i, 0))
        plan.backward()
        torch.cuda.synchronize()
        assert torch.equal(y, plan.y.cpu()) and torch.equal(dx, plan.dx.cpu()) and torch.equal(dw, plan.dw.cpu()), i


def test_pipeline_rejects_device_inputs(sd):
    from paper_2411_01238_b200.pipeline import HostLayerPipeline

    x = torch.zeros(256, 256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="host tensor"):
        HostLayerPipeline(x, x, x, 0.5)
