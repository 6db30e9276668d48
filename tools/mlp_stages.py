"""Per-stage timing of the ViT-B MLP step (configs[2]) — sparse vs dense (dev tool).
python tools/mlp_stages.py [P ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_01238_b200.api import effective_seed  # noqa: E402
from paper_2411_01238_b200.mlp import SparseDropMLP, gelu, gelu_grad  # noqa: E402

T, D, H = 65536, 768, 3072
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randn(T, D, device="cuda", generator=g).to(torch.bfloat16)
w1 = (torch.randn(D, H, device="cuda", generator=g) * 0.03).to(torch.bfloat16)
w2 = (torch.randn(H, D, device="cuda", generator=g) * 0.03).to(torch.bfloat16)
dy = torch.randn(T, D, device="cuda", generator=g).to(torch.bfloat16)


def stages(m, dense, seed):
    f1, f2 = m.fc1, m.fc2
    return [
        ("fc1 fwd", lambda: f1.dense_forward() if dense else f1.forward(effective_seed(0, seed, 0))),
        ("gelu", lambda: gelu(f1.y, out=m.act)),
        ("fc2 fwd", lambda: f2.dense_forward() if dense else f2.forward(effective_seed(0, seed, 1))),
        ("fc2 bwd", lambda: f2.dense_backward() if dense else f2.backward()),
        ("gelu'", lambda: gelu_grad(f1.y, f2.dx, out=m.dact)),
        ("fc1 bwd", lambda: f1.dense_backward() if dense else f1.backward()),
    ]


for P in [float(v) for v in sys.argv[1:]] or [0.1, 0.5]:
    out = {}
    for name, dense in (("sparse", False), ("dense", True)):
        m = SparseDropMLP(x, w1, w2, dy, P, dense=dense)
        for _ in range(3):
            m.step(1)
        st = stages(m, dense, 5)
        ts = {k: [] for k, _ in st}
        for r in range(10):
            for k, fn in st:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts[k].append(e0.elapsed_time(e1) * 1e3)
        out[name] = {k: sorted(v)[len(v) // 2] for k, v in ts.items()}
    print(f"cfg3 p={P} (us):  " + "  ".join(f"{k}: {out['sparse'][k]:.0f}/{out['dense'][k]:.0f}" for k in out['sparse'])
          + f"  | total {sum(out['sparse'].values()):.0f} / {sum(out['dense'].values()):.0f}  (sparse/dense)", flush=True)
