"""dX alone, back to back (spin-gated device time): the 1-CTA sdd kernel vs the
transposed 2-CTA kernel (sd_dxt.cu, tuning kTuneDxt) vs the dense dX (dev tool).
   python tools/dx_kernels.py SIZE|M,N,K P [P ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
S = sys.argv[1]
M, N, K = (int(v) for v in S.split(",")) if "," in S else (int(S),) * 3
for P in [float(v) for v in sys.argv[2:]] or [0.5]:
    sets = [(torch.randn(M, K, device="cuda").to(torch.bfloat16), torch.randn(K, N, device="cuda").to(torch.bfloat16),
             torch.randn(M, N, device="cuda").to(torch.bfloat16)) for _ in range(3)]
    plans = [sd.LayerPlan(x, w, dy, P, dy_ready=True) for x, w, dy in sets]
    for i, pl in enumerate(plans):
        pl.forward(i)
    torch.cuda.synchronize()
    res = {}
    for name, tune in (("sdd", 0), ("dxt", 1048576), ("sdd", 0), ("dxt", 1048576)):
        lib.sd_set_tuning(tune)
        for j in range(30):
            plans[j % 3].backward_dx()
        torch.cuda.synchronize()
        torch.cuda._sleep(400000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        n = 30
        for j in range(n):
            plans[j % 3].backward_dx()
        b.record()
        torch.cuda.synchronize()
        res.setdefault(name, []).append(a.elapsed_time(b) / n * 1e3)
    lib.sd_set_tuning(0)
    keep = plans[0].mask.keep_count() / plans[0].mask.total_blocks()
    fl = keep * 2 * M * N * K
    print(f"S={S} p={P} keep={keep:.3f}: " + "  ".join(f"{k} {min(v):8.1f} us ({fl / min(v) / 1e6:6.0f} TFLOP/s)" for k, v in res.items()),
          flush=True)
