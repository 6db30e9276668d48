"""e2e ms/step of HostLayerPipeline vs buffer sets and timed-step count (dev tool).
   python tools/e2e_slots.py [SIZE] [P]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_01238_b200.pipeline import HostLayerPipeline  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
P = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
xh, wh, dyh = (torch.randn(S, S).to(torch.bfloat16).pin_memory() for _ in range(3))
for nslots in (2, 3):
    pipe = HostLayerPipeline(xh, wh, dyh, P, nslots=nslots)
    for n in (10, 20, 40):
        res = []
        for r in range(3):
            for i in range(3):
                pipe.step(i)
            pipe.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(pipe.s_h2d)
            pipe.s_cmp.wait_stream(pipe.s_h2d)
            for i in range(n):
                pipe.step(3 + i)
            pipe.s_d2h.wait_stream(pipe.s_cmp)
            pipe.s_d2h.wait_stream(pipe.s_h2d)
            e1.record(pipe.s_d2h)
            pipe.synchronize()
            res.append(e0.elapsed_time(e1) / n)
        print(f"S={S} p={P} nslots={nslots} steps={n}: {sorted(res)[1]:.3f} ms/step (all {[round(v, 3) for v in res]})",
              flush=True)
    del pipe
    torch.cuda.empty_cache()
