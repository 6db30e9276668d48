"""Isolated (one step at a time, synchronized) layer-step latency: eager
launches vs one CUDA-graph launch of the same step (dev probe, round 2)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2411_01238_b200 as sd  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(3)
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
for S in (1024, 2048):
    x, w, dy = ((torch.rand(S, S, generator=g, device="cuda") - 0.5).to(torch.bfloat16) for _ in range(3))
    for p in (0.1, 0.5, 0.9):
        plan = sd.LayerPlan(x, w, dy, p, dy_ready=True)
        out = {"S": S, "p": p}
        for name, fn in (("sparse", lambda: (plan.forward(seed=1), plan.backward())),
                         ("sparse_graph_step_api", lambda: plan.graph_step(1)),
                         ("dense", lambda: (plan.dense_forward(), plan.dense_backward()))):
            for i in range(50):
                fn()
            torch.cuda.synchronize()
            modes = [("eager", fn)]
            if name != "sparse_graph_step_api":  # that one is itself a graph launch
                gr = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream()
                cs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.graph(gr, stream=cs):
                    fn()
                torch.cuda.synchronize()
                modes.append(("graph", gr.replay))
            for mode, run in modes:
                ts = []
                for i in range(40):
                    flush.fill_(1.0)
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    run()
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b) * 1e3)
                out[f"{name}_{mode}_us"] = sorted(ts)[len(ts) // 2]
        print(json.dumps(out), flush=True)
        del plan
