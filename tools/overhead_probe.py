"""Where does a small layer step's time go? (round-2 probe, 1 GPU)

For a few shapes: host issue time per step (Python + ctypes + cudaLaunchKernelEx,
no sync), device time per step back-to-back (CUDA events), and the device time
of the same steps replayed from a CUDA graph (captured once with distinct
seeds), plus the dense step for reference.
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2411_01238_b200 as sd  # noqa: E402


def rnd(g, r, c):
    return ((0.25 + torch.rand(r, c, generator=g, device="cuda")) *
            torch.where(torch.rand(r, c, generator=g, device="cuda") < 0.5, -1.0, 1.0)).to(torch.bfloat16)


def main():
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    res = []
    for (S, p) in [(1024, 0.5), (1024, 0.1), (1024, 0.9), (2048, 0.5), (4096, 0.5), (4096, 0.9)]:
        x, w, dy = rnd(g, S, S), rnd(g, S, S), rnd(g, S, S)
        plan = sd.LayerPlan(x, w, dy, p, dy_ready=True)

        def step(i):
            plan.forward(seed=i)
            plan.backward()

        def dense(i):
            plan.dense_forward()
            plan.dense_backward()

        out = {"S": S, "p": p}
        for name, fn in (("sparse", step), ("dense", dense)):
            for i in range(200):
                fn(i)
            torch.cuda.synchronize()
            n = 200
            t0 = time.perf_counter()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(n):
                fn(i)
            b.record()
            t_host = (time.perf_counter() - t0) / n * 1e3
            torch.cuda.synchronize()
            out[f"{name}_host_ms"] = t_host
            out[f"{name}_dev_ms"] = a.elapsed_time(b) / n
            # graph: capture 20 steps once, replay
            try:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    fn(0)
                    torch.cuda.synchronize()
                    with torch.cuda.graph(gr, stream=s):
                        for i in range(20):
                            fn(1000 + i)
                torch.cuda.synchronize()
                for _ in range(5):
                    gr.replay()
                torch.cuda.synchronize()
                a.record()
                for _ in range(10):
                    gr.replay()
                b.record()
                torch.cuda.synchronize()
                out[f"{name}_graph_dev_ms"] = a.elapsed_time(b) / 200
            except Exception as e:  # noqa: BLE001
                out[f"{name}_graph_error"] = repr(e)[:200]
        res.append(out)
        print(json.dumps(out), flush=True)
        del plan


if __name__ == "__main__":
    main()
