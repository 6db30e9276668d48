"""Host-bound or device-bound? Back-to-back layer steps with and without a
stream gate (dev tool, 1 GPU).

    python tools/gated_probe.py [SIZE,P ...]

ungated: K steps enqueued back to back between two events (bench.py's regime);
         when the host enqueues slower than the GPU runs, this measures the host.
gated:   a torch.cuda._sleep spin kernel is enqueued first, so all K steps are in
         the queue before the first one runs: device time only.
host:    wall time per step of the enqueue calls alone.
Prints one JSON line per configuration (sparse step and dense step)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2411_01238_b200 as sd  # noqa: E402

K = 40


def rnd(r, c):
    return torch.randn(r, c, device="cuda").to(torch.bfloat16)


def measure(fn, gated):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if gated:
        torch.cuda._sleep(int(4e6))  # ~2 ms spin: covers the host enqueue of K steps
    a.record()
    t0 = time.perf_counter()
    for i in range(K):
        fn(i)
    host = (time.perf_counter() - t0) / K * 1e6
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3, host


def main():
    cfgs = sys.argv[1:] or ["1024,0.5", "1024,0.1", "1024,0.9", "2048,0.5", "4096,0.5", "4096,0.9"]
    for c in cfgs:
        S, p = c.split(",")
        S, p = int(S), float(p)
        plans = [sd.LayerPlan(rnd(S, S), rnd(S, S), rnd(S, S), p, dy_ready=True) for _ in range(3)]

        def step(i):
            pl = plans[i % 3]
            pl.forward(seed=i)
            pl.backward()

        def dense(i):
            pl = plans[i % 3]
            pl.dense_forward()
            pl.dense_backward()

        def gstep(i):
            plans[i % 3].graph_step(seed=i)

        ins = [(pl._x, pl._w, pl._dy) for pl in plans] if hasattr(plans[0], "_x") else None
        tens = [(rnd(S, S), rnd(S, S), rnd(S, S)) for _ in range(3)]

        def cublas(i):
            x, w, dy = tens[i % 3]
            x @ w
            x.t() @ dy
            dy @ w.t()

        out = {"S": S, "p": p}
        t_end = time.time() + 1.0
        while time.time() < t_end:
            for i in range(10):
                step(i)
                dense(i)
        for name, fn in (("sparse", step), ("dense", dense), ("graph", gstep), ("cublas", cublas)):
            for gated in (False, True):
                vals = sorted(measure(fn, gated) for _ in range(5))
                dev, host = vals[len(vals) // 2]
                out[f"{name}_{'gated' if gated else 'ungated'}_us"] = round(dev, 2)
                out[f"{name}_host_us"] = round(host, 2)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
