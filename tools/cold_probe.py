"""Why is an isolated 1024^3 step (~45 us) so much slower than a step inside a
back-to-back stream (~18 us)? One step between CUDA events under several
preconditions (dev tool): all queued behind a spin kernel (device time only)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2411_01238_b200 as sd  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
P = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
x, w, dy = (torch.randn(S, S, device="cuda").to(torch.bfloat16) for _ in range(3))
plan = sd.LayerPlan(x, w, dy, P, dy_ready=True)
tiny = sd.LayerPlan(*(torch.randn(256, 256, device="cuda").to(torch.bfloat16) for _ in range(3)), P, dy_ready=True)
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
small = torch.empty(1024, device="cuda")


def run(pre, n_steps=1, reps=15):
    ts = []
    for r in range(reps):
        torch.cuda.synchronize()
        pre()
        torch.cuda._sleep(200000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(n_steps):
            plan.forward(r * 10 + i)
            plan.backward()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / n_steps)
    ts.sort()
    return ts[len(ts) // 2]


for _ in range(20):
    plan.forward(0), plan.backward()
cases = {
    "gate only": lambda: None,
    "flush+gate": lambda: flush.fill_(1.0),
    "small fill+gate": lambda: small.fill_(1.0),
    "flush, tiny plan step, gate": lambda: (flush.fill_(1.0), tiny.forward(1), tiny.backward()),
    "gate only, 2 steps": None,
    "gate only, 10 steps": None,
}
for name, pre in cases.items():
    if name.endswith("2 steps"):
        v = run(lambda: None, 2)
    elif name.endswith("10 steps"):
        v = run(lambda: None, 10)
    else:
        v = run(pre)
    print(f"S={S} p={P} {name:32s}: {v:7.1f} us/step", flush=True)
