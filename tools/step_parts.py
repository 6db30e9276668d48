"""Where a layer step's time goes, in the back-to-back regime (dev tool).

    python tools/step_parts.py SIZE|M,N,K P [rounds]

Three plans over rotating input sets (> L2), K = 20 steps back to back per
window, after a sustained warm-up. Variants of the step:
  full     mask + forward + backward (bench.py's step)
  fwd      mask + forward
  fwd+dx   mask + forward + dX launch only
  fwd+dw   mask + forward + dW launch only
  dense    the dense step (dense_forward + dense_backward)
  dfwd     dense forward only
Prints the median us/step per variant; differences estimate each launch's
share of the step under launch overlap."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

S = sys.argv[1]
M, N, K_ = (int(v) for v in S.split(",")) if "," in S else (int(S),) * 3
P = float(sys.argv[2])
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 8
STEPS = 20
plans = []
for _ in range(3):
    x = torch.randn(M, K_, device="cuda").to(torch.bfloat16)
    w = torch.randn(K_, N, device="cuda").to(torch.bfloat16)
    dy = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    plans.append(sd.LayerPlan(x, w, dy, P, dy_ready=True))


def full(pl, s):
    pl.forward(s)
    pl.backward()


def fwd(pl, s):
    pl.forward(s)


def fwd_dx(pl, s):
    pl.forward(s)
    pl.backward_dx()


def fwd_dw(pl, s):
    pl.forward(s)
    pl.backward_dw()


def dense(pl, s):
    pl.dense_forward()
    pl.dense_backward()


def dfwd(pl, s):
    pl.dense_forward()


variants = {"full": full, "fwd": fwd, "fwd+dx": fwd_dx, "fwd+dw": fwd_dw, "dense": dense, "dfwd": dfwd}


def run(fn, n, s0):
    for i in range(n):
        fn(plans[i % 3], s0 + i)


t_end = time.time() + 1.5
while time.time() < t_end:
    for fn in variants.values():
        run(fn, 6, 0)
torch.cuda.synchronize()
res = {k: [] for k in variants}
for r in range(rounds):
    for name, fn in variants.items():
        run(fn, 3, 1000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(fn, STEPS, 10 * r)
        b.record()
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / STEPS * 1e3)
print(f"S={S} p={P}: " + "  ".join(f"{k} {sorted(v)[len(v) // 2]:7.1f}" for k, v in res.items()), flush=True)
