import os, sys, time, torch
sys.path.insert(0, "/root/repo")
import paper_2411_01238_b200 as sd
S = 4096
sets = [tuple(torch.randn(S, S, device="cuda").to(torch.bfloat16) for _ in range(3)) for _ in range(3)]
pl5 = [sd.LayerPlan(*s, 0.5) for s in sets]
pl0 = [sd.LayerPlan(*s, 0.0) for s in sets]
def dense(n):
    for i in range(n):
        p = pl5[i % 3]; p.dense_forward(); p.dense_backward()
def p0(n):
    for i in range(n):
        p = pl0[i % 3]; p.forward(i); p.backward()
def p0_nomask(n):
    for i in range(n):
        p = pl0[i % 3]; p.dense_forward(); p.dense_backward()
fns = {"dense(p=0.5 plans)": dense, "p=0 plan fwd+bwd": p0, "dense(p=0 plans)": p0_nomask}
t_end = time.time() + 1.5
while time.time() < t_end:
    for f in fns.values(): f(6)
res = {k: [] for k in fns}
for r in range(8):
    for k, f in fns.items():
        f(3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(20); b.record(); torch.cuda.synchronize()
        res[k].append(a.elapsed_time(b) / 20 * 1e3)
for k, v in res.items():
    v = sorted(v); print(f"{k:22s} {v[len(v)//2]:7.1f} us/step (min {v[0]:.1f})")
