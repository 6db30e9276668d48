"""Interleaved A/B of scheduler tuning switches on the layer step (dev tool).
python tools/ab_tuning.py SIZE P flagsA flagsB [rounds]"""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
S = int(sys.argv[1]); P = float(sys.argv[2])
variants = [int(v) for v in sys.argv[3].split(",")]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 8
x = torch.randn(S, S, device="cuda").to(torch.bfloat16)
w = torch.randn(S, S, device="cuda").to(torch.bfloat16)
dy = torch.randn(S, S, device="cuda").to(torch.bfloat16)
plan = sd.LayerPlan(x, w, dy, P)
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
res = {v: {"step": [], "fwd": [], "bwd": [], "dw": [], "dx": [], "dense": []} for v in variants}


def run(v, n=10):
    lib.sd_set_tuning(v)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(9)] for _ in range(n)]
    for i in range(n):
        flush.fill_(1.0)
        e = ev[i]
        e[0].record(); plan.forward(i); e[1].record(); plan.backward(); e[2].record()
        flush.fill_(1.0)
        e[3].record(); plan.dense_forward(); plan.dense_backward(); e[4].record()
        flush.fill_(1.0)
        e[5].record(); plan.backward_dw(); e[6].record()
        flush.fill_(1.0)
        e[7].record(); plan.backward_dx(); e[8].record()
    torch.cuda.synchronize()
    for e in ev:
        res[v]["step"].append(e[0].elapsed_time(e[2]) * 1e3)
        res[v]["fwd"].append(e[0].elapsed_time(e[1]) * 1e3)
        res[v]["bwd"].append(e[1].elapsed_time(e[2]) * 1e3)
        res[v]["dense"].append(e[3].elapsed_time(e[4]) * 1e3)
        res[v]["dw"].append(e[5].elapsed_time(e[6]) * 1e3)
        res[v]["dx"].append(e[7].elapsed_time(e[8]) * 1e3)


for v in variants:
    run(v, 3)
t_end = time.time() + 1.0
while time.time() < t_end:
    plan.forward(0); plan.backward()
for r in range(rounds):
    for v in variants:
        run(v)
for v in variants:
    med = {k: sorted(a)[len(a) // 2] for k, a in res[v].items()}
    print(f"S={S} p={P} tuning={v}: step {med['step']:.1f} us (fwd {med['fwd']:.1f}, bwd {med['bwd']:.1f}; "
          f"dw {med['dw']:.1f}, dx {med['dx']:.1f}), dense {med['dense']:.1f} us", flush=True)
lib.sd_set_tuning(0)
