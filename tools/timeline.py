"""Device timeline of one SparseDrop layer step (dev tool; needs `make trace`).

  SPARSEDROP_B200_LIB=paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so python tools/timeline.py [SIZE] [P] [STEPS]
Prints, per launch of the step, the first CTA's start, when it passed
griddepcontrol.wait (PDL), and the last CTA's end (globaltimer, ns)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SPARSEDROP_B200_LIB", os.path.join(ROOT, "paper_2411_01238_b200/lib/libsparsedrop_b200_trace.so"))
import paper_2411_01238_b200 as sd  # noqa: E402

lib = sd.load_library()
lib.sd_timeline_read.argtypes = [ctypes.c_void_p]
lib.sd_mask_timeline_read.argtypes = [ctypes.c_void_p]
S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
P = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
BACK_TO_BACK = int(sys.argv[3]) if len(sys.argv) > 3 else 1  # steps per timed burst (bench.py runs them back to back)
GATE = len(sys.argv) > 4 and sys.argv[4] == "gate"  # spin first: every step is queued before the first runs
x = torch.randn(S, S, device="cuda").to(torch.bfloat16)
w = torch.randn(S, S, device="cuda").to(torch.bfloat16)
dy = torch.randn(S, S, device="cuda").to(torch.bfloat16)
plan = sd.LayerPlan(x, w, dy, P, dy_ready=True)
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
g = np.zeros(256 * 4, dtype=np.uint64)
mk = np.zeros(256 * 4, dtype=np.uint64)
for it in range(4):
    lib.sd_timeline_read(g.ctypes.data)
    lib.sd_mask_timeline_read(mk.ctypes.data)
    flush.fill_(1.0)
    torch.cuda.synchronize()
    l0 = sd.launch_count()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if GATE:
        torch.cuda._sleep(int(4e6))
    a.record()
    for rep in range(BACK_TO_BACK):
        plan.forward(it * 8 + rep)
        plan.backward()
    b.record()
    torch.cuda.synchronize()
    l1 = sd.launch_count()
    lib.sd_timeline_read(g.ctypes.data)
    lib.sd_mask_timeline_read(mk.ctypes.data)
    rows = []
    for lid in range(l0, l1):
        i = lid & 255
        for name, arr in (("gemm", g), ("mask", mk)):
            st, wt, en = int(arr[4 * i]), int(arr[4 * i + 1]), int(arr[4 * i + 2])
            if en and st != 0xFFFFFFFFFFFFFFFF:
                rows.append((st, name, lid, wt, en))
    rows.sort()
    t0 = rows[0][0]
    print(f"-- step {it}: event time {a.elapsed_time(b) * 1e3:.1f} us; device span {(max(r[4] for r in rows) - t0) / 1e3:.1f} us")
    prev_end = None
    for st, name, lid, wt, en in rows:
        if name == "mask":
            lw, od = int(mk[4 * (lid & 255) + 1]), int(mk[4 * (lid & 255) + 3])
            wait = (f" last-past-wait {(lw - t0) / 1e3:7.1f}" if lw else "") + (f" order {(od - t0) / 1e3:7.1f}" if od else "")
        else:
            wait = "" if wt == 0xFFFFFFFFFFFFFFFF else f" past-wait {(wt - t0) / 1e3:7.1f}"
            rl = int(g[4 * (lid & 255) + 3])
            if rl and rl != 0xFFFFFFFFFFFFFFFF:
                wait += f" released {(rl - t0) / 1e3:7.1f}"
        gap = "" if prev_end is None else f" (gap from prev end {(st - prev_end) / 1e3:+.1f})"
        print(f"   {name:5s} #{lid}: start {(st - t0) / 1e3:7.1f}{wait} end {(en - t0) / 1e3:7.1f}  dur {(en - st) / 1e3:6.1f} us{gap}")
        prev_end = en
