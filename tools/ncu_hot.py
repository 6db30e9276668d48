"""Top stall-sampled SASS lines per kernel from `ncu -i rep --page source --csv --print-source sass`."""
import csv, io, subprocess, sys
rep = sys.argv[1]; want = sys.argv[2] if len(sys.argv) > 2 else ""; top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name",')[1:]
for b in blocks:
    name = b.split("\n", 1)[0]
    if want not in name: continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]; data = rows[1:]
    si = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source"); ad = h.index("Address")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(float(r[si] or 0) for r in data if len(r) > si)
    print("==", name[:100], "total samples", tot)
    data.sort(key=lambda r: -float(r[si] or 0) if len(r) > si else 0)
    for r in data[:top]:
        s = float(r[si] or 0)
        if s == 0: break
        det = sorted(((float(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:3]
        print(f"{s/tot*100:5.1f}% {r[ad]} {r[src][:60]:60s} " + " ".join(f"{n[6:]}={v:.0f}" for v, n in det if v > 0))
