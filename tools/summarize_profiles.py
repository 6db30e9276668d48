"""Summarise a capture_profiles.sh run into profiles/ (run here, after gpurun).

  python tools/summarize_profiles.py r01
writes profiles/<tag>_ncu_full.json (per-kernel metrics from ncu --set full),
profiles/<tag>_launches.txt (launch list shares), profiles/<tag>_bench.json,
profiles/<tag>_bench_ref.json and profiles/ncu_traffic.json (DRAM bytes per
launch of each GEMM, read by bench.py for roofline.traffic)."""
import io
import json
import shutil
import sys
from contextlib import redirect_stdout
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import ncu_summary  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
g = ROOT / "gpurun_out"
prof = ROOT / "profiles"
prof.mkdir(exist_ok=True)

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# capture order of tools/capture_profiles.sh (all GEMMs share one kernel name)
ROLES_IN_ORDER = ["mask_gen+compact", "dsd_fwd", "bwd_fused(dsd_dw+sdd_dx)"]

rep = g / f"{tag}_full.ncu-rep"
if rep.exists():
    buf = io.StringIO()
    with redirect_stdout(buf):
        res = ncu_summary.full(str(rep))
    out, traffic = [], {}
    for idx, e in enumerate(res):
        role = ROLES_IN_ORDER[idx] if idx < len(ROLES_IN_ORDER) else e["kernel"][:60]
        e["role"] = role
        rd = e.get("dram_read", 0) * UNIT.get(e.get("dram_read_unit", "byte"), 1)
        wr = e.get("dram_write", 0) * UNIT.get(e.get("dram_write_unit", "byte"), 1)
        e["dram_bytes_per_launch"] = rd + wr
        traffic[role] = rd + wr
        out.append(e)
    (prof / f"{tag}_ncu_full.json").write_text(json.dumps(out, indent=1))
    (prof / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1))
    print("ncu full:", {e["role"]: (e.get("duration"), e["dram_bytes_per_launch"]) for e in out})

lc = g / f"{tag}_launches.csv"
if lc.exists():
    buf = io.StringIO()
    with redirect_stdout(buf):
        ncu_summary.launches(str(lc))
    (prof / f"{tag}_launches.txt").write_text(
        "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) of\n"
        "`python bench.py --profile --steps 3 --warmup 2 --no-cpu`; per kernel: launches, mean and last duration\n\n"
        + buf.getvalue())
    print(buf.getvalue())
for name in (f"{tag}_bench.json", f"{tag}_bench_ref.json", "host.txt"):
    if (g / name).exists():
        shutil.copy(g / name, prof / (name if name != "host.txt" else f"{tag}_host.txt"))
