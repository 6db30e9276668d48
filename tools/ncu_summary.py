"""Summarise an ncu report (--set full) or a launch-list CSV for profiles/.

  python tools/ncu_summary.py full   <report.ncu-rep>   [--json out.json]
  python tools/ncu_summary.py launches <launches.csv>
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_to_sm_read_sectors"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct"),
    # tcgen05 (UTC*) tensor pipe: the metrics that see sm_100 MMAs. The legacy
    # HMMA-pipe counters (sm__pipe_tensor_cycles_active_realtime,
    # sm__inst_executed_pipe_tensor_subpipe_hmma) stay at ~0 for tcgen05 kernels.
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc_pipe_pct_active"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "tc_pipe_pct_elapsed"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tmem_pct_active"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_tc_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
]


def _raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(report, json_out=None):
    h, units, data = _raw(report)
    col = {name: i for i, name in enumerate(h)}
    res = []
    for d in data:
        name = d[col["Kernel Name"]]
        ent = {"kernel": name[:120]}
        for key, short in KEYS:
            full_key = next((k for k in col if k.endswith(key)), None)
            if full_key is None:
                continue
            v = d[col[full_key]].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            ent[short] = v
            ent[short + "_unit"] = units[col[full_key]]
        res.append(ent)
    for e in res:
        print(json.dumps(e))
    if json_out:
        with open(json_out, "w") as f:
            json.dump(res, f, indent=1)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        if r[ui] == "ns":
            v /= 1000.0
        elif r[ui] == "ms":
            v *= 1000.0
        agg.setdefault(r[ki][:110], []).append(v)
    for k, v in agg.items():
        print(f"{len(v):4d} launches  mean {sum(v) / len(v):9.2f} us  last {v[-1]:9.2f} us  {k}")


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "full":
        full(path, sys.argv[4] if len(sys.argv) > 4 and sys.argv[3] == "--json" else None)
    else:
        launches(path)
