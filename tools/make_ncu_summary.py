"""Merges one `ncu --set full` capture of a bench workload into
profiles/ncu_summary.json (per config and terrain: the per-launch DRAM traffic
and issue-active figures bench.py reports beside its rooflines).

  python tools/make_ncu_summary.py REPORT.ncu-rep CONFIG TERRAIN "source note"
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, cfg, terrain, note = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]


def val(d, k):
    i = hdr.index(k)
    u = units[i]
    v = float(d[i].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, None)
    return v * scale if scale else v


names = {"scan2_kernel": "scan_kernel", "scan3_kernel": "scan_kernel", "relocate_kernel": "relocate_kernel",
         "unskew_pipe_kernel": "unskew_kernel", "unskew_tma_kernel": "unskew_kernel",
         "fixup_kernel": "fixup_kernel"}
out = {"source": note}
for d in data:
    full = d[hdr.index("Kernel Name")]
    for key, name in names.items():
        if key in full and name not in out:
            try:
                out[name] = {
                    "kernel": full.split("(")[0].split("::")[-1],
                    "duration_ms": val(d, "gpu__time_duration.sum") / (1e6 if units[hdr.index("gpu__time_duration.sum")] == "ns" else 1e3 if units[hdr.index("gpu__time_duration.sum")] == "us" else 1),
                    "dram_bytes_per_launch": val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum"),
                    "issue_active": val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100.0,
                    "warp_instructions": val(d, "smsp__inst_executed.sum"),
                    "fma_pipe": val(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active") / 100.0,
                    "alu_pipe": val(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active") / 100.0,
                }
            except (ValueError, IndexError):
                pass
import math
for k, v in out.items():
    if isinstance(v, dict):
        for kk, vv in v.items():
            if isinstance(vv, float) and math.isnan(vv):
                v[kk] = None
path = os.path.join(ROOT, "profiles", "ncu_summary.json")
try:
    with open(path) as f:
        allsum = json.load(f)
    if "workloads" not in allsum:
        allsum = {"workloads": {}}
except (OSError, ValueError):
    allsum = {"workloads": {}}
allsum["workloads"][f"{cfg}/{terrain}"] = out
with open(path, "w") as f:
    json.dump(allsum, f, indent=1)
print(json.dumps(out, indent=1))
