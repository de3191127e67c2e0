"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

  python tools/launch_summary.py profiles/r01_launches.csv
"""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
tot, cnt = {}, {}
for r in rows[1:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
    try:
        v = float(r[hdr.index("Metric Value")])
    except ValueError:
        continue
    tot[name] = tot.get(name, 0) + v
    cnt[name] = cnt.get(name, 0) + 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:45s} x{cnt[k]:<3d} {v / 1e6:9.3f} ms  {100 * v / s:5.1f}%")
