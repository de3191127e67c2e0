"""Per-instruction / per-opcode breakdown of one kernel in an ncu report.

  python tools/sass_hot.py REPORT.ncu-rep KERNEL_REGEX [top_n]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
ie = hdr.index("Instructions Executed")
smp = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
tot = sum(float(r[ie] or 0) for r in data)
ts = sum(float(r[smp] or 0) for r in data)
print(f"{tot / 1e6:.1f}M warp instructions, {ts:.0f} samples, {len(data)} SASS lines")
op, ops = collections.Counter(), collections.Counter()
for r in data:
    o = [x for x in r[src].split() if not x.startswith("@")]
    name = o[0].split(".")[0] if o else "?"
    op[name] += float(r[ie] or 0)
    ops[name] += float(r[smp] or 0)
for k, v in op.most_common(top):
    print(f"  {k:10s} inst {100 * v / tot:5.1f}%  samples {100 * ops[k] / ts:5.1f}%")
print("hot lines:")
for i, r in enumerate(data):
    v, s = float(r[ie] or 0), float(r[smp] or 0)
    if v > 0.01 * tot or s > 0.015 * ts:
        print(f"  {i:4d} {r[src][:70]:70s} inst {100 * v / tot:5.1f}% samples {100 * s / ts:5.1f}%")
