"""Per-CUDA-source-line instruction / stall breakdown of one kernel in an ncu report.

  python tools/ncu_lines.py REPORT.ncu-rep [KERNEL_REGEX] [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
ie, smp, te = (hdr.index(k) for k in ("Instructions Executed", "Warp Stall Sampling (All Samples)",
                                       "Thread Instructions Executed"))
lines = [r for r in rows[hi + 1:] if len(r) > ie and r[2] == "-" and r[0].isdigit()]
tot = sum(float(r[ie] or 0) for r in lines)
ts = sum(float(r[smp] or 0) for r in lines)
print(f"{tot / 1e9:.2f} G warp instructions, {ts:.0f} samples")
for r in sorted(lines, key=lambda r: -float(r[smp] or 0))[:top]:
    w, t = float(r[ie] or 0), float(r[te] or 0)
    print(f"{r[0]:>4} inst {100 * w / tot:5.1f}% smp {100 * float(r[smp] or 0) / ts:5.1f}% "
          f"thr/warp {t / max(w, 1):5.1f}  {r[1][:88]}")
