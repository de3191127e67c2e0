#!/bin/bash
# Quick GPU check: parity suite + fractal/smooth bench lines (no CPU baseline).
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for t in fractal smooth; do
  timeout 300 python bench.py --no-cpu-baseline --terrain $t > $OUT/bench_$t.json 2> $OUT/bench_$t.err; echo "bench $t rc=$?"
done
python - <<PY
import json,glob
for f in sorted(glob.glob("$OUT/bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"],2), {k:round(v,3) for k,v in d["phase_ms_per_step"].items()}, round(d.get("skip_decided_frac"),3), round(d["roofline"]["frac"],3), round(d["roofline_relocation"]["frac"],3))
    except Exception as e: print(f, "ERR", e)
PY
