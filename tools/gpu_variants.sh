#!/bin/bash
# usage: bash tools/gpu_variants.sh TAG "ENV1" "ENV2" ...   (runs the GPU parity suite, then bench per env setting)
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
i=0
for ENV in "$@"; do
  i=$((i+1))
  env $ENV timeout 300 python bench.py --no-cpu-baseline > $OUT/bench_$i.json 2> $OUT/bench_$i.err
  python - "$OUT/bench_$i.json" "$ENV" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "| ms/step", round(d["ms_per_step"],2), "| phases", {k:round(v,2) for k,v in d["phase_ms_per_step"].items()}, "| skip", round(d.get("skip_decided_frac") or 0,3), "| frac", round(d["roofline"]["frac"],3), "| e2e", "%.3e"%d["e2e"]["value"])
except Exception as e: print(sys.argv[2], "ERR", e)
PY
done
