#!/bin/bash
# State check: GPU parity suite + bench on fractal and smooth terrain (no CPU baseline).
TAG=${1:-state}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/gpuinfo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for t in fractal smooth; do
  timeout 300 python bench.py --no-cpu-baseline --terrain $t > $OUT/bench_$t.json 2> $OUT/bench_$t.err; echo "bench $t rc=$?"
done
for c in 3 4; do
  timeout 300 python bench.py --no-cpu-baseline --config $c --steps 3 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; echo "bench c$c rc=$?"
done
timeout 300 python bench.py --no-cpu-baseline --terrain smooth --config 4 --steps 3 > $OUT/bench_c4s.json 2> $OUT/bench_c4s.err
python - <<PY
import json,glob
for f in sorted(glob.glob("$OUT/bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"],2), {k:round(v,2) for k,v in d["phase_ms_per_step"].items()}, round(d.get("skip_decided_frac"),3), round(d["roofline"]["frac"],3), d["flagged_groups_per_step"])
    except Exception as e: print(f, "ERR", e)
PY
