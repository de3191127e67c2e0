#!/bin/bash
# Quick GPU pass: parity suite + bench (new scan and, for comparison, the distance-lockstep scan).
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
if [ -n "$2" ]; then SKS_SCAN=1 timeout 300 python bench.py --no-cpu-baseline > $OUT/bench_v1.json 2> $OUT/bench_v1.err; fi
python - <<PY
import json
for f in ["$OUT/bench.json","$OUT/bench_v1.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["phase_ms_per_step"], d.get("skip_decided_frac"), d["roofline"]["frac"])
    except Exception as e: print(f, "ERR", e)
PY
