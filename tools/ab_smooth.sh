#!/bin/bash
# A/B of library variants on config 2 smooth terrain, 3 reps: tools/ab_smooth.sh TAG lib1.so ...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for rep in 1 2 3; do
  for lib in "$@"; do
    name=$(basename $lib .so)
    if [ "$lib" = "-" ]; then name=intree; L=""; else L="SKS_LIB=$lib"; fi
    env $L timeout 600 python bench.py --no-cpu-baseline --terrain smooth --steps 5 > $OUT/${name}_$rep.json 2> $OUT/${name}_$rep.err
    python - "$name" $OUT/${name}_$rep.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"], 2), {k: round(v, 3) for k, v in d["phase_ms_per_step"].items()})
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
  done
done
