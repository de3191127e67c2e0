#!/bin/bash
# A/B of library variants over configs: tools/ab_cfg.sh TAG "configs" lib1.so lib2.so ...
# (variants built with build.py --out paper_2003_02200_b200/variants/NAME.so; "-" = the in-tree library)
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
for c in $CFGS; do
  for lib in "$@"; do
    name=$(basename $lib .so)
    steps=5; [ $c -ge 4 ] && steps=2
    if [ "$lib" = "-" ]; then name=intree; L=""; else L="SKS_LIB=$lib"; fi
    env $L timeout 600 python bench.py --no-cpu-baseline --config $c --steps $steps > $OUT/c${c}_${name}.json 2> $OUT/c${c}_${name}.err
    python - "$name" $c $OUT/c${c}_${name}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    print("cfg", sys.argv[2], sys.argv[1], round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["phase_ms_per_step"].items()},
          round(d.get("skip_decided_frac"), 4), d.get("flagged_groups_per_step"))
except Exception as e:
    print("cfg", sys.argv[2], sys.argv[1], "ERR", e)
PY
  done
done
