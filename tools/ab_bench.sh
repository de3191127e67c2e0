#!/bin/bash
# A/B of env-selected variants on the config-2 bench: tools/ab_bench.sh "ENV=1" "ENV=0" ...
mkdir -p gpurun_out/ab
i=0
for v in "$@"; do
  for rep in 1 2; do
    env $v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab/b_${i}_${rep}.json 2>/dev/null
    python - "$v" gpurun_out/ab/b_${i}_${rep}.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["phase_ms_per_step"].items()},
      d.get("skip_decided_frac"), d.get("flagged_groups_per_step"))
PY
  done
  i=$((i+1))
done
