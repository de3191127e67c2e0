#!/bin/bash
# Fixup resume mode A/B on configs 4 and 5: in-tree (resume), resume off, flush-interval variants.
mkdir -p gpurun_out/resab
run() {  # name env... 
  name=$1; shift
  for c in 4 5; do
    st=3; [ $c = 5 ] && st=1
    env "$@" timeout 900 python bench.py --no-cpu-baseline --config $c --steps $st > gpurun_out/resab/${name}_c$c.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/resab/${name}_c$c.json').read().strip().splitlines()[-1]); print('$name cfg $c', round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})"
  done
}
run resume8 SKS_X=1
run off SKS_RESUME_MIN=1000000
run resume4 SKS_LIB=paper_2003_02200_b200/variants/rf4.so
run resume16 SKS_LIB=paper_2003_02200_b200/variants/rf16.so
