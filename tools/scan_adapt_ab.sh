#!/bin/bash
# scan2 fine-test adaptation A/B (variants fa1/fa2 vs default), scan2 forced.
O=gpurun_out/${1:-sadapt}; mkdir -p $O
run() {  # name config terrain steps env...
  n=$1; c=$2; t=$3; st=$4; shift 4
  env "$@" timeout 900 python bench.py --no-cpu-baseline --config $c --terrain $t --steps $st > $O/c${c}${t}_$n.json 2>$O/c${c}${t}_$n.err
  python -c "
import json; d=json.loads(open('$O/c${c}${t}_$n.json').read().strip().splitlines()[-1]); print('cfg $c $t $n', round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})"
}
for spec in "2 smooth 5" "2 fractal 5" "4 smooth 2" "5 fractal 1"; do
  set -- $spec
  run dflt $1 $2 $3 SKS_SCAN3=0
  for v in fa1 fa2; do run $v $1 $2 $3 SKS_SCAN3=0 SKS_LIB=paper_2003_02200_b200/variants/$v.so; done
done
