#!/bin/bash
# Relocation tile-height variants: parity on each variant (relocation + whole-map tests), then configs 2/4.
O=gpurun_out/${1:-rab}; mkdir -p $O
for v in $VARIANTS; do
  SKS_LIB=paper_2003_02200_b200/variants/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "relocation or build_skw or total_viewshed or config or row_block" > $O/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -n 1 $O/pytest_$v.log
done
run() {  # name config env...
  n=$1; c=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu-baseline --config $c --steps 5 > $O/c${c}_$n.json 2>$O/c${c}_$n.err
  python -c "
import json; d=json.loads(open('$O/c${c}_$n.json').read().strip().splitlines()[-1]); print('cfg $c $n', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['roofline_relocation']['frac'],3))"
}
for c in 2 4; do
  run dflt $c SKS_SCAN3=4
  for v in $VARIANTS; do run $v $c SKS_SCAN3=4 SKS_LIB=paper_2003_02200_b200/variants/$v.so; done
done
