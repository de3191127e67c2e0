#!/bin/bash
# Relocation A/B: default build vs variants ($VARIANTS) at configs 2/4; GPU suite on the default build.
O=gpurun_out/${1:-rab}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -n 2 $O/pytest.log
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
if [ -n "$NCU" ]; then
SKS_SCAN3=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"relocate_kernel" -c 1 \
  -o $O/reloc python tools/prof_step.py --steps 1 > $O/ncu.log 2>&1
fi
