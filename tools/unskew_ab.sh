#!/bin/bash
# Unskew A/B: TMA-staged (default) vs register-staged (SKS_UNSKEW_TMA=0); parity suite; ncu of the TMA kernel.
O=gpurun_out/${1:-uab}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
run() {  # name config env...
  n=$1; c=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu-baseline --config $c --steps 5 > $O/c${c}_$n.json 2>$O/c${c}_$n.err
  python -c "
import json; d=json.loads(open('$O/c${c}_$n.json').read().strip().splitlines()[-1]); print('cfg $c $n', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})"
}
for c in 2 4; do
  run tma $c
  run reg $c SKS_UNSKEW_TMA=0
done
SKS_SCAN3=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"unskew_tma_kernel" -c 1 \
  -o $O/unskew python tools/prof_step.py --steps 1 > $O/ncu.log 2>&1
tail -n 3 $O/ncu.log
