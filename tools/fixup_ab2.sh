#!/bin/bash
# fixup window-batch variants: default (8 windows + coarse pretest), coarse0, wm16, wm4
O=gpurun_out/${1:-fxc}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -n 2 $O/pytest.log
run() {  # name config steps env...
  n=$1; c=$2; st=$3; shift 3
  env "$@" timeout 900 python bench.py --no-cpu-baseline --config $c --steps $st > $O/c${c}_$n.json 2>$O/c${c}_$n.err
  python -c "
import json; d=json.loads(open('$O/c${c}_$n.json').read().strip().splitlines()[-1]); print('cfg $c $n', round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d['flagged_groups_per_step'])"
}
for c in 2 4; do
  run default $c 3 X=1
  for v in coarse0 wm16 wm4; do run $v $c 3 SKS_LIB=paper_2003_02200_b200/variants/$v.so; done
done
run default 5 1 X=1
run wm16 5 1 SKS_LIB=paper_2003_02200_b200/variants/wm16.so
