#!/bin/bash
# Fixup A/B: cooperative band blocks (default build) vs per-lane eval_block (variants/nocoop.so); GPU suite on the default.
O=gpurun_out/${1:-fcoop}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -n 2 $O/pytest.log
run() {  # name config steps env...
  n=$1; c=$2; st=$3; shift 3
  env "$@" timeout 900 python bench.py --no-cpu-baseline --config $c --steps $st > $O/c${c}_$n.json 2>$O/c${c}_$n.err
  python -c "
import json; d=json.loads(open('$O/c${c}_$n.json').read().strip().splitlines()[-1]); print('cfg $c $n', round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d['flagged_groups_per_step'])"
}
for c in 2 4 5; do
  st=5; [ $c = 5 ] && st=1
  run coop $c $st
  run nocoop $c $st SKS_LIB=paper_2003_02200_b200/variants/nocoop.so
done
