#!/bin/bash
# scan kernel modes A/B (SKS_SCAN3: 0 scan2, 1 row pairs, 4 row quads, unset autotune) + parity under quads
mkdir -p gpurun_out/s3ab
SKS_SCAN3=4 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for t in fractal smooth; do
  for v in 4 1 0 auto; do
    if [ $v = auto ]; then E=""; else E="SKS_SCAN3=$v"; fi
    env $E timeout 300 python bench.py --no-cpu-baseline --terrain $t --steps 5 > gpurun_out/s3ab/${t}_$v.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/s3ab/${t}_$v.json').read().strip().splitlines()[-1]); print('$t mode=$v', round(d['ms_per_step'],2), {k: round(x,3) for k,x in d['phase_ms_per_step'].items()}, round(d['skip_decided_frac'],4), d['flagged_groups_per_step'])"
  done
done
