timeout 600 python tools/dbg_tma.py 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for rep in 1 2; do
for t in fractal smooth; do
  for v in 1 0; do
    SKS_SCAN3=$v timeout 300 python bench.py --no-cpu-baseline --terrain $t --steps 5 > gpurun_out/s3_${t}_$v.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/s3_${t}_$v.json').read().strip().splitlines()[-1]); print('$t scan3=$v', round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['skip_decided_frac'],4), d['flagged_groups_per_step'])"
  done
done
done
