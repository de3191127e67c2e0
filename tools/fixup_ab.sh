mkdir -p gpurun_out/r02n
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02n/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02n/pytest_gpu.log
tail -3 gpurun_out/r02n/pytest_gpu.log
for c in 2 4; do
  for f in warp thread; do
    SKS_FIXUP=$f timeout 600 python bench.py --no-cpu-baseline --config $c --steps 3 > gpurun_out/r02n/c${c}_$f.json 2>gpurun_out/r02n/c${c}_$f.err
    python -c "
import json; d=json.loads(open('gpurun_out/r02n/c${c}_$f.json').read().strip().splitlines()[-1]); print('cfg $c $f', round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d['flagged_groups_per_step'])"
  done
done
for f in warp thread; do
  SKS_FIXUP=$f timeout 900 python bench.py --no-cpu-baseline --config 5 --steps 1 --warmup 3 > gpurun_out/r02n/c5_$f.json 2>gpurun_out/r02n/c5_$f.err
  python -c "
import json; d=json.loads(open('gpurun_out/r02n/c5_$f.json').read().strip().splitlines()[-1]); print('cfg 5 $f', round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d['flagged_groups_per_step'])"
done
