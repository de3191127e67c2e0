mkdir -p gpurun_out/cfg
for c in 1 3 4; do
  timeout 600 python bench.py --no-cpu-baseline --config $c --steps 3 --warmup 3 > gpurun_out/cfg/bench_c$c.json 2> gpurun_out/cfg/bench_c$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/cfg/bench_c$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phase_ms_per_step'].items()}, d.get('skip_decided_frac'), d['roofline']['frac'], d['flagged_groups_per_step'])" || tail -5 gpurun_out/cfg/bench_c$c.err
done
