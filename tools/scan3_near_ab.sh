for c in 2 3 4; do for v in "" ne0 ne32 ne48; do
  if [ -z "$v" ]; then L=""; n=default; else L="SKS_LIB=paper_2003_02200_b200/variants/$v.so"; n=$v; fi
  st=5; [ $c = 4 ] && st=2
  env SKS_SCAN3=4 $L timeout 600 python bench.py --no-cpu-baseline --config $c --steps $st > gpurun_out/ne_${c}_$n.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ne_${c}_$n.json').read().strip().splitlines()[-1]); print('cfg $c $n', round(d['ms_per_step'],2), round(d['phase_ms_per_step']['scan'],3), round(d['skip_decided_frac'],4))"
done; done
for c in 3 4; do for m in 1 0; do
  st=5; [ $c = 4 ] && st=2
  SKS_SCAN3=$m timeout 600 python bench.py --no-cpu-baseline --config $c --steps $st > gpurun_out/ne_m${m}_$c.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ne_m${m}_$c.json').read().strip().splitlines()[-1]); print('cfg $c mode $m', round(d['ms_per_step'],2), round(d['phase_ms_per_step']['scan'],3))"
done; done
