#!/bin/bash
# One bench line per config (diagnostics): tools/cfg_probe.sh 4 5 [-- extra bench args]
mkdir -p gpurun_out/cfg
for c in "$@"; do
  timeout 900 python bench.py --no-cpu-baseline --config $c --steps 1 --warmup 1 > gpurun_out/cfg/probe_c$c.json 2> gpurun_out/cfg/probe_c$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/cfg/probe_c{c}.json").read().strip().splitlines()[-1])
    print(c, round(d["ms_per_step"], 1), {k: round(v, 1) for k, v in d["phase_ms_per_step"].items()},
          d.get("skip_decided_frac"), d.get("flagged_groups_per_step"))
except Exception as e:
    print(c, "ERR", e, open(f"gpurun_out/cfg/probe_c{c}.err").read()[-500:])
PY
done
