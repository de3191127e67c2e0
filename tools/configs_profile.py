"""Runs bench.py once per BASELINE config (and terrain) and writes one JSON
with the per-phase times, skip rate, flagged POVs and the bench line's own
rooflines (diagnostic runs, not the bench line).

  python tools/configs_profile.py OUT.json [--terrains fractal,smooth] [--configs 1,2,3,4,5]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--terrains", default="fractal,smooth")
ap.add_argument("--configs", default="1,2,3,4,5")
a = ap.parse_args()
res = {}
for t in a.terrains.split(","):
    for c in [int(x) for x in a.configs.split(",")]:
        steps, warm = (1, 3) if c == 5 else (3, 3)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", "--config", str(c),
                            "--terrain", t, "--steps", str(steps), "--warmup", str(warm)],
                           capture_output=True, text=True, timeout=1800)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            res[f"{c}/{t}"] = {"error": r.stderr[-800:]}
            continue
        res[f"{c}/{t}"] = {
            "workload": d["config"]["workload"], "ms_per_step": d["ms_per_step"], "value": d["value"],
            "unit": d["unit"], "e2e": d["e2e"]["value"], "phase_ms_per_step": d["phase_ms_per_step"],
            "skip_decided_frac": d.get("skip_decided_frac"), "flagged_groups_per_step": d.get("flagged_groups_per_step"),
            "scan_frac": d["roofline"]["frac"], "scan_executed_frac": d["roofline"].get("executed_frac"),
            "relocation_hbm_frac": d["roofline_relocation"]["frac"],
            "unskew_hbm_frac": d.get("roofline_unskew", {}).get("frac"),
            "clocks": d.get("clocks"), "steps": steps, "warmup": warm,
        }
        print(c, t, round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["phase_ms_per_step"].items()},
              flush=True)
res["note"] = ("bench.py --no-cpu-baseline --config N --terrain T (3 timed steps after 3 warm-up, config 5: 1 after "
               "3); diagnostic runs on one B200, not the bench line")
with open(a.out, "w") as f:
    json.dump(res, f, indent=1)
