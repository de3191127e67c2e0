"""Per-sector device time of the full pipeline (one sector per run) at a
config, and the imbalance of the static LPT partition at 2/4/8 ranks when
judged by those measured times (multi-GPU load-balance check).

  python tools/sector_costs.py [--config 2] [--out gpurun_out/sector_costs.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_02200_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--out", default="gpurun_out/sector_costs.json")
a = ap.parse_args()
c = bench.CONFIGS[a.config]
n, ns = c["n"], c["ns"]
cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=c["max_distance"])
dem = bench.make_dem(a.config, "fractal")
ctx = sk.Context(0)
d_dem = torch.from_numpy(dem).cuda()
d_map = torch.zeros((n, n), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
times = []
for k in range(ns // 2):
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.run_sectors(d_dem.data_ptr(), n, n, 10.0, cfg, [k], d_map.data_ptr(), stream=st)
        e1.record()
        torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
times = np.array(times)
work = np.array([sk.sector_target_evals(k, ns, n, n, 10.0, c["max_distance"]) for k in range(ns // 2)], float)
res = {"config": a.config, "sector_ms": times.tolist(), "work": work.tolist()}
for world in (2, 4, 8):
    owner = sk.partition_sectors(ns, n, n, world, 10.0, c["max_distance"])
    loads = np.array([times[owner == r].sum() for r in range(world)])
    res[f"lpt_work_eff_{world}"] = float(times.sum() / world / loads.max())
    # LPT on the measured times (what a cost model could reach)
    order = np.argsort(-times)
    bins = np.zeros(world)
    for k in order:
        bins[np.argmin(bins)] += times[k]
    res[f"lpt_time_eff_{world}"] = float(times.sum() / world / bins.max())
print(json.dumps({k: v for k, v in res.items() if not isinstance(v, list)}))
print("corr(time, work) =", float(np.corrcoef(times, work)[0, 1]), "time range", times.min(), times.max())
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    json.dump(res, f)
