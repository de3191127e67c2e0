"""Emulates N-GPU strong scaling on one GPU: times each rank's share of the
bench workload (row-block sharding, Context.run_rows; or whole sectors by
LPT) one after the other. The N-GPU step time is about the slowest share
(plus one NCCL reduce of the map, ~0.1 ms over NVLink at 2000^2).

  python tools/scaling_emulate.py [--config 2] [--mode rows|sectors]
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
from paper_2003_02200_b200.distributed import RowBalancer, my_sectors  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--mode", default="rows")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--balance", type=int, default=3, help="rebalancing rounds (rows mode, as bench.py's warm-up)")
a = ap.parse_args()
c = bench.CONFIGS[a.config]
n, ns, maxd = c["n"], c["ns"], c["max_distance"]
cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=maxd)
dem = bench.make_dem(a.config, "fractal")
ctx = sk.Context(0)
d_dem = torch.from_numpy(dem).cuda()
d_map = torch.zeros((n, n), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


CUTS = {}


def run(world, rank):
    if a.mode == "rows":
        ctx.run_rows(d_dem.data_ptr(), n, n, 10.0, cfg, rank, world, d_map.data_ptr(), stream=st,
                     cuts=CUTS.get(world))
    else:
        ctx.run_sectors(d_dem.data_ptr(), n, n, 10.0, cfg, my_sectors(ns, n, n, world, rank, 10.0, maxd),
                        d_map.data_ptr(), stream=st)


def time_rank(world, rank, reps):
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        run(world, rank)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {"config": a.config, "mode": a.mode, "balance_rounds": a.balance if a.mode == "rows" else 0}
for world in (1, 2, 4, 8):
    if a.mode == "rows" and world > 1 and a.balance > 0:
        bal = RowBalancer(world)
        hist = []
        for _ in range(a.balance):  # bench.py's warm-up: measure (kernel phases), move the cuts
            CUTS[world] = bal.cuts
            t = []
            for r in range(world):
                es = ctx.run_rows(d_dem.data_ptr(), n, n, 10.0, cfg, r, world, d_map.data_ptr(), stream=st,
                                  want_stats=True, cuts=bal.cuts)
                t.append((es.skew_seconds + es.scan_seconds + es.fixup_seconds + es.unskew_seconds) * 1e3)
            hist.append(round(max(t) / (sum(t) / world), 4))
            bal.update(t)
        CUTS[world] = bal.cuts
        out[f"imbalance_history_{world}"] = hist
        out[f"cuts_{world}"] = [round(float(x), 5) for x in bal.cuts]
    times = []
    for rank in range(world):
        run(world, rank)  # warm (plans, pools)
        best = 1e30
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            run(world, rank)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        times.append(best)
    out[world] = {"rank_ms": [round(x, 3) for x in times], "max_ms": max(times)}
    if world == 8 and a.mode == "rows":
        phases = []
        for rank in range(world):
            es = ctx.run_rows(d_dem.data_ptr(), n, n, 10.0, cfg, rank, world, d_map.data_ptr(), stream=st,
                              want_stats=True, cuts=CUTS.get(world))
            phases.append({k: round(getattr(es, k) * 1e3, 3) for k in
                           ("skew_seconds", "scan_seconds", "fixup_seconds", "unskew_seconds")})
        out["phases_8"] = phases
base = out[1]["max_ms"]
for world in (1, 2, 4, 8):
    out[world]["efficiency"] = base / world / out[world]["max_ms"]
print(json.dumps(out))
