"""Full-size parity evidence: the whole config-2 total viewshed (2000^2
fractal, 180 sectors, raw map) from the GPU path against the reference's own
total_viewshed_raw (oracle/_ref, all host threads). Writes a JSON summary.

  python tools/full_parity.py [--config 2] [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
import paper_2003_02200_b200 as sk  # noqa: E402
from _oracle import Ref  # noqa: E402

cfgid = 2
out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "full_parity.json")
c = bench.CONFIGS[cfgid]
dem = sk.Dem(bench.make_dem(cfgid, "fractal"), 10.0)
cfg = sk.RunConfig(ns=c["ns"], h0=1.5, max_distance=c["max_distance"], units=sk.Units.SquareMeters)
t0 = time.perf_counter()
ours = sk.total_viewshed_raw(dem, cfg)
t_gpu = time.perf_counter() - t0
threads = os.cpu_count() or 1
t0 = time.perf_counter()
ref = Ref().total_viewshed(dem.values, 10.0, c["ns"], 1.5, max_distance=c["max_distance"] or 0.0, raw=True,
                           workers=threads)
t_ref = time.perf_counter() - t0
same = bool(np.array_equal(ours.view(np.uint64), ref.view(np.uint64)))
rel = np.abs(ours - ref) / np.maximum(np.abs(ref), 1e-300)
res = {"workload": bench.workload_name(cfgid, "fractal"), "map": "total_viewshed_raw (sum of cv * (1 + tan^2))",
       "bit_identical": same, "max_rel_err": float(rel.max()), "cells": int(ours.size),
       "gpu_s_incl_first_call": round(t_gpu, 3), "reference_s": round(t_ref, 2), "reference_threads": threads}
print(json.dumps(res))
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump(res, open(out, "w"), indent=1)
