"""Times the GPU rotational sweep (total_viewshed_reference, oracle.cpp) against
the reference's own CPU implementation (oracle/_ref, all host threads) and
writes profiles/sweep_bench.json. Usage: python tools/sweep_bench.py [out]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2003_02200_b200 as sk  # noqa: E402
from _oracle import Ref, have_ref  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "sweep_bench.json")
rows = []
for n, ns in ((64, 180), (256, 180), (500, 180), (1000, 180)):
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, n, n, 10.0, 7)
    cfg = sk.RunConfig(ns=ns, h0=1.5, units=sk.Units.SquareMeters)
    sk.sweep.total_viewshed_reference(dem, cfg, force=True)  # warm-up
    t0 = time.perf_counter()
    g = sk.sweep.total_viewshed_reference(dem, cfg, force=True)
    tg = time.perf_counter() - t0
    row = {"n": n, "ns": ns, "gpu_s": tg, "povs_per_s": n * n / tg}
    if have_ref() and n <= 256:
        ref = Ref()
        t0 = time.perf_counter()
        want = ref.total_viewshed_reference(dem.values, ns, 1.5)
        row["ref_cpu_s"] = time.perf_counter() - t0
        row["ref_threads"] = os.cpu_count()
        row["bit_exact"] = bool(np.array_equal(want.view(np.uint64), g.values.view(np.uint64)))
    rows.append(row)
    print(json.dumps(row), flush=True)
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump(rows, open(out, "w"), indent=1)
