"""Experiment: where do the fixup's first band targets fall (config N)?
Needs the SKS_EXP_BANDHIST variant: SKS_LIB=.../bandhist.so python tools/bandhist.py 5"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2003_02200_b200 as sk  # noqa: E402
from paper_2003_02200_b200 import _lib  # noqa: E402

cfgid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
terrain = sys.argv[2] if len(sys.argv) > 2 else "fractal"
c = bench.CONFIGS[cfgid]
dem = sk.Dem(bench.make_dem(cfgid, terrain), 10.0)
cfg = sk.RunConfig(ns=c["ns"], h0=1.5, max_distance=c["max_distance"])
lib = ctypes.CDLL(_lib.LIB_PATH)
h = (ctypes.c_ulonglong * 64)()
lib.sks_exp_bandhist(h, 1)
sk.total_viewshed_raw(dem, cfg)
lib.sks_exp_bandhist(h, 1)
v = np.array(list(h), dtype=np.float64)
pov = v[44]
print(f"config {cfgid} {terrain}: fixup POVs {pov:.0f}, without band {v[45]:.0f}")
print("first band at fraction of D (deciles):", np.round(v[0:10] / max(pov, 1), 3).tolist())
print("log2(first band dd):", {i: int(v[10 + i]) for i in range(16) if v[10 + i]})
print("log2(gap to last record + 1):", {i: int(v[26 + i]) for i in range(16) if v[26 + i]})
print(f"evaluated blocks before first band {v[42]:.0f}, after {v[43]:.0f} (prefix share {v[42] / max(v[42] + v[43], 1):.3f})")
