"""Isolates the TMA kernels: relocation alone, then a scan of a given sDEM."""
import sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_02200_b200 as sk
dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 200, 160, 10.0, 7)
for name, fn in [
    ("build_sector_sdem k=0", lambda: sk.build_sector_sdem(dem.values, 0, 180)),
    ("build_sector_sdem k=60", lambda: sk.build_sector_sdem(dem.values, 60, 180)),
    ("sector_viewshed", lambda: sk.sector_viewshed(sk.build_skw(dem.values, 0.3), 1.5)),
    ("total", lambda: sk.total_viewshed(dem, sk.RunConfig(ns=36, h0=1.5, device=0))),
]:
    try:
        fn()
        print("ok", name, flush=True)
    except Exception as e:
        print("FAIL", name, e, flush=True)
        break
