"""Generates tests/golden/golden.npz from the REFERENCE ITSELF.

Run in the dev container (needs oracle/_ref/libskewshed_ref.so, which
oracle/Makefile builds from the unmodified sources under /root/reference):

    python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/liboracle.so) and the product's
host planning on machines where the reference is absent (the GPU box).
Everything is small: KAT rows, a few sDEMs, sector sweeps and whole-map
totals on grids <= 64^2, plus SHA-256 digests of larger outputs.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from _oracle import NO_CAP, Ref  # noqa: E402

KIND = {"flat": 0, "ramp": 1, "cone": 2, "smooth": 3}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    r = Ref()
    g = {}
    # synthetic DEMs (dem.cpp:118-173)
    for name, k in KIND.items():
        g[f"dem_{name}_17x13_s7"] = r.make_synthetic(k, 17, 13, 7)
    # plan_sector on a rectangular grid for several ns (skew.cpp:23-95)
    plans = []
    for ns in (2, 8, 36, 180):
        for k in range(ns // 2):
            p = r.plan_sector(k, ns, 11, 7)
            plans.append([ns, k, p.sector_deg, p.shear_deg, p.shear_tan, p.rows, p.cols, *p.to_source,
                          len(p.ops), *(list(p.ops) + [-1] * (3 - len(p.ops)))])
    g["plans_11x7"] = np.array(plans, dtype=np.float64)
    # shear params (skew.cpp:97-101)
    sp = []
    for t in (0.0, 1.0, np.tan(np.deg2rad(30.0)), 0.1763269807084649, 0.9999999):
        for j in (0, 1, 3, 4, 17, 1999):
            d, f = r.shear_params(float(t), j)
            sp.append([t, j, d, f])
    g["shear_params"] = np.array(sp)
    # build_skw on a noisy grid at several shears (skew.cpp:144-196)
    grid = r.make_synthetic(3, 20, 24, 5) * 100.0 - 50.0
    grid = grid.astype(np.float32)
    g["skw_grid"] = grid
    for i, t in enumerate([0.0, 0.25, np.tan(np.deg2rad(37.0)), 1.0]):
        v, w, rr, base = r.build_skw(grid, float(t))
        g[f"skw_{i}_t"] = np.array([t])
        g[f"skw_{i}_values"] = v
        g[f"skw_{i}_ranges"] = rr
        g[f"skw_{i}_base"] = np.array([base])
    # linear_viewshed_row KATs (test_scan.cpp:48-150) + random rows
    kat = []
    kat.append(([0, 0, 0, 0, 0], 0, 5, 0, 1.5, 0, NO_CAP))
    kat.append(([3, 17], 0, 2, 0, 5.0, 0, NO_CAP))
    kat.append(([0, 5, 0, 0, 10, 0], 0, 6, 0, 1.0, 0, NO_CAP))
    kat.append(([0, 0, 0], 0, 1, 0, 1.5, 0, NO_CAP))
    kat.append(([0, 0, 0], 2, 3, 2, 1.5, 1, NO_CAP))
    kat.append(([0] * 11, 0, 11, 0, 1.5, 0, 3))
    rng = np.random.default_rng(1234)
    for _ in range(40):
        n = int(rng.integers(2, 60))
        row = list((rng.standard_normal(n) * 20).astype(np.float32))
        first = int(rng.integers(0, n - 1))
        last = int(rng.integers(first + 1, n + 1))
        j0 = int(rng.integers(first, last))
        kat.append((row, first, last, j0, float(row[j0]) + 1.5, int(rng.integers(0, 2)),
                    int(rng.choice([NO_CAP, 4, 17]))))
    rows, meta, cvs, vis = [], [], [], []
    for row, first, last, j0, h, d, cap in kat:
        row = np.array(row, np.float32)
        cv, v = r.linear_viewshed_row(row, first, last, j0, h, d, cap, want_visible=True)
        rows.append(np.pad(row, (0, 64 - len(row)), constant_values=np.nan))
        meta.append([len(row), first, last, j0, h, d, cap])
        cvs.append(cv)
        vis.append(np.pad(v, (0, 64 - len(v))))
    g["kat_rows"] = np.array(rows, np.float32)
    g["kat_meta"] = np.array(meta, np.float64)
    g["kat_cv"] = np.array(cvs)
    g["kat_vis"] = np.array(vis, np.uint8)
    # whole pipeline on small grids (engine.cpp:109-244)
    cases = [("smooth", 3, 16, 16, 7, 36, 0.0), ("cone", 2, 17, 17, 0, 90, 0.0),
             ("ramp", 1, 12, 20, 0, 8, 0.0), ("smooth", 3, 24, 40, 9, 180, 0.0),
             ("smooth", 3, 32, 32, 9, 90, 50.0)]
    for i, (name, k, dy, dx, seed, ns, md) in enumerate(cases):
        dem = r.make_synthetic(k, dy, dx, seed)
        g[f"total_{i}_dem"] = dem
        g[f"total_{i}_cfg"] = np.array([ns, md])
        g[f"total_{i}_raw"] = r.total_viewshed(dem, 10.0, ns, 1.5, max_distance=md, raw=True)
        g[f"total_{i}_sweep3"] = r.sector_sweep(dem, 10.0, ns, 1.5, md, min(3, ns // 2 - 1))
    # digests of a larger case
    dem = r.make_synthetic(3, 64, 64, 7)
    g["digest_64_smooth_ns180_raw"] = np.array(
        [sha(r.total_viewshed(dem, 10.0, 180, 1.5, raw=True))])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
