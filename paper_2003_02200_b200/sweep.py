"""Rotational-sweep viewshed on the GPU — the reference's independent oracle
(skewshed::oracle, oracle.hpp:10-68 / oracle.cpp:26-194) with the same API:
rays rasterised per azimuth in unskewed grid space, Euclidean distances, no
relocation. Results are bit-identical to the reference's (the per-azimuth
ray tables come from the host's glibc cos/sin/lround/hypot; the FP64 ring
recurrence runs in sweep_dirs_kernel, csrc/sweep.cu).

Areas are in m^2 (total_viewshed_reference: in cfg.units).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib
from .engine import Dem, RunConfig, Units, VsGrid

kReferenceCellGuard = 65536  # oracle.hpp:62


@dataclass(frozen=True)
class GridPoint:
    """oracle.hpp:17-20"""
    i: int = 0
    j: int = 0


@dataclass(frozen=True)
class RingSector:
    """oracle.hpp:24-27: visible interval [r_open, r_close) in cell units."""
    r_open: float = 0.0
    r_close: float = 0.0


@dataclass
class MultiViewshed:
    """oracle.hpp:53-56: grid nonzero only at the observer cells (m^2)."""
    grid: VsGrid
    total_area: float = 0.0


def _md(max_distance: Optional[float]) -> float:
    return 0.0 if max_distance is None else float(max_distance)


def select_axis_point_set(dem: Dem, i0: int, j0: int, azimuth_deg: float) -> list:
    """oracle.cpp:62-71: ray cells nearest first, observer excluded."""
    cnt = C.c_int()
    check(lib.sks_axis_point_set(dem.dimy(), dem.dimx(), i0, j0, float(azimuth_deg), None, 0, C.byref(cnt)))
    ij = np.empty(2 * max(cnt.value, 1), np.int32)
    check(lib.sks_axis_point_set(dem.dimy(), dem.dimx(), i0, j0, float(azimuth_deg), ij.ctypes.data, cnt.value,
                                 C.byref(cnt)))
    return [GridPoint(int(ij[2 * t]), int(ij[2 * t + 1])) for t in range(cnt.value)]


def linear_scan(dem: Dem, i0: int, j0: int, pov_h: float, azimuth_deg: float,
                max_dist_cells: float = float("inf"), rings_out: Optional[list] = None, device: int = 0) -> float:
    """oracle.cpp:74-106: ring sum of one ray (sum of r_close^2 - r_open^2);
    appends the ring sectors to rings_out when given."""
    cv = C.c_double()
    nr = C.c_int()
    check(lib.sks_linear_scan(dem.values.ctypes.data, dem.dimy(), dem.dimx(), int(i0), int(j0), float(pov_h),
                              float(azimuth_deg), float(max_dist_cells), int(device), C.byref(cv), None, 0,
                              C.byref(nr)))
    if rings_out is not None and nr.value > 0:
        buf = np.empty(2 * nr.value, np.float64)
        check(lib.sks_linear_scan(dem.values.ctypes.data, dem.dimy(), dem.dimx(), int(i0), int(j0), float(pov_h),
                                  float(azimuth_deg), float(max_dist_cells), int(device), C.byref(cv),
                                  buf.ctypes.data, nr.value, C.byref(nr)))
        rings_out.extend(RingSector(float(buf[2 * t]), float(buf[2 * t + 1])) for t in range(nr.value))
    return cv.value


def singular_viewshed(dem: Dem, i0: int, j0: int, h0: float, ns: int, max_distance: Optional[float] = None,
                      device: int = 0) -> float:
    """oracle.cpp:108-129: viewshed area (m^2) of one observer."""
    out = C.c_double()
    check(lib.sks_singular_viewshed(dem.values.ctypes.data, dem.dimy(), dem.dimx(), float(dem.cellsize), int(i0),
                                    int(j0), float(h0), int(ns), _md(max_distance), int(device), C.byref(out)))
    return out.value


def multi_viewshed(dem: Dem, povs: Sequence, h0: float, ns: int, max_distance: Optional[float] = None,
                   device: int = 0) -> MultiViewshed:
    """oracle.cpp:131-141: every observer's area at its cell (summed in list
    order for repeated cells) and the total."""
    ij = np.ascontiguousarray([(p.i, p.j) if isinstance(p, GridPoint) else tuple(p) for p in povs],
                              np.int32).reshape(-1, 2)
    grid = np.zeros((dem.dimy(), dem.dimx()), np.float64)
    total = C.c_double()
    check(lib.sks_multi_viewshed(dem.values.ctypes.data, dem.dimy(), dem.dimx(), float(dem.cellsize),
                                 ij.ctypes.data, ij.shape[0], float(h0), int(ns), _md(max_distance), int(device),
                                 None, grid.ctypes.data, C.byref(total)))
    return MultiViewshed(VsGrid(grid, Units.SquareMeters), total.value)


def total_viewshed_reference(dem: Dem, cfg: RunConfig, force: bool = False) -> VsGrid:
    """oracle.cpp:143-194: the singular viewshed of every cell, in cfg.units.
    Grids above kReferenceCellGuard cells raise RuntimeError unless force."""
    out = np.empty((dem.dimy(), dem.dimx()), np.float64)
    nod = C.c_float(dem.nodata) if dem.nodata is not None else None
    check(lib.sks_total_viewshed_reference(dem.values.ctypes.data, dem.dimy(), dem.dimx(), float(dem.cellsize),
                                           C.byref(nod) if nod is not None else None, C.byref(cfg.to_c()),
                                           1 if force else 0, out.ctypes.data))
    return VsGrid(out, Units(cfg.units))


def random_povs(dem: Dem, count: int, seed: int) -> list:
    """cli.cpp:207-221: count observers from raw std::mt19937(seed) draws."""
    ij = np.empty(2 * max(count, 1), np.int32)
    check(lib.sks_random_povs(dem.dimy(), dem.dimx(), int(count), int(seed) & 0xFFFFFFFF, ij.ctypes.data))
    return [GridPoint(int(ij[2 * t]), int(ij[2 * t + 1])) for t in range(count)]
