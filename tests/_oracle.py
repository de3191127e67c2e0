"""TEST INFRASTRUCTURE: ctypes bindings to the two CPU oracles.

* ``Ref``  — the unmodified reference library (oracle/_ref/libskewshed_ref.so,
  built by oracle/Makefile from /root/reference/proj/src + oracle/ref_shim.cpp).
* ``Orc``  — the plain-C restatement (oracle/liboracle.so from
  oracle/skewshed_oracle.c).

Both expose the same small numpy-level API so a test can be parametrised over
them. Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg
import this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libskewshed_ref.so")
ORC_SO = os.path.join(ROOT, "oracle", "liboracle.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")

NO_CAP = 2147483647


def base_offset(src_rows: int, cols: int, shear_tan: float) -> int:
    """skew.cpp:16-19."""
    dest_max = int(shear_tan * (cols - 1))
    return max(src_rows, dest_max + 1)


@dataclass
class Plan:
    k: int
    ns: int
    sector_deg: float
    shear_deg: float
    shear_tan: float
    rows: int
    cols: int
    to_source: tuple  # ii, ij, ci, ji, jj, cj
    ops: tuple


class _OrcPlan(C.Structure):
    _fields_ = [
        ("sector_index", C.c_int), ("ns", C.c_int),
        ("sector_deg", C.c_double), ("shear_deg", C.c_double), ("shear_tan", C.c_double),
        ("n_ops", C.c_int), ("ops", C.c_int * 3),
        ("rows", C.c_int), ("cols", C.c_int), ("src_rows", C.c_int), ("src_cols", C.c_int),
        ("ii", C.c_int), ("ij", C.c_int), ("ci", C.c_int),
        ("ji", C.c_int), ("jj", C.c_int), ("cj", C.c_int),
    ]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def have_orc() -> bool:
    return os.path.exists(ORC_SO)


class Ref:
    """The reference itself (via oracle/ref_shim.cpp)."""

    name = "ref"

    def __init__(self):
        lib = C.CDLL(REF_SO)
        self.lib = lib
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_make_synthetic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint32, _f32p]
        lib.ref_plan_sector.argtypes = [C.c_int] * 4 + [_f64p, _i32p, _i32p, _i32p, _i32p]
        lib.ref_shear_params.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)]
        lib.ref_apply_pre_ops.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p]
        lib.ref_build_skw.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, _f32p, _f32p,
                                      _i32p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.ref_linear_viewshed_row.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                                C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_int)]
        lib.ref_linear_viewshed_row.restype = C.c_double
        lib.ref_sector_viewshed.argtypes = [_f32p, _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                            C.c_double, C.c_int, _f64p]
        lib.ref_unskew_accumulate.argtypes = [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64p]
        lib.ref_sector_sweep.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                         C.c_int, _f64p, C.c_void_p]
        lib.ref_total_viewshed.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int,
                                           C.c_double, C.c_int, C.c_int, _f64p, C.c_void_p]
        lib.ref_area_scale_factor.argtypes = [C.c_int, C.c_double, C.c_int]
        lib.ref_area_scale_factor.restype = C.c_double
        lib.ref_rotational_total_viewshed.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double,
                                                      C.c_double, _f64p]
        lib.ref_make_fractal.argtypes = [C.c_int, C.c_int, C.c_uint32, _f32p]
        lib.ref_sweep_sample.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                         _i32p, C.c_int, C.c_int, C.POINTER(C.c_double)]
        lib.ref_sector_work.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double]
        lib.ref_sector_work.restype = C.c_longlong

        lib.ref_singular_viewshed.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                              C.c_int, C.c_double, C.POINTER(C.c_double)]
        lib.ref_multi_viewshed.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int, C.c_double,
                                           C.c_int, C.c_double, _f64p, C.POINTER(C.c_double)]
        lib.ref_total_viewshed_reference.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                                     C.c_double, C.c_double, C.c_int, C.c_int, _f64p]
        lib.ref_axis_point_set.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                           C.POINTER(C.c_int)]
        lib.ref_write_heatmap.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
        lib.ref_fill_nodata_nearest.argtypes = [_f32p, C.c_int, C.c_int, C.c_float, _f32p]
        lib.ref_linear_scan.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.POINTER(C.c_double), C.c_void_p, C.c_int, C.POINTER(C.c_int)]

    # ---- rotational sweep (oracle.cpp) / heatmap (heatmap.cpp) ----
    def singular_viewshed(self, dem, i, j, h0, ns, max_distance=None, cellsize=10.0):
        out = C.c_double()
        d = np.ascontiguousarray(dem, np.float32)
        self._check(self.lib.ref_singular_viewshed(d, d.shape[0], d.shape[1], cellsize, i, j, h0, ns,
                                                   max_distance or 0.0, C.byref(out)))
        return out.value

    def multi_viewshed(self, dem, povs, h0, ns, max_distance=None, cellsize=10.0):
        d = np.ascontiguousarray(dem, np.float32)
        ij = np.ascontiguousarray(povs, np.int32).reshape(-1, 2)
        grid = np.empty(d.shape, np.float64)
        tot = C.c_double()
        self._check(self.lib.ref_multi_viewshed(d, d.shape[0], d.shape[1], cellsize, ij.ctypes.data, ij.shape[0],
                                                h0, ns, max_distance or 0.0, grid, C.byref(tot)))
        return grid, tot.value

    def total_viewshed_reference(self, dem, ns, h0, max_distance=None, units=0, force=True, cellsize=10.0,
                                 nodata=None):
        d = np.ascontiguousarray(dem, np.float32)
        out = np.empty(d.shape, np.float64)
        nod = C.c_float(nodata) if nodata is not None else None
        self._check(self.lib.ref_total_viewshed_reference(d, d.shape[0], d.shape[1], cellsize,
                                                          C.byref(nod) if nod is not None else None, ns, h0,
                                                          max_distance or 0.0, units, 1 if force else 0, out))
        return out

    def axis_point_set(self, dimy, dimx, i0, j0, az):
        cnt = C.c_int()
        ij = np.empty(2 * (dimy + dimx + 2), np.int32)
        self._check(self.lib.ref_axis_point_set(dimy, dimx, i0, j0, az, ij.ctypes.data, dimy + dimx + 1,
                                                C.byref(cnt)))
        return [(int(ij[2 * t]), int(ij[2 * t + 1])) for t in range(cnt.value)]

    def fill_nodata_nearest(self, dem, nodata):
        d = np.ascontiguousarray(dem, np.float32)
        out = np.empty_like(d)
        self._check(self.lib.ref_fill_nodata_nearest(d, d.shape[0], d.shape[1], nodata, out))
        return out

    def linear_scan(self, dem, i0, j0, pov_h, az, max_cells=float("inf")):
        d = np.ascontiguousarray(dem, np.float32)
        cv, nr = C.c_double(), C.c_int()
        buf = np.empty(2 * (d.shape[0] + d.shape[1] + 2), np.float64)
        self._check(self.lib.ref_linear_scan(d, d.shape[0], d.shape[1], i0, j0, pov_h, az, max_cells, C.byref(cv),
                                             buf.ctypes.data, buf.size // 2, C.byref(nr)))
        return cv.value, [(float(buf[2 * t]), float(buf[2 * t + 1])) for t in range(nr.value)]

    def write_heatmap(self, path, values, palette):
        v = np.ascontiguousarray(values, np.float64)
        rows, cols = v.shape if v.ndim == 2 else (0, 0)
        self._check(self.lib.ref_write_heatmap(str(path).encode(), v.ctypes.data, rows, cols, palette))

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            if rc == 1:
                raise ValueError(msg)
            if rc == 2:
                raise IndexError(msg)
            raise RuntimeError(msg)

    def make_synthetic(self, kind: int, dimy: int, dimx: int, seed: int = 0) -> np.ndarray:
        out = np.empty((dimy, dimx), np.float32)
        self._check(self.lib.ref_make_synthetic(kind, dimy, dimx, 10.0, seed, out))
        return out

    def plan_sector(self, k, ns, dimy, dimx) -> Plan:
        degs = np.zeros(3, np.float64)
        shape = np.zeros(2, np.int32)
        m = np.zeros(6, np.int32)
        ops = np.zeros(3, np.int32)
        nops = np.zeros(1, np.int32)
        self._check(self.lib.ref_plan_sector(k, ns, dimy, dimx, degs, shape, m, ops, nops))
        return Plan(k, ns, degs[0], degs[1], degs[2], int(shape[0]), int(shape[1]),
                    tuple(int(x) for x in m), tuple(int(x) for x in ops[: nops[0]]))

    def shear_params(self, t, j):
        d = C.c_int()
        f = C.c_double()
        self.lib.ref_shear_params(t, j, C.byref(d), C.byref(f))
        return d.value, f.value

    def apply_pre_ops(self, dem, k, ns):
        p = self.plan_sector(k, ns, *dem.shape)
        out = np.empty((p.rows, p.cols), np.float32)
        self._check(self.lib.ref_apply_pre_ops(np.ascontiguousarray(dem), dem.shape[0], dem.shape[1], k, ns, out))
        return out

    def build_skw(self, g, shear_tan):
        rows, cols = g.shape
        cap = rows + max(rows, cols) + 2
        vals = np.zeros((cap, cols), np.float32)
        w = np.zeros((cap, cols), np.float32)
        rr = np.zeros((cap, 2), np.int32)
        sr = C.c_int()
        b = C.c_int()
        self._check(self.lib.ref_build_skw(np.ascontiguousarray(g), rows, cols, shear_tan, cap, vals, w, rr,
                                           C.byref(sr), C.byref(b)))
        n = sr.value
        return vals[:n].copy(), w[:n].copy(), rr[:n].copy(), b.value

    def linear_viewshed_row(self, row, first, last, j0, h, direction, max_dd=NO_CAP, want_visible=False):
        row = np.ascontiguousarray(row, np.float32)
        vis = np.zeros(max(1, len(row)), np.uint8)
        nv = C.c_int()
        cv = self.lib.ref_linear_viewshed_row(row, len(row), first, last, j0, h, direction, max_dd,
                                              vis.ctypes.data if want_visible else None, C.byref(nv))
        if want_visible:
            return cv, vis[: nv.value].copy()
        return cv

    def sector_viewshed(self, vals, ranges, src_rows, base, shear_tan, h0, max_dd=NO_CAP):
        skw_rows, cols = vals.shape
        out = np.zeros((skw_rows, cols), np.float64)
        self._check(self.lib.ref_sector_viewshed(np.ascontiguousarray(vals), np.ascontiguousarray(ranges, np.int32),
                                                 skw_rows, cols, src_rows, base, shear_tan, h0, max_dd, out))
        return out

    def unskew_accumulate(self, skw_vs, k, ns, dimy, dimx, out=None):
        if out is None:
            out = np.zeros((dimy, dimx), np.float64)
        self._check(self.lib.ref_unskew_accumulate(np.ascontiguousarray(skw_vs), skw_vs.shape[0], skw_vs.shape[1],
                                                   k, ns, dimy, dimx, out))
        return out

    def sector_sweep(self, dem, cellsize, ns, h0, max_distance, k):
        out = np.zeros(dem.shape, np.float64)
        self._check(self.lib.ref_sector_sweep(np.ascontiguousarray(dem), dem.shape[0], dem.shape[1], cellsize, ns,
                                              h0, max_distance or 0.0, k, out, None))
        return out

    def total_viewshed(self, dem, cellsize, ns, h0, max_distance=0.0, units=0, raw=False, workers=None):
        out = np.zeros(dem.shape, np.float64)
        stats = np.zeros(5, np.float64)
        workers = workers or (os.cpu_count() or 1)
        self._check(self.lib.ref_total_viewshed(np.ascontiguousarray(dem), dem.shape[0], dem.shape[1], cellsize, ns,
                                                h0, workers, max_distance or 0.0, units, int(raw), out,
                                                stats.ctypes.data))
        return out

    def area_scale_factor(self, ns, cellsize, units):
        return self.lib.ref_area_scale_factor(ns, cellsize, units)

    def rotational_total_viewshed(self, dem, cellsize, ns, h0, max_distance=0.0):
        out = np.zeros(dem.shape, np.float64)
        self._check(self.lib.ref_rotational_total_viewshed(np.ascontiguousarray(dem), dem.shape[0], dem.shape[1],
                                                           cellsize, ns, h0, max_distance or 0.0, out))
        return out

    def make_fractal(self, dimy, dimx, seed=7) -> np.ndarray:
        """The bench's fractal terrain (restated in ref_shim.cpp)."""
        out = np.empty((dimy, dimx), np.float32)
        self._check(self.lib.ref_make_fractal(dimy, dimx, seed, out))
        return out

    def sweep_sample(self, dem, cellsize, ns, h0, max_distance, sectors, threads) -> float:
        """Wall seconds of the reference's sector_sweep on `sectors`, claimed
        dynamically by `threads` host threads."""
        sec = C.c_double()
        s = np.ascontiguousarray(sectors, np.int32)
        self._check(self.lib.ref_sweep_sample(np.ascontiguousarray(dem), dem.shape[0], dem.shape[1], cellsize, ns,
                                              h0, max_distance or 0.0, s, len(s), threads, C.byref(sec)))
        return sec.value

    def sector_work(self, dimy, dimx, cellsize, ns, k, max_distance=None) -> int:
        """Exact target evaluations of sector k from the reference's own row ranges."""
        w = self.lib.ref_sector_work(dimy, dimx, cellsize, ns, k, max_distance or 0.0)
        if w < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return int(w)


class Orc:
    """The C restatement (oracle/skewshed_oracle.c)."""

    name = "orc"

    def __init__(self):
        lib = C.CDLL(ORC_SO)
        self.lib = lib
        lib.orc_make_synthetic.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint32, _f32p]
        lib.orc_plan_sector.argtypes = [C.c_int] * 4 + [C.POINTER(_OrcPlan)]
        lib.orc_shear_params.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)]
        lib.orc_apply_pre_ops.argtypes = [_f32p, C.POINTER(_OrcPlan), _f32p]
        lib.orc_build_skw.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, _f32p, _f32p, _i32p, C.POINTER(C.c_int)]
        lib.orc_linear_viewshed_row.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                                C.c_void_p, C.POINTER(C.c_int)]
        lib.orc_linear_viewshed_row.restype = C.c_double
        lib.orc_sector_viewshed.argtypes = [_f32p, _i32p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _f64p]
        lib.orc_unskew_accumulate.argtypes = [_f64p, C.c_int, C.c_int, C.POINTER(_OrcPlan), _f64p]
        lib.orc_distance_cap_cells.argtypes = [C.c_double, C.c_double, C.c_double]
        lib.orc_sector_sweep.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                         C.c_int, _f64p]
        lib.orc_area_scale_factor.argtypes = [C.c_int, C.c_double, C.c_int]
        lib.orc_area_scale_factor.restype = C.c_double
        lib.orc_total_viewshed.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                           C.c_int, C.c_int, C.c_int, C.c_int, _f64p]
        lib.orc_mt19937_nth.argtypes = [C.c_uint32, C.c_int]
        lib.orc_mt19937_nth.restype = C.c_uint32
        lib.orc_singular_viewshed.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                              C.c_int, C.c_double, C.POINTER(C.c_double)]
        lib.orc_rotational_rows.argtypes = [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                            C.c_int, C.c_int, C.c_int, _f64p]

    def singular_viewshed(self, dem, i, j, h0, ns, max_distance=None, cellsize=10.0):
        out = C.c_double()
        d = np.ascontiguousarray(dem, np.float32)
        self._check(self.lib.orc_singular_viewshed(d, d.shape[0], d.shape[1], cellsize, i, j, h0, ns,
                                                   max_distance or 0.0, C.byref(out)))
        return out.value

    def rotational_rows(self, dem, ns, h0, max_distance=None, units=0, rows=None, cellsize=10.0):
        """total_viewshed_reference restated, on rows [lo, hi) (NaN elsewhere)."""
        d = np.ascontiguousarray(dem, np.float32)
        out = np.full(d.shape, np.nan)
        lo, hi = rows if rows else (0, d.shape[0])
        self._check(self.lib.orc_rotational_rows(d, d.shape[0], d.shape[1], cellsize, ns, h0, max_distance or 0.0,
                                                 units, lo, hi, out))
        return out

    def _check(self, rc):
        if rc == 1:
            raise ValueError("invalid argument")
        if rc == 2:
            raise IndexError("out of range")
        if rc:
            raise RuntimeError(f"oracle error {rc}")

    def make_synthetic(self, kind, dimy, dimx, seed=0):
        out = np.empty((dimy, dimx), np.float32)
        self._check(self.lib.orc_make_synthetic(kind, dimy, dimx, seed, out))
        return out

    def _plan(self, k, ns, dimy, dimx):
        p = _OrcPlan()
        self._check(self.lib.orc_plan_sector(k, ns, dimy, dimx, C.byref(p)))
        return p

    def plan_sector(self, k, ns, dimy, dimx) -> Plan:
        p = self._plan(k, ns, dimy, dimx)
        return Plan(k, ns, p.sector_deg, p.shear_deg, p.shear_tan, p.rows, p.cols,
                    (p.ii, p.ij, p.ci, p.ji, p.jj, p.cj), tuple(p.ops[i] for i in range(p.n_ops)))

    def shear_params(self, t, j):
        d = C.c_int()
        f = C.c_double()
        self.lib.orc_shear_params(t, j, C.byref(d), C.byref(f))
        return d.value, f.value

    def apply_pre_ops(self, dem, k, ns):
        p = self._plan(k, ns, *dem.shape)
        out = np.empty((p.rows, p.cols), np.float32)
        self.lib.orc_apply_pre_ops(np.ascontiguousarray(dem), C.byref(p), out)
        return out

    def build_skw(self, g, shear_tan):
        rows, cols = g.shape
        base = base_offset(rows, cols, shear_tan)
        n = base + rows
        vals = np.zeros((n, cols), np.float32)
        w = np.zeros((n, cols), np.float32)
        rr = np.zeros((n, 2), np.int32)
        b = C.c_int()
        self._check(self.lib.orc_build_skw(np.ascontiguousarray(g), rows, cols, shear_tan, vals, w, rr, C.byref(b)))
        return vals, w, rr, b.value

    def linear_viewshed_row(self, row, first, last, j0, h, direction, max_dd=NO_CAP, want_visible=False):
        row = np.ascontiguousarray(row, np.float32)
        vis = np.zeros(max(1, len(row)), np.uint8)
        nv = C.c_int()
        cv = self.lib.orc_linear_viewshed_row(row, first, last, j0, h, direction, max_dd,
                                              vis.ctypes.data if want_visible else None, C.byref(nv))
        if want_visible:
            return cv, vis[: nv.value].copy()
        return cv

    def sector_viewshed(self, vals, ranges, src_rows, base, shear_tan, h0, max_dd=NO_CAP):
        skw_rows, cols = vals.shape
        out = np.zeros((skw_rows, cols), np.float64)
        self.lib.orc_sector_viewshed(np.ascontiguousarray(vals), np.ascontiguousarray(ranges, np.int32), skw_rows,
                                     cols, shear_tan, h0, max_dd, out)
        return out

    def unskew_accumulate(self, skw_vs, k, ns, dimy, dimx, out=None):
        p = self._plan(k, ns, dimy, dimx)
        if out is None:
            out = np.zeros((dimy, dimx), np.float64)
        self._check(self.lib.orc_unskew_accumulate(np.ascontiguousarray(skw_vs), skw_vs.shape[0], skw_vs.shape[1],
                                                   C.byref(p), out))
        return out

    def distance_cap_cells(self, max_distance, shear_tan, cellsize):
        return self.lib.orc_distance_cap_cells(max_distance or 0.0, shear_tan, cellsize)

    def sector_sweep(self, dem, cellsize, ns, h0, max_distance, k):
        out = np.zeros(dem.shape, np.float64)
        self._check(self.lib.orc_sector_sweep(np.ascontiguousarray(dem), dem.shape[0], dem.shape[1], cellsize, ns,
                                              h0, max_distance or 0.0, k, out))
        return out

    def total_viewshed(self, dem, cellsize, ns, h0, max_distance=0.0, units=0, raw=False, k_lo=0, k_hi=0):
        out = np.zeros(dem.shape, np.float64)
        self._check(self.lib.orc_total_viewshed(np.ascontiguousarray(dem), dem.shape[0], dem.shape[1], cellsize, ns,
                                                h0, max_distance or 0.0, units, int(raw), k_lo, k_hi, out))
        return out

    def area_scale_factor(self, ns, cellsize, units):
        return self.lib.orc_area_scale_factor(ns, cellsize, units)
