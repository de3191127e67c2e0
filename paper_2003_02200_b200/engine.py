"""Host-side mirror of the reference's public API (proj/include/skewshed/).

Names, argument meaning and error behaviour follow the reference so that
parity tests read like its own tests:

* ``make_synthetic``            dem.cpp:118-173 (+ Fractal)
* ``plan_sector``/``shear_params``  skew.cpp:23-101
* ``build_skw``                 skew.cpp:144-196 (GPU relocation kernel)
* ``sector_viewshed``           scan.cpp:64-85 (GPU scan + fixup kernels)
* ``linear_viewshed_row``       scan.cpp:8-62 (GPU scan, one POV)
* ``unskew_accumulate``         skew.cpp:204-263 (GPU unskew kernel)
* ``total_viewshed[_raw]``      engine.cpp:109-233 (whole GPU pipeline)
* ``sector_sweep``              engine.cpp:235-244
* ``area_scale_factor``         engine.cpp:103-107

``std::invalid_argument`` becomes ValueError and ``std::out_of_range``
IndexError. All compute goes through the native library (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import NO_CAP, check, lib

kNoDistanceCap = NO_CAP


class Units(enum.IntEnum):
    SquareMeters = 0
    SquareKilometers = 1


class SyntheticKind(enum.IntEnum):
    Flat = 0
    Ramp = 1
    Cone = 2
    SmoothedNoise = 3
    Fractal = 4  # diamond-square, not in the reference


class AxisOp(enum.IntEnum):
    Transpose = 0
    FlipCols = 1
    FlipRows = 2


class ScanDir(enum.IntEnum):
    Forward = 0
    Backward = 1


ALL_GPUS = -1  # RunConfig.n_gpus: every visible GPU


@dataclass
class RunConfig:
    """dem.hpp:40-46. The reference's ``workers`` (host threads sharing one
    call) becomes ``n_gpus`` (GPUs sharing one call: devices ``device`` ..
    ``device + n_gpus - 1``, or ALL_GPUS), one NCCL reduce of the maps."""
    ns: int = 360
    h0: float = 1.5
    max_distance: Optional[float] = None
    units: Units = Units.SquareKilometers
    device: int = 0
    n_gpus: int = 1

    def to_c(self) -> _lib.RunConfigC:
        md = 0.0 if self.max_distance is None else float(self.max_distance)
        if self.max_distance is not None and not md > 0.0:
            raise ValueError(f"invalid config: max distance must be a positive finite number, got {md}")
        return _lib.RunConfigC(int(self.ns), float(self.h0), md, int(self.units), int(self.device),
                               int(self.n_gpus))


@dataclass
class GridOrigin:
    """dem.hpp:13-17: lower-left corner of the grid (ESRI xll/yllcorner)."""
    easting: float = 0.0
    northing: float = 0.0


@dataclass
class Dem:
    """dem.hpp:26-37: float32 elevations, row 0 = north, col 0 = west."""
    values: np.ndarray
    cellsize: float = 1.0
    nodata: Optional[float] = None
    origin: GridOrigin = field(default_factory=GridOrigin)

    def __post_init__(self):
        self.values = np.ascontiguousarray(self.values, dtype=np.float32)

    def dimy(self) -> int:
        return int(self.values.shape[0])

    def dimx(self) -> int:
        return int(self.values.shape[1])


@dataclass
class VsGrid:
    values: np.ndarray
    units: Units = Units.SquareMeters


@dataclass
class SectorPlan:
    sector_index: int
    ns: int
    sector_deg: float
    shear_deg: float
    shear_tan: float
    pre_ops: list
    rows: int
    cols: int
    src_rows: int
    src_cols: int
    to_source: tuple  # (ii, ij, ci, ji, jj, cj)
    base: int
    skw_rows: int

    def source(self, i: int, j: int) -> tuple:
        ii, ij, ci, ji, jj, cj = self.to_source
        return ii * i + ij * j + ci, ji * i + jj * j + cj


@dataclass
class SkwGrid:
    values: np.ndarray            # (base+rows) x cols float32
    row_ranges: np.ndarray        # (skw_rows, 2) int32 [first, last)
    base: int
    src_rows: int
    shear_tan: float

    @property
    def cols(self) -> int:
        return int(self.values.shape[1])

    def skw_rows(self) -> int:
        return int(self.values.shape[0])


@dataclass
class EngineStats:
    skew_seconds: float = 0.0
    scan_seconds: float = 0.0
    fixup_seconds: float = 0.0
    unskew_seconds: float = 0.0
    reduce_seconds: float = 0.0
    total_seconds: float = 0.0
    sectors: int = 0
    batches: int = 0
    kernel_launches: int = 0
    target_evals: int = 0
    flagged_groups: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    skipped_target_slots: int = 0
    scan_kernel: int = 0  # 2: one row x 64 positions, 3: row pairs, 4: row quads

    @classmethod
    def from_c(cls, s: _lib.StatsC) -> "EngineStats":
        d = s.as_dict()
        d.pop("pad_", None)
        return cls(**d)


@dataclass
class SectorResult:
    sector_index: int
    contribution: np.ndarray


# ---- planning (host) ------------------------------------------------------

def plan_sector(k: int, ns: int, dimy: int, dimx: int) -> SectorPlan:
    p = _lib.SectorPlanC()
    check(lib.sks_plan_sector(k, ns, dimy, dimx, C.byref(p)))
    return SectorPlan(p.sector_index, p.ns, p.sector_deg, p.shear_deg, p.shear_tan,
                      [AxisOp(p.ops[i]) for i in range(p.n_ops)], p.rows, p.cols, p.src_rows,
                      p.src_cols, tuple(p.to_source), p.base, p.skw_rows)


def shear_params(shear_tan: float, j: int) -> tuple:
    d = C.c_int()
    f = C.c_double()
    lib.sks_shear_params(shear_tan, j, C.byref(d), C.byref(f))
    return d.value, f.value


def distance_cap_cells(max_distance: Optional[float], shear_tan: float, cellsize: float) -> int:
    return lib.sks_distance_cap_cells(0.0 if max_distance is None else max_distance, shear_tan, cellsize)


def area_scale_factor(cfg: RunConfig, cellsize: float) -> float:
    return lib.sks_area_scale_factor(cfg.ns, cellsize, int(cfg.units))


def area_scale(cv_sum: float, ns: int, cellsize: float) -> float:
    """scan.cpp:93-95."""
    return cv_sum * (np.pi / ns) * cellsize * cellsize


def row_ranges(rows: int, cols: int, shear_tan: float) -> np.ndarray:
    n = C.c_int()
    check(lib.sks_row_ranges(rows, cols, shear_tan, None, C.byref(n)))
    out = np.zeros((n.value, 2), np.int32)
    check(lib.sks_row_ranges(rows, cols, shear_tan, out.ctypes.data, C.byref(n)))
    return out


def sector_target_evals(k: int, ns: int, dimy: int, dimx: int, cellsize: float = 1.0,
                        max_distance: Optional[float] = None) -> int:
    return int(lib.sks_sector_target_evals(k, ns, dimy, dimx, cellsize, max_distance or 0.0))


def total_target_evals(ns: int, dimy: int, dimx: int, cellsize: float = 1.0,
                       max_distance: Optional[float] = None) -> int:
    return sum(sector_target_evals(k, ns, dimy, dimx, cellsize, max_distance) for k in range(ns // 2))


def partition_sectors(ns: int, dimy: int, dimx: int, world: int, cellsize: float = 1.0,
                      max_distance: Optional[float] = None) -> np.ndarray:
    owner = np.zeros(ns // 2, np.int32)
    check(lib.sks_partition_sectors(ns, dimy, dimx, cellsize, max_distance or 0.0, world, owner))
    return owner


def make_synthetic(kind: SyntheticKind, dimy: int, dimx: int, cellsize: float,
                   seed: int = 0) -> Dem:
    if not cellsize > 0.0:
        raise ValueError("synthetic cellsize must be positive")
    out = np.empty((dimy, dimx), np.float32) if dimy > 0 and dimx > 0 else np.empty((1, 1), np.float32)
    check(lib.sks_make_synthetic(int(kind), dimy, dimx, seed, out))
    return Dem(out, cellsize)


def validate(dem: Dem, cfg: RunConfig) -> None:
    nod = None
    if dem.nodata is not None:
        nod = C.byref(C.c_float(dem.nodata))
    c = cfg.to_c()
    check(lib.sks_validate(dem.values, dem.dimy(), dem.dimx(), dem.cellsize,
                           C.cast(nod, C.c_void_p) if nod is not None else None, C.byref(c)))


# ---- per-phase GPU entry points ------------------------------------------

def build_skw(g: np.ndarray, shear_tan: float, device: int = 0) -> SkwGrid:
    g = np.ascontiguousarray(g, np.float32)
    rows, cols = g.shape
    rr = row_ranges(rows, cols, shear_tan)
    vals = np.zeros((rr.shape[0], cols), np.float32)
    base = C.c_int()
    check(lib.sks_build_skw(g, rows, cols, shear_tan, device, vals, rr, C.byref(base)))
    return SkwGrid(vals, rr, base.value, rows, shear_tan)


def build_sector_sdem(dem: np.ndarray, k: int, ns: int, device: int = 0) -> SkwGrid:
    dem = np.ascontiguousarray(dem, np.float32)
    p = plan_sector(k, ns, *dem.shape)
    vals = np.zeros((p.skw_rows, p.cols), np.float32)
    rr = np.zeros((p.skw_rows, 2), np.int32)
    check(lib.sks_build_sector_sdem(dem, dem.shape[0], dem.shape[1], k, ns, device, vals, rr))
    return SkwGrid(vals, rr, p.base, p.rows, p.shear_tan)


def sector_viewshed(skw: SkwGrid, h0: float, max_dd: int = NO_CAP, device: int = 0,
                    return_cv: bool = False):
    vals = np.ascontiguousarray(skw.values, np.float32)
    rr = np.ascontiguousarray(skw.row_ranges, np.int32)
    out = np.zeros(vals.shape, np.float64)
    cvf = np.zeros(vals.shape, np.int32)
    cvb = np.zeros(vals.shape, np.int32)
    check(lib.sks_sector_viewshed(vals, rr, vals.shape[0], vals.shape[1], skw.shear_tan, h0, max_dd,
                                  device, out, cvf.ctypes.data, cvb.ctypes.data))
    if return_cv:
        return out, cvf, cvb
    return out


def linear_viewshed_row(row, first: int, last: int, j0: int, h: float, direction: ScanDir,
                        max_dd: int = NO_CAP, want_visible: bool = False, device: int = 0):
    row = np.ascontiguousarray(row, np.float32)
    cv = C.c_double()
    nv = C.c_int()
    vis = np.zeros(max(1, len(row)), np.uint8)
    check(lib.sks_linear_viewshed_row(row, len(row), first, last, j0, h, int(direction), max_dd, device,
                                      C.byref(cv), vis.ctypes.data if want_visible else None,
                                      C.byref(nv)))
    if want_visible:
        return cv.value, vis[: nv.value].copy()
    return cv.value


def unskew_accumulate(skw_vs: np.ndarray, plan: SectorPlan, out: np.ndarray, device: int = 0) -> None:
    if out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array")
    if out.shape != (plan.src_rows, plan.src_cols):
        raise ValueError(f"output shape {out.shape[0]}x{out.shape[1]} does not match source grid "
                         f"{plan.src_rows}x{plan.src_cols}")
    vs = np.ascontiguousarray(skw_vs, np.float64)
    check(lib.sks_unskew_accumulate(vs, vs.shape[0], vs.shape[1], plan.sector_index, plan.ns,
                                    plan.src_rows, plan.src_cols, device, out))


# ---- end to end ------------------------------------------------------------

def _total(dem: Dem, cfg: RunConfig, raw: bool, stats: Optional[EngineStats]):
    out = np.empty((dem.dimy(), dem.dimx()), np.float64)
    c = cfg.to_c()
    st = _lib.StatsC()
    fn = lib.sks_total_viewshed_raw if raw else lib.sks_total_viewshed
    check(fn(dem.values.ctypes.data, dem.dimy(), dem.dimx(), dem.cellsize, C.byref(c),
             out.ctypes.data, C.byref(st)))
    if stats is not None:
        for k, v in st.as_dict().items():
            setattr(stats, k, v)
    return out


def _require_no_nodata(dem: Dem, cfg: RunConfig) -> None:
    if dem.nodata is not None:
        validate(dem, cfg)


def _report_progress(dem: Dem, cfg: RunConfig, st: "EngineStats", progress) -> None:
    """ProgressFn (engine.hpp:34-36): once per sector, ascending k, on the
    calling thread. Sectors run batched on the GPU, so each gets the batch
    phases' device time attributed by its exact scan work."""
    busy = st.skew_seconds + st.scan_seconds + st.fixup_seconds + st.unskew_seconds
    work = [sector_target_evals(k, cfg.ns, dem.dimy(), dem.dimx(), dem.cellsize, cfg.max_distance)
            for k in range(cfg.ns // 2)]
    total = float(sum(work)) or 1.0
    for k, w in enumerate(work):
        progress(k, busy * w / total)


def total_viewshed_raw(dem: Dem, cfg: RunConfig, stats: Optional[EngineStats] = None,
                       progress=None) -> np.ndarray:
    _require_no_nodata(dem, cfg)
    st = stats if stats is not None else (EngineStats() if progress is not None else None)
    out = _total(dem, cfg, True, st)
    if progress is not None:
        _report_progress(dem, cfg, st, progress)
    return out


def total_viewshed(dem: Dem, cfg: RunConfig, stats: Optional[EngineStats] = None,
                   progress=None) -> VsGrid:
    _require_no_nodata(dem, cfg)
    st = stats if stats is not None else (EngineStats() if progress is not None else None)
    out = _total(dem, cfg, False, st)
    if progress is not None:
        _report_progress(dem, cfg, st, progress)
    return VsGrid(out, Units(cfg.units))


def total_viewshed_devices(dem: Dem, cfg: RunConfig, devices, raw: bool = False,
                           stats: Optional[EngineStats] = None) -> np.ndarray:
    """One total viewshed shared by the listed GPUs in this process (one host
    thread per GPU, one NCCL reduce; repeated devices reduce by peer adds).
    Returns the raw map if ``raw``, else the scaled areas."""
    _require_no_nodata(dem, cfg)
    devs = np.ascontiguousarray(devices, np.int32)
    out = np.empty((dem.dimy(), dem.dimx()), np.float64)
    c = cfg.to_c()
    st = _lib.StatsC()
    check(lib.sks_total_viewshed_devices(dem.values.ctypes.data, dem.dimy(), dem.dimx(), dem.cellsize, C.byref(c),
                                         devs.ctypes.data, len(devs), int(raw), out.ctypes.data, C.byref(st)))
    if stats is not None:
        for k, v in st.as_dict().items():
            setattr(stats, k, v)
    return out


def config_devices(cfg: RunConfig) -> list:
    """The GPUs a run config names (device, n_gpus)."""
    c = cfg.to_c()
    buf = np.zeros(256, np.int32)
    n = int(lib.sks_config_devices(C.byref(c), buf.ctypes.data, len(buf)))
    return buf[:min(n, len(buf))].tolist()


def row_cuts_update(cuts, times) -> np.ndarray:
    """One measured-time rebalancing step of the row-block cuts (C++,
    sks_row_cuts_update; distributed.RowBalancer wraps it)."""
    c = np.ascontiguousarray(cuts, np.float64)
    t = np.ascontiguousarray(times, np.float64)
    if c.shape != (len(t) + 1,):
        raise ValueError("cuts must hold len(times) + 1 fractions")
    out = np.empty_like(c)
    lib.sks_row_cuts_update(c.ctypes.data, t.ctypes.data, len(t), out.ctypes.data)
    return out


def sector_sweep(dem: Dem, cfg: RunConfig, k: int) -> SectorResult:
    _require_no_nodata(dem, cfg)
    out = np.empty((dem.dimy(), dem.dimx()), np.float64)
    c = cfg.to_c()
    check(lib.sks_sector_sweep(dem.values, dem.dimy(), dem.dimx(), dem.cellsize, C.byref(c), k, out))
    return SectorResult(k, out)


def accumulate_into(accum: np.ndarray, contribution: np.ndarray) -> None:
    """engine.cpp:85-92."""
    if accum.shape != contribution.shape:
        raise ValueError("cannot accumulate grids of different shape")
    accum += contribution


def reduce_ordered(buffers) -> np.ndarray:
    """engine.cpp:94-101."""
    if len(buffers) == 0:
        raise ValueError("nothing to reduce")
    acc = np.zeros_like(buffers[0], dtype=np.float64)
    for b in buffers:
        accumulate_into(acc, b)
    return acc


def convert_units(grid: VsGrid, target: Units) -> VsGrid:
    """dem.cpp:24-34."""
    if grid.units == target:
        return grid
    f = 1e-6 if target == Units.SquareKilometers else 1e6
    return VsGrid(grid.values * f, target)


# ---- device-resident context ----------------------------------------------

class Context:
    """One GPU's engine context (sks_context). Works on device pointers so a
    caller (e.g. torch) owns device memory, streams and collectives."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.sks_context_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if self._h:
            lib.sks_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run_sectors(self, d_dem: int, dimy: int, dimx: int, cellsize: float, cfg: RunConfig,
                    sectors, d_map: int, stream: int = 0, want_stats: bool = False):
        ks = np.ascontiguousarray(np.asarray(sectors, dtype=np.int32))
        c = cfg.to_c()
        st = _lib.StatsC()
        check(lib.sks_context_run_sectors(self._h, d_dem, dimy, dimx, cellsize, C.byref(c), ks, len(ks),
                                          d_map, stream, C.byref(st) if want_stats else None))
        return EngineStats.from_c(st) if want_stats else None

    def run_rows(self, d_dem: int, dimy: int, dimx: int, cellsize: float, cfg: RunConfig, part: int,
                 nparts: int, d_map: int, stream: int = 0, want_stats: bool = False, cuts=None):
        """All sectors, row block `part` of `nparts` of every sector (row-block
        sharding across GPUs; the nparts maps sum to the total raw map).
        ``cuts`` (nparts + 1 non-decreasing fractions of the modelled cost,
        identical on every rank) places the blocks; None = equal shares."""
        c = cfg.to_c()
        st = _lib.StatsC()
        cp = None
        if cuts is not None:
            cuts_arr = np.ascontiguousarray(cuts, np.float64)
            if cuts_arr.shape != (nparts + 1,):
                raise ValueError(f"cuts must hold nparts + 1 = {nparts + 1} fractions")
            cp = cuts_arr.ctypes.data
        check(lib.sks_context_run_rows_cuts(self._h, d_dem, dimy, dimx, cellsize, C.byref(c), part, nparts, cp,
                                            d_map, stream, C.byref(st) if want_stats else None))
        return EngineStats.from_c(st) if want_stats else None

    def scale(self, d_map: int, n: int, ns: int, cellsize: float, units: int, stream: int = 0):
        check(lib.sks_context_scale(self._h, d_map, n, ns, cellsize, units, stream))

    def total_viewshed(self, dem_host: np.ndarray, cellsize: float, cfg: RunConfig, raw: bool = False,
                       out: Optional[np.ndarray] = None, want_stats: bool = False):
        """Host buffers in, host map out (H2D + D2H inside). dem_host / out may
        be pinned numpy views (torch pin_memory) for full-speed copies."""
        dem_host = np.ascontiguousarray(dem_host, np.float32)
        if out is None:
            out = np.empty(dem_host.shape, np.float64)
        c = cfg.to_c()
        st = _lib.StatsC()
        check(lib.sks_context_total_viewshed(self._h, dem_host.ctypes.data, dem_host.shape[0],
                                             dem_host.shape[1], cellsize, C.byref(c), int(raw),
                                             out.ctypes.data, C.byref(st)))
        if want_stats:
            return out, EngineStats.from_c(st)
        return out


def device_count() -> int:
    return int(lib.sks_device_count())


def scan_row_limit() -> int:
    """Longest skewed row the shared-memory scan holds (longer rows run POV by
    POV through the exact kernel)."""
    return int(lib.sks_scan_row_limit())


# ---- ESRI ASCII grid I/O (ascii_grid.hpp:15-31) ----------------------------

GridFormatError = _lib.GridFormatError


def _grid_from_handle(h) -> Dem:
    try:
        hdr = _lib.GridHeaderC()
        check(lib.sks_ascii_grid_header(h, C.byref(hdr)))
        vals = np.empty((hdr.nrows, hdr.ncols), np.float32)
        check(lib.sks_ascii_grid_values(h, vals.ctypes.data))
    finally:
        lib.sks_ascii_grid_free(h)
    return Dem(vals, hdr.cellsize, float(hdr.nodata) if hdr.has_nodata else None,
               GridOrigin(hdr.xllcorner, hdr.yllcorner))


def read_ascii_grid(path) -> Dem:
    """read_ascii_grid(path) (ascii_grid.cpp:198-204); GridFormatError on bad input."""
    h = C.c_void_p()
    check(lib.sks_ascii_grid_read(str(path).encode(), C.byref(h)))
    return _grid_from_handle(h)


def parse_ascii_grid(text, source_name: str = "<input>") -> Dem:
    """read_ascii_grid(istream, source_name) (ascii_grid.cpp:110-196) on text/bytes."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    check(lib.sks_ascii_grid_parse(data, len(data), source_name.encode(), C.byref(h)))
    return _grid_from_handle(h)


def read_float_grid(path) -> Dem:
    """Binary side format (ESRI .hdr + .flt float32): the fast DEM load for
    large grids. GridFormatError on a bad header or file size."""
    h = C.c_void_p()
    check(lib.sks_float_grid_read(str(path).encode(), C.byref(h)))
    return _grid_from_handle(h)


def write_float_grid(dem: Dem, path) -> None:
    """Writes dem as <base>.hdr + <base>.flt (LSBFIRST)."""
    hdr = _lib.GridHeaderC(dem.dimy(), dem.dimx(), dem.origin.easting, dem.origin.northing, dem.cellsize,
                           1 if dem.nodata is not None else 0, float(dem.nodata) if dem.nodata is not None else 0.0)
    check(lib.sks_write_float_grid(str(path).encode(), dem.values.ctypes.data, C.byref(hdr)))


def write_ascii_grid(grid, path, units: Optional["Units"] = None, cellsize: Optional[float] = None,
                     origin: Optional[GridOrigin] = None) -> None:
    """write_ascii_grid for a Dem (ascii_grid.cpp:225-245) or a VsGrid in
    `units` with the source DEM's cellsize and origin (:247-272)."""
    if isinstance(grid, Dem):
        hdr = _lib.GridHeaderC(grid.dimy(), grid.dimx(), grid.origin.easting, grid.origin.northing,
                               grid.cellsize, 1 if grid.nodata is not None else 0,
                               float(grid.nodata) if grid.nodata is not None else 0.0)
        check(lib.sks_write_ascii_grid_dem(str(path).encode(), grid.values.ctypes.data, C.byref(hdr)))
        return
    vals = np.ascontiguousarray(grid.values, np.float64)
    o = origin or GridOrigin()
    out_units = grid.units if units is None else units
    check(lib.sks_write_ascii_grid_vs(str(path).encode(), vals.ctypes.data, vals.shape[0], vals.shape[1],
                                      int(grid.units), int(out_units), float(cellsize if cellsize else 1.0),
                                      o.easting, o.northing))


class Palette(enum.IntEnum):
    """heatmap.hpp:9"""
    Gray = 0
    BlueRed = 1


def write_heatmap(grid: VsGrid, path, palette: Palette = Palette.Gray) -> None:
    """write_heatmap (heatmap.cpp:11-56): binary PGM (Gray) or PPM (BlueRed)
    of the min-max normalised map."""
    vals = np.ascontiguousarray(grid.values if isinstance(grid, VsGrid) else grid, np.float64)
    rows, cols = (vals.shape + (0, 0))[:2] if vals.ndim == 2 else (0, 0)
    check(lib.sks_write_heatmap(str(path).encode(), vals.ctypes.data, rows, cols, int(palette)))


def fill_nodata_nearest(dem: Dem) -> Dem:
    """fill_nodata_nearest (dem.cpp:175-213): nodata cells take the value the
    reference's breadth-first search reaches them from; nodata is cleared."""
    if dem.nodata is None:
        return Dem(dem.values.copy(), dem.cellsize, None, dem.origin)
    out = np.empty_like(dem.values)
    check(lib.sks_fill_nodata_nearest(dem.values.ctypes.data, dem.dimy(), dem.dimx(), float(dem.nodata),
                                      out.ctypes.data))
    return Dem(out, dem.cellsize, None, dem.origin)


@dataclass
class BenchReport:
    """bench.hpp:14-28. scan_seconds here is the whole scan phase on the GPU
    (scan + exact fixup kernels); workers is the number of GPUs."""
    dataset: str = ""
    dimy: int = 0
    dimx: int = 0
    ns: int = 0
    workers: int = 0
    skew_seconds: float = 0.0
    scan_seconds: float = 0.0
    unskew_seconds: float = 0.0
    reduce_seconds: float = 0.0
    total_seconds: float = 0.0
    povs_per_second: float = 0.0
    speedup: float = 0.0


def make_bench_report(dataset: str, dimy: int, dimx: int, cfg: RunConfig, stats: EngineStats,
                      baseline_total_seconds: float = 0.0, workers: int = 1) -> BenchReport:
    """make_bench_report (bench.cpp:8-28): one observer scan per cell per
    sector over the scan-phase seconds; speedup against a baseline total."""
    scan = stats.scan_seconds + stats.fixup_seconds
    r = BenchReport(dataset, dimy, dimx, cfg.ns, workers, stats.skew_seconds, scan, stats.unskew_seconds,
                    stats.reduce_seconds, stats.total_seconds)
    r.povs_per_second = float(dimy) * float(dimx) * float(cfg.ns // 2) / scan if scan > 0 else float("inf")
    if baseline_total_seconds > 0.0:
        # C++ double division (bench.cpp:25): a zero total gives inf, not an exception
        r.speedup = baseline_total_seconds / r.total_seconds if r.total_seconds != 0.0 else float("inf")
    return r


def format_bench_report(r: BenchReport) -> str:
    """format_bench_report (bench.cpp:30-52): stable key: value lines."""
    num = lambda v: "%.17g" % v  # noqa: E731
    lines = [f"dataset: {r.dataset}", f"dimy: {r.dimy}", f"dimx: {r.dimx}", f"ns: {r.ns}", f"workers: {r.workers}",
             f"skew_seconds: {num(r.skew_seconds)}", f"scan_seconds: {num(r.scan_seconds)}",
             f"unskew_seconds: {num(r.unskew_seconds)}", f"reduce_seconds: {num(r.reduce_seconds)}",
             f"total_seconds: {num(r.total_seconds)}", f"povs_per_second: {num(r.povs_per_second)}"]
    if r.speedup > 0.0:
        lines.append(f"speedup: {num(r.speedup)}")
    return "\n".join(lines) + "\n"
