"""ctypes binding of the in-tree native library (libskewshed_b200.so).

The library is the product: every compute entry point below runs the sm_100a
kernels. There is no Python or CPU fallback — if the .so is missing this
module raises ImportError, and compute calls on a host without a GPU raise
RuntimeError from the CUDA runtime.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SKS_LIB selects a variant build of the same library (kernel experiments,
# paper_2003_02200_b200/build.py -D ... --out ...); default: the in-tree build.
LIB_PATH = os.environ.get("SKS_LIB") or os.path.join(HERE, "libskewshed_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or python paper_2003_02200_b200/build.py)")

lib = C.CDLL(LIB_PATH)

SKS_OK = 0
SKS_INVALID_ARGUMENT = 1
SKS_OUT_OF_RANGE = 2
SKS_CUDA_ERROR = 3
SKS_NCCL_ERROR = 4
SKS_INTERNAL = 5
SKS_FORMAT_ERROR = 6
NO_CAP = 2147483647


class RunConfigC(C.Structure):
    _fields_ = [("ns", C.c_int), ("h0", C.c_double), ("max_distance", C.c_double),
                ("units", C.c_int), ("device", C.c_int), ("n_gpus", C.c_int)]


class StatsC(C.Structure):
    _fields_ = [("skew_seconds", C.c_double), ("scan_seconds", C.c_double),
                ("fixup_seconds", C.c_double), ("unskew_seconds", C.c_double),
                ("reduce_seconds", C.c_double), ("total_seconds", C.c_double),
                ("sectors", C.c_int), ("batches", C.c_int),
                ("kernel_launches", C.c_longlong), ("target_evals", C.c_longlong),
                ("flagged_groups", C.c_longlong), ("h2d_bytes", C.c_longlong),
                ("d2h_bytes", C.c_longlong), ("skipped_target_slots", C.c_longlong),
                ("scan_kernel", C.c_int), ("pad_", C.c_int)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class SectorPlanC(C.Structure):
    _fields_ = [("sector_index", C.c_int), ("ns", C.c_int), ("sector_deg", C.c_double),
                ("shear_deg", C.c_double), ("shear_tan", C.c_double), ("n_ops", C.c_int),
                ("ops", C.c_int * 3), ("rows", C.c_int), ("cols", C.c_int),
                ("src_rows", C.c_int), ("src_cols", C.c_int), ("to_source", C.c_int * 6),
                ("base", C.c_int), ("skw_rows", C.c_int)]


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)

# Every symbol declared in include/skewshed_b200.h, with its signature.
class GridHeaderC(C.Structure):
    _fields_ = [("nrows", C.c_int), ("ncols", C.c_int), ("xllcorner", C.c_double), ("yllcorner", C.c_double),
                ("cellsize", C.c_double), ("has_nodata", C.c_int), ("nodata", C.c_float)]


SIGNATURES = {
    "sks_last_error": (C.c_char_p, []),
    "sks_version": (C.c_char_p, []),
    "sks_device_count": (C.c_int, []),
    "sks_scan_row_limit": (C.c_int, []),
    "sks_plan_sector": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(SectorPlanC)]),
    "sks_shear_params": (None, [C.c_double, C.c_int, _ip, _dp]),
    "sks_distance_cap_cells": (C.c_int, [C.c_double, C.c_double, C.c_double]),
    "sks_area_scale_factor": (C.c_double, [C.c_int, C.c_double, C.c_int]),
    "sks_row_ranges": (C.c_int, [C.c_int, C.c_int, C.c_double, _vp, _ip]),
    "sks_sector_target_evals": (C.c_longlong, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double]),
    "sks_partition_sectors": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _i32p]),
    "sks_make_synthetic": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint32, _f32p]),
    "sks_validate": (C.c_int, [_f32p, C.c_int, C.c_int, C.c_double, _vp, C.POINTER(RunConfigC)]),
    "sks_total_viewshed": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, C.POINTER(RunConfigC), _vp,
                                     C.POINTER(StatsC)]),
    "sks_total_viewshed_raw": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, C.POINTER(RunConfigC), _vp,
                                         C.POINTER(StatsC)]),
    "sks_total_viewshed_devices": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, C.POINTER(RunConfigC), _vp, C.c_int,
                                             C.c_int, _vp, C.POINTER(StatsC)]),
    "sks_config_devices": (C.c_int, [C.POINTER(RunConfigC), _vp, C.c_int]),
    "sks_row_cuts_update": (None, [_vp, _vp, C.c_int, _vp]),
    "sks_sector_sweep": (C.c_int, [_f32p, C.c_int, C.c_int, C.c_double, C.POINTER(RunConfigC), C.c_int,
                                   _f64p]),
    "sks_build_sector_sdem": (C.c_int, [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f32p, _i32p]),
    "sks_build_skw": (C.c_int, [_f32p, C.c_int, C.c_int, C.c_double, C.c_int, _f32p, _i32p, _ip]),
    "sks_sector_viewshed": (C.c_int, [_f32p, _i32p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                      C.c_int, _f64p, _vp, _vp]),
    "sks_linear_viewshed_row": (C.c_int, [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                          C.c_int, C.c_int, _dp, _vp, _ip]),
    "sks_unskew_accumulate": (C.c_int, [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, _f64p]),
    "sks_context_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "sks_context_destroy": (None, [_vp]),
    "sks_context_run_sectors": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_double, C.POINTER(RunConfigC),
                                          _i32p, C.c_int, _vp, _vp, C.POINTER(StatsC)]),
    "sks_ascii_grid_read": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "sks_ascii_grid_parse": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.POINTER(_vp)]),
    "sks_ascii_grid_header": (C.c_int, [_vp, C.POINTER(GridHeaderC)]),
    "sks_ascii_grid_values": (C.c_int, [_vp, _vp]),
    "sks_ascii_grid_free": (None, [_vp]),
    "sks_float_grid_read": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "sks_write_float_grid": (C.c_int, [C.c_char_p, _vp, C.POINTER(GridHeaderC)]),
    "sks_write_ascii_grid_dem": (C.c_int, [C.c_char_p, _vp, C.POINTER(GridHeaderC)]),
    "sks_write_ascii_grid_vs": (C.c_int, [C.c_char_p, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                          C.c_double, C.c_double]),
    "sks_context_run_rows": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_double, C.POINTER(RunConfigC),
                                       C.c_int, C.c_int, _vp, _vp, C.POINTER(StatsC)]),
    "sks_context_run_rows_cuts": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_double, C.POINTER(RunConfigC),
                                            C.c_int, C.c_int, _vp, _vp, _vp, C.POINTER(StatsC)]),
    "sks_singular_viewshed": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                        C.c_int, C.c_double, C.c_int, _vp]),
    "sks_multi_viewshed": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, _vp, C.c_int, C.c_double, C.c_int,
                                     C.c_double, C.c_int, _vp, _vp, _vp]),
    "sks_total_viewshed_reference": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, _vp, C.POINTER(RunConfigC),
                                               C.c_int, _vp]),
    "sks_linear_scan": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                  C.c_int, _vp, _vp, C.c_int, _vp]),
    "sks_axis_point_set": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _vp, C.c_int, _vp]),
    "sks_random_povs": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint32, _vp]),
    "sks_fill_nodata_nearest": (C.c_int, [_vp, C.c_int, C.c_int, C.c_float, _vp]),
    "sks_write_heatmap": (C.c_int, [C.c_char_p, _vp, C.c_int, C.c_int, C.c_int]),
    "sks_context_scale": (C.c_int, [_vp, _vp, C.c_longlong, C.c_int, C.c_double, C.c_int, _vp]),
    "sks_context_total_viewshed": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_double,
                                             C.POINTER(RunConfigC), C.c_int, _vp, C.POINTER(StatsC)]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    return lib.sks_last_error().decode()


class GridFormatError(RuntimeError):
    """ascii_grid.hpp:15-18: malformed grid text (message carries source:line:col)."""


def check(status: int) -> None:
    """Maps sks_status to the reference's exception types."""
    if status == SKS_OK:
        return
    msg = last_error()
    if status == SKS_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == SKS_OUT_OF_RANGE:
        raise IndexError(msg)
    if status == SKS_FORMAT_ERROR:
        raise GridFormatError(msg)
    raise RuntimeError(msg)


def header_symbols(header: str | None = None) -> list[str]:
    """Names of the functions include/skewshed_b200.h declares."""
    import re
    header = header or os.path.join(os.path.dirname(HERE), "include", "skewshed_b200.h")
    text = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(sks_\w+)\s*\(", text, re.M)))
