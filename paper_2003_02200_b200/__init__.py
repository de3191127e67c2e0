"""skewshed-b200: B200-native sDEM total viewshed (arXiv 2003.02200).

The hot path (relocation -> line-of-sight scan -> unskew/accumulate) runs in
hand-written sm_100a kernels inside libskewshed_b200.so, reached through its C
ABI (include/skewshed_b200.h). This package is the host-side mirror of the
reference's C++ API (proj/include/skewshed/*.hpp) plus the multi-GPU sharding.
"""
from .engine import (ALL_GPUS, config_devices, row_cuts_update, total_viewshed_devices, AxisOp, BenchReport, Palette, fill_nodata_nearest, format_bench_report, make_bench_report, read_float_grid, write_float_grid, write_heatmap, Context, Dem, EngineStats, GridFormatError, GridOrigin, parse_ascii_grid,
                     read_ascii_grid, write_ascii_grid, RunConfig, ScanDir, SectorPlan, SectorResult,
                     SkwGrid, SyntheticKind, Units, VsGrid, accumulate_into, area_scale, area_scale_factor,
                     build_sector_sdem, build_skw, convert_units, device_count, distance_cap_cells,
                     kNoDistanceCap, linear_viewshed_row, make_synthetic, partition_sectors, plan_sector,
                     reduce_ordered, row_ranges, scan_row_limit, sector_sweep, sector_target_evals, sector_viewshed,
                     shear_params, total_target_evals, total_viewshed, total_viewshed_raw,
                     unskew_accumulate, validate)
from . import sweep  # noqa: E402  (rotational-sweep oracle API, oracle.hpp)

__all__ = [
    "ALL_GPUS", "config_devices", "row_cuts_update", "total_viewshed_devices", "AxisOp", "BenchReport", "Palette", "fill_nodata_nearest", "format_bench_report", "make_bench_report", "read_float_grid", "write_float_grid", "write_heatmap", "sweep", "Context", "Dem", "EngineStats", "GridFormatError", "GridOrigin", "parse_ascii_grid",
    "read_ascii_grid", "write_ascii_grid", "RunConfig", "ScanDir", "SectorPlan", "SectorResult",
    "SkwGrid", "SyntheticKind", "Units", "VsGrid", "accumulate_into", "area_scale", "area_scale_factor",
    "build_sector_sdem", "build_skw", "convert_units", "device_count", "distance_cap_cells",
    "kNoDistanceCap", "linear_viewshed_row", "make_synthetic", "partition_sectors", "plan_sector",
    "reduce_ordered", "row_ranges", "scan_row_limit", "sector_sweep", "sector_target_evals", "sector_viewshed",
    "shear_params", "total_target_evals", "total_viewshed", "total_viewshed_raw", "unskew_accumulate",
    "validate",
]
