"""Multi-GPU total viewshed with one reduce of the viewshed maps.

Replaces the reference's single-process sector pool (engine.cpp:115-176) and
the paper's host-side multi-GPU reduction (Alg. 10): one process per
GPU (torch.distributed, NCCL over NVLink), each rank accumulating its share
into a private FP64 map on its GPU, then a single ``reduce(SUM)`` of the maps
to rank 0. That reduce is the path's only exchange step; the DEM itself is
copied host->device on every rank (it is the caller's input).

Two ways to share the work:

* ``mode="rows"`` (default): every rank runs all sectors but only its block
  of every sector's skewed rows (contiguous blocks of equal exact scan work,
  ``sks_context_run_rows``). Measured per-sector costs at 2000^2 vary 4x
  and correlate weakly with the exact work model (the hidden-window skip
  depends on terrain and angle), so whole-sector assignment balances poorly
  (LPT on the work model: 68% at 8 GPUs); a block of every sector averages
  the terrain out (SURVEY §8e's sub-sector work items).
* ``mode="sectors"``: whole sectors by LPT on the exact work
  (``sks_partition_sectors``), the paper's scheme.

``RowBalancer`` moves the row-block boundaries from measured per-rank times
(bench.py adapts during its warm-up steps and then freezes them).

``compute`` lets CPU tests (gloo, world_size 2) exercise exactly this
sharding/reduce logic with the oracle standing in for the GPU pipeline; the
product path (compute=None) always runs the CUDA kernels.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np

from .engine import RunConfig, Units, area_scale_factor, partition_sectors, row_cuts_update


class RowBalancer:
    """Measured-time rebalancing of the row blocks across ranks.

    The static split gives every rank an equal share of each sector's
    MODELLED row cost (sks_plan.cpp set_row_block); terrain makes the real
    cost per share differ by ~10 % between blocks at 8 GPUs. After a run with
    cuts c and per-rank times t, the time is modelled as piecewise linear in
    the cost fraction (density t_r / (c[r+1] - c[r]) on block r) and the new
    cuts put an equal share of the total time in every block. Every rank
    feeds the same all-gathered times, so every rank computes the same cuts
    (deterministic float64 arithmetic).
    """

    def __init__(self, world: int):
        self.world = int(world)
        self.cuts = np.linspace(0.0, 1.0, self.world + 1)

    def update(self, times: Sequence[float]) -> np.ndarray:
        t = np.asarray(times, np.float64)
        if t.shape != (self.world,):
            return self.cuts
        # the same step the in-process multi-GPU path takes (sks_row_cuts_update)
        self.cuts = row_cuts_update(self.cuts, t)
        return self.cuts


def my_sectors(ns: int, dimy: int, dimx: int, world: int, rank: int, cellsize: float = 1.0,
               max_distance: Optional[float] = None) -> list:
    owner = partition_sectors(ns, dimy, dimx, world, cellsize, max_distance)
    return [k for k in range(ns // 2) if int(owner[k]) == rank]


def total_viewshed_distributed(dem: np.ndarray, cellsize: float, cfg: RunConfig, raw: bool = False,
                               compute: Optional[Callable[[Sequence[int]], np.ndarray]] = None,
                               context=None, stream=None, stats: Optional[dict] = None, mode: str = "rows",
                               cuts=None):
    """Total viewshed of ``dem`` sharded over the default process group.

    Returns the (scaled unless ``raw``) map on rank 0 and None elsewhere.
    ``compute`` (CPU tests) replaces the GPU pipeline for sector sharding.
    """
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    dimy, dimx = dem.shape
    mine = my_sectors(cfg.ns, dimy, dimx, world, rank, cellsize, cfg.max_distance)
    factor = area_scale_factor(cfg, cellsize)
    if compute is not None:
        part = torch.from_numpy(np.ascontiguousarray(compute(mine), dtype=np.float64))
        dist.reduce(part, dst=0, op=dist.ReduceOp.SUM)
        if rank != 0:
            return None
        out = part.numpy()
        return out if raw else out * factor

    from .engine import Context
    dev = torch.device("cuda", torch.cuda.current_device())
    ctx = context or Context(dev.index)
    st = stream or torch.cuda.current_stream(dev)
    # everything below is ordered on `st`: the DEM copy and the map clear
    # before the engine's kernels, the kernels before the reduce and the D2H
    with torch.cuda.stream(st):
        d_dem = torch.from_numpy(np.ascontiguousarray(dem, np.float32)).to(dev, non_blocking=True)
        d_map = torch.zeros((dimy, dimx), dtype=torch.float64, device=dev)
        if mode == "rows":
            es = ctx.run_rows(d_dem.data_ptr(), dimy, dimx, cellsize, cfg, rank, world, d_map.data_ptr(),
                              stream=st.cuda_stream, want_stats=stats is not None, cuts=cuts)
        else:
            es = ctx.run_sectors(d_dem.data_ptr(), dimy, dimx, cellsize, cfg, mine, d_map.data_ptr(),
                                 stream=st.cuda_stream, want_stats=stats is not None)
        if stats is not None:
            stats["rank_stats"] = es
            stats["sectors"] = mine if mode != "rows" else f"rows {rank}/{world} of every sector"
        dist.reduce(d_map, dst=0, op=dist.ReduceOp.SUM)
        if rank != 0:
            return None
        if not raw:
            ctx.scale(d_map.data_ptr(), dimy * dimx, cfg.ns, cellsize, int(cfg.units), st.cuda_stream)
        return d_map.cpu().numpy()
