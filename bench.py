#!/usr/bin/env python
"""Benchmark: sDEM total viewshed, POV-sector evaluations per second.

Workload (BASELINE.json configs[1], "config 2"): synthetic 2000x2000 fractal
DEM at 10 m (seed 7), 180 sectors, observer height 1.5 m, unlimited radius.
A step is one full total viewshed: relocation + scan + fixup + unskew of all
90 sector axes (N > 1: every rank runs its block of every sector's skewed
rows, cuts rebalanced from measured times during warm-up) + the reduce of the
maps to rank 0 + area scaling, with the DEM resident in HBM. The warm-up
steps also cover the engine's scan-kernel autotune.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 1..5] [--terrain fractal|smooth]

One JSON line on rank 0. See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(n=500, ns=180, max_distance=None),
    2: dict(n=2000, ns=180, max_distance=None),
    3: dict(n=2000, ns=360, max_distance=10000.0),
    4: dict(n=4000, ns=180, max_distance=None),
    5: dict(n=10000, ns=180, max_distance=None),
}
METRIC = "POV-sector evals/sec & total-viewshed time (2000² DEM, 180 sectors) @1/2/4/8 GPU"
UNIT = "POV-sector/s"
CELLSIZE = 10.0
H0 = 1.5
SEED = 7


def workload_name(cfgid, terrain):
    c = CONFIGS[cfgid]
    cap = "unlimited radius" if c["max_distance"] is None else f"max radius {c['max_distance'] / 1000:g} km"
    return (f"config {cfgid}: synthetic {c['n']}x{c['n']} {terrain} DEM at 10 m (seed {SEED}), "
            f"{c['ns']} sectors, observer height 1.5 m, {cap}")


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return p, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    every 20 ms from a thread (nvidia_ml_py; one sample is also taken when
    the thread starts, so even a ~1 s region has samples), else nvidia-smi
    -lms 100 (whose own start-up can outlast a short region)."""

    # NVML clocks-event reason bits (nvml.h)
    _BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _nvml_sample(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except AttributeError:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        try:
            pw = nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0
        except Exception:
            pw = float("nan")
        flags = ["Active" if bits & b else "Not Active" for b in self._BITS.values()]
        self.samples.append([str(sm), str(self._max), str(pw), hex(bits), *flags])

    def _nvml_loop(self):
        while True:
            try:
                self._nvml_sample()
            except Exception:
                return
            if self._stop.wait(0.02):
                return

    def start(self):
        if self._nvml is not None:
            self._t = threading.Thread(target=self._nvml_loop, daemon=True)
            self._t.start()
            return
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self._proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=2)
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for name, v in zip(names, s[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        loaded = sorted(sm)[len(sm) // 4:] if sm else []
        med = float(np.median(loaded)) if loaded else None
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def dist_setup(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # one GPU per rank; ranks beyond the visible GPUs share them (only
        # for exercising the multi-rank logic on a smaller box)
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        backend = os.environ.get("SKS_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def make_dem(cfgid, terrain):
    import paper_2003_02200_b200 as sk
    n = CONFIGS[cfgid]["n"]
    kind = sk.SyntheticKind.Fractal if terrain == "fractal" else sk.SyntheticKind.SmoothedNoise
    return sk.make_synthetic(kind, n, n, CELLSIZE, SEED).values


def parallelism(world):
    return (f"row-block sharded x{world} (every sector), NCCL reduce of f64 maps" if world > 1
            else "single GPU, all sectors")


def bench_config(cfgid, terrain, world):
    """The workload description; identical in both arms."""
    c = CONFIGS[cfgid]
    return {"workload": workload_name(cfgid, terrain), "dimy": c["n"], "dimx": c["n"], "ns": c["ns"], "h0": H0,
            "max_distance": c["max_distance"], "terrain": terrain, "cellsize": CELLSIZE,
            "l2": "GPU arm: flushed between timed steps (256 MiB device write, untimed)",
            "parallelism": parallelism(world)}


# ---- the reference on the host (oracle/_ref: the unmodified reference sources) ------
# Nothing below imports the product package: the DEM comes from the shim
# (ref_make_fractal, or the reference's own make_synthetic for SmoothedNoise).

def _ref():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import Ref, have_ref
    if not have_ref():
        raise RuntimeError("oracle/_ref/libskewshed_ref.so missing (build() it where /root/reference exists)")
    return Ref()


def ref_dem(ref, cfgid, terrain):
    n = CONFIGS[cfgid]["n"]
    if terrain == "fractal":
        return ref.make_fractal(n, n, SEED)
    out = np.empty((n, n), np.float32)
    ref._check(ref.lib.ref_make_synthetic(3, n, n, CELLSIZE, SEED, out))  # SyntheticKind::SmoothedNoise
    return out


def stratified_sectors(half, count, phase=0.0):
    """`count` sector indices spread evenly over [0, half) (costs vary with the
    shear angle, so a sample must span all of them)."""
    count = min(count, half)
    return sorted({int((t + phase) * half / count) % half for t in range(count)})


def cpu_sweep_sample(ref, dem, cfgid, threads, per_thread=2, phase=0.0):
    """The reference's public sector_sweep on a stratified sample of
    per_thread x threads sectors, claimed dynamically by `threads` host threads
    (as total_viewshed's workers claim them). Returns (POV-sector/s, seconds,
    sectors); the rate is measured directly (sample POV-sectors / wall)."""
    c = CONFIGS[cfgid]
    n, half = c["n"], c["ns"] // 2
    ks = stratified_sectors(half, per_thread * threads, phase)
    secs = ref.sweep_sample(dem, CELLSIZE, c["ns"], H0, c["max_distance"], ks, threads)
    return n * n * len(ks) / secs, secs, ks


def cpu_baseline_main(args):
    """--cpu-baseline-only: runs in a subprocess of the GPU arm, so the GPU
    arm's process never maps oracle code."""
    ref = _ref()
    threads = os.cpu_count() or 1
    dem = ref_dem(ref, args.config, args.terrain)
    value, secs, ks = cpu_sweep_sample(ref, dem, args.config, threads)
    print(json.dumps({"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                      "sample": (f"the reference's sector_sweep (engine.cpp:235-244: relocation, scan, unskew) "
                                 f"on {len(ks)} stratified sectors {ks} of the same workload, {threads} host threads "
                                 f"claiming sectors dynamically, {secs:.1f} s wall; value = sample POV-sectors / wall "
                                 f"(no extrapolation)")}), flush=True)


def run_reference(args, world, rank):
    """--impl reference: the reference's own stock code path on the host
    cores, rank 0 only. Configs 1-3: the stock total_viewshed (engine.cpp:
    222-233, workers = all host threads) over the WHOLE workload, timed in full
    as many times as fit the time budget (at least once). Configs 4-5 (hours
    of CPU): stratified sector_sweep samples, projected with the exact scan
    work from the reference's own row ranges."""
    if rank != 0:
        return
    cfgid = args.config
    c = CONFIGS[cfgid]
    n, ns, half = c["n"], c["ns"], c["ns"] // 2
    ref = _ref()
    dem = ref_dem(ref, cfgid, args.terrain)
    threads = os.cpu_count() or 1
    povs = n * n * half
    walls = []
    t_start = time.perf_counter()
    if cfgid <= 3:
        out = np.empty((n, n), np.float64)
        stats = np.zeros(5, np.float64)
        while True:
            t0 = time.perf_counter()
            ref._check(ref.lib.ref_total_viewshed(dem, n, n, CELLSIZE, ns, H0, threads, c["max_distance"] or 0.0,
                                                  1, 0, out, stats.ctypes.data))
            walls.append(time.perf_counter() - t0)
            elapsed = time.perf_counter() - t_start
            if len(walls) >= args.steps or elapsed + walls[-1] > args.ref_budget:
                break
        wall = float(np.mean(walls))
        value = povs / wall
        sample = (f"the stock total_viewshed (engine.cpp:222-233) on the whole workload, workers = {threads} "
                  f"host threads; {len(walls)} full run(s) timed ({', '.join(f'{w:.1f}' for w in walls)} s), "
                  f"value = {povs} POV-sectors / mean wall")
        kind_steps = len(walls)
    else:
        work = [ref.sector_work(n, n, CELLSIZE, ns, k, c["max_distance"]) for k in range(half)]
        total = float(sum(work))
        rates = []
        while True:
            ks = stratified_sectors(half, threads, phase=len(walls) / max(args.steps, 1))
            secs = ref.sweep_sample(dem, CELLSIZE, ns, H0, c["max_distance"], ks, threads)
            walls.append(secs)
            rates.append(sum(work[k] for k in ks) / secs)
            elapsed = time.perf_counter() - t_start
            if len(walls) >= args.steps or elapsed + walls[-1] > args.ref_budget:
                break
        wall = total / float(np.mean(rates))  # projected whole-workload wall
        value = povs / wall
        sample = (f"the reference's sector_sweep (engine.cpp:235-244) on {len(walls)} stratified samples of "
                  f"{threads} sectors ({threads} host threads); whole-workload wall projected from the exact "
                  f"scan work of every sector (the reference's own build_skw row ranges; scan = 99.3% of its "
                  f"time, SURVEY 6): {wall:.0f} s")
        kind_steps = len(walls)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": kind_steps, "warmup": 0, "steps_requested": args.steps, "warmup_requested": args.warmup,
        "steps_note": ("each step is one full stock run of the workload (a CPU needs no warm-up); as many as "
                       f"fit the {args.ref_budget:.0f} s budget" if cfgid <= 3 else
                       f"each step is one sector sample; as many as fit the {args.ref_budget:.0f} s budget"),
        "ms_per_step": float(np.mean(walls)) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(cfgid, args.terrain, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm -------------------------------------------------------------------------

def run_ours(args, world, rank, local):
    import torch

    import paper_2003_02200_b200 as sk
    from paper_2003_02200_b200.distributed import RowBalancer, my_sectors, total_viewshed_distributed

    cfgid = args.config
    c = CONFIGS[cfgid]
    n, ns, maxd = c["n"], c["ns"], c["max_distance"]
    cfg = sk.RunConfig(ns=ns, h0=H0, max_distance=maxd, units=sk.Units.SquareKilometers, device=local)
    dem = make_dem(cfgid, args.terrain)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = sk.Context(local)
    mine = my_sectors(ns, n, n, world, rank, CELLSIZE, maxd)
    d_dem = torch.from_numpy(dem).to(dev)
    d_map = torch.zeros((n, n), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    factor = sk.area_scale_factor(cfg, CELLSIZE)
    balancer = RowBalancer(world)

    def step(want_stats):
        d_map.zero_()
        if world > 1:  # row-block sharding (distributed.py: balances terrain-dependent costs)
            st = ctx.run_rows(d_dem.data_ptr(), n, n, CELLSIZE, cfg, rank, world, d_map.data_ptr(),
                              stream=stream.cuda_stream, want_stats=want_stats, cuts=balancer.cuts)
        else:
            st = ctx.run_sectors(d_dem.data_ptr(), n, n, CELLSIZE, cfg, mine, d_map.data_ptr(),
                                 stream=stream.cuda_stream, want_stats=want_stats)
        if world > 1:
            import torch.distributed as dist
            dist.reduce(d_map, dst=0, op=dist.ReduceOp.SUM)
        if rank == 0:
            ctx.scale(d_map.data_ptr(), n * n, ns, CELLSIZE, int(cfg.units), stream.cuda_stream)
        return st

    rank_ms = []
    for _ in range(args.warmup):
        wst = step(world > 1)
        if world > 1:
            # warm-up doubles as the row-block rebalancing: every rank's kernel
            # time for its blocks (the phase events, which exclude the host's
            # plan building for new cuts), all-gathered, moves the cuts; they
            # are frozen for the timed steps
            import torch.distributed as dist
            torch.cuda.synchronize()
            busy = (wst.skew_seconds + wst.scan_seconds + wst.fixup_seconds + wst.unskew_seconds) * 1e3
            mine_t = torch.tensor([busy], dtype=torch.float64, device=dev)
            got = [torch.zeros_like(mine_t) for _ in range(world)]
            dist.all_gather(got, mine_t)
            rank_ms = [float(x.item()) for x in got]
            balancer.update(rank_ms)
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    total_ms = 0.0
    phases = dict(skew=0.0, scan=0.0, fixup=0.0, unskew=0.0)
    launches = 0
    flagged = 0
    evals = 0
    skipped = 0
    scan_kernel = 0
    for _ in range(args.steps):
        flush.fill_(1)  # evict L2 (126 MB) between steps, outside the timed region
        torch.cuda.synchronize()
        barrier(world)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = step(True)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        total_ms += e0.elapsed_time(e1)
        phases["skew"] += st.skew_seconds
        phases["scan"] += st.scan_seconds
        phases["fixup"] += st.fixup_seconds
        phases["unskew"] += st.unskew_seconds
        launches += st.kernel_launches + (1 if rank == 0 else 0)
        flagged += st.flagged_groups
        evals += st.target_evals
        skipped += st.skipped_target_slots
        scan_kernel = st.scan_kernel
    sampler.stop()
    total_ms = max_over_ranks(total_ms, world)
    scan_s = max_over_ranks(phases["scan"], world)
    skew_s = max_over_ranks(phases["skew"], world)
    unskew_s = max_over_ranks(phases["unskew"], world)
    evals_all = sum_over_ranks(evals, world)
    launches_all = int(sum_over_ranks(launches, world))
    flagged_all = int(sum_over_ranks(flagged, world))
    skipped_all = sum_over_ranks(skipped, world)
    ms_per_step = total_ms / args.steps
    povs = n * n * (ns // 2)
    value = povs / (ms_per_step * 1e-3)

    # e2e through the public API with host buffers (H2D of the DEM and D2H of
    # the map inside every timed step)
    pinned_dem = torch.from_numpy(dem).pin_memory()
    pinned_out = torch.empty((n, n), dtype=torch.float64).pin_memory()
    # cold: a fresh context's first call (host plans, batch metadata uploads,
    # device buffer allocation, the run, the copies), once, reported beside
    # the warm e2e
    cold_s = None
    if world == 1:
        cold = sk.Context(local)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cold.total_viewshed(pinned_dem.numpy(), CELLSIZE, cfg, out=pinned_out.numpy())
        cold_s = time.perf_counter() - t0
        cold.close()
        del cold
    e2e_times = []
    for i in range(args.warmup + args.steps):
        barrier(world)
        t0 = time.perf_counter()
        if world == 1:
            ctx.total_viewshed(pinned_dem.numpy(), CELLSIZE, cfg, out=pinned_out.numpy())
        else:
            total_viewshed_distributed(pinned_dem.numpy(), CELLSIZE, cfg, context=ctx, cuts=balancer.cuts)
            torch.cuda.synchronize()
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_times.append(t1 - t0)
    e2e_s = max_over_ranks(float(np.mean(e2e_times)), world)
    e2e_value = povs / e2e_s

    if rank != 0:
        return
    peaks, peak_kind = load_peaks()
    clocks = sampler.summary()
    props = torch.cuda.get_device_properties(dev)
    sm_max = float(peaks.get("sm_max_mhz") or clocks.get("sm_max_mhz") or 1965.0)
    fp32_peak = props.multi_processor_count * 128 * sm_max * 1e6  # lane-ops/s
    scan_achieved = 4.0 * evals_all / max(scan_s, 1e-12) if world == 1 else 4.0 * evals_all / max(scan_s * world, 1e-12)
    traffic = None
    reloc_traffic = unskew_traffic = None
    issue_active = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):  # dram read+write bytes per launch from one ncu --set full capture
        try:
            with open(prof) as f:
                nsum = json.load(f)
            wl = nsum.get("workloads", {}).get(f"{cfgid}/{args.terrain}", {})
            traffic = wl.get("scan_kernel", {}).get("dram_bytes_per_launch")
            issue_active = wl.get("scan_kernel", {}).get("issue_active")
            reloc_traffic = wl.get("relocate_kernel", {}).get("dram_bytes_per_launch")
            unskew_traffic = wl.get("unskew_kernel", {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = reloc_traffic = unskew_traffic = issue_active = None
    reloc_bytes = 8.0 * n * n * (ns // 2) * args.steps / world
    # unskew: 4 B of cv per cell and sector + the FP64 map read and written once
    unskew_bytes = (4.0 * (ns // 2) + 16.0) * n * n * args.steps / world
    executed = 4.0 * (evals_all - skipped_all) / max(scan_s * (world if world > 1 else 1), 1e-12)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32+f64",
        "dtype_note": "certified f32 filter for the line-of-sight decisions, f64 for every uncertain decision "
                      "(the reference's own operations) and for the accumulated map; integer ring sums",
        "data": "synthetic",
        "config": bench_config(cfgid, args.terrain, world),
        "row_balance": ({"cuts": [round(float(x), 6) for x in balancer.cuts],
                         "last_warmup_rank_ms": [round(x, 3) for x in rank_ms],
                         "note": "row-block cuts moved from measured per-rank times during warm-up, then frozen"}
                        if world > 1 else None),
        "scan_kernel": {2: "scan2 (one row x 64 positions per task)", 3: "scan3 row pairs",
                        4: "scan3 row quads"}.get(scan_kernel, str(scan_kernel)),
        "roofline": {"kernel": ({2: "scan2_kernel", 3: "scan3_kernel<2>", 4: "scan3_kernel<4>"}.get(scan_kernel, "scan")
                                + " (FP32-issue bound)"), "bound": "fp32",
                     "achieved": scan_achieved / 1e12, "peak": fp32_peak / 1e12, "unit": "TFLOP/s",
                     "frac": scan_achieved / fp32_peak, "traffic": traffic,
                     "executed_frac": executed / fp32_peak,
                     "issue_active": issue_active,
                     "note": (f"4 algorithmic FP32 ops per target evaluation (SURVEY 8d) x "
                              f"{evals_all / args.steps:.4g} evals/step / scan-kernel CUDA-event time; peak = "
                              f"{props.multi_processor_count} SMs x 128 lanes x {sm_max:g} MHz (sm_max). "
                              f"{100.0 * skipped_all / max(evals_all, 1):.1f}% of the evaluations were decided "
                              f"(hidden, certified) by the hidden-block skip test without per-target FP32 work; "
                              f"they are counted as evaluated. executed_frac counts only the evaluations the "
                              f"kernel performed; issue_active is the scan kernel's smsp issue-active fraction "
                              f"from the committed ncu capture of this workload (profiles/ncu_summary.json)")},
        "roofline_relocation": {"kernel": "relocate_kernel", "bound": "hbm",
                                "achieved": reloc_bytes / max(skew_s, 1e-12) / 1e9,
                                "peak": float(peaks.get("hbm_gbs", 6650.0)), "unit": "GB/s",
                                "frac": reloc_bytes / max(skew_s, 1e-12) / 1e9 / float(peaks.get("hbm_gbs", 6650.0)),
                                "peak_kind": peak_kind, "traffic": reloc_traffic,
                                "note": ("algorithmic 8N bytes per sector (read N, write N covered cells); the "
                                         "kernel also zeroes the N cv cells it covers (4N more written)")},
        # the TMA-staged kernel when both DEM sides are multiples of 4 (engine.cu unskew_maps)
        "roofline_unskew": {"kernel": ("unskew_tma_kernel" if n % 4 == 0 and os.environ.get("SKS_UNSKEW_TMA", "1")[:1] != "0"
                                       else "unskew_pipe_kernel"), "bound": "hbm",
                            "achieved": unskew_bytes / max(unskew_s, 1e-12) / 1e9,
                            "peak": float(peaks.get("hbm_gbs", 6650.0)), "unit": "GB/s",
                            "frac": unskew_bytes / max(unskew_s, 1e-12) / 1e9
                            / float(peaks.get("hbm_gbs", 6650.0)),
                            "peak_kind": peak_kind, "traffic": unskew_traffic,
                            "note": "algorithmic 4 B of cv per cell and sector + 16 B of FP64 map per cell"},
        "phase_ms_per_step": {k: v * 1e3 / args.steps for k, v in phases.items()},
        "target_evals_per_s": evals_all / args.steps / (ms_per_step * 1e-3),
        "flagged_groups_per_step": flagged_all / args.steps,
        "skip_decided_frac": skipped_all / max(evals_all, 1),
        "e2e": {"value": e2e_value, "unit": UNIT, "seconds": e2e_s,
                "h2d_bytes_per_step": int(n * n * 4 * world), "d2h_bytes_per_step": int(n * n * 8)},
        "e2e_cold": ({"value": povs / cold_s, "unit": UNIT, "seconds": cold_s,
                      "note": "a fresh context's first total_viewshed call: host plans, metadata uploads and "
                              "device allocations included (the warm e2e reuses them)"}
                     if cold_s else None),
        "gpu_launches": launches_all,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        # the reference on the host cores, in a subprocess (this process never
        # maps oracle code); a bounded sample of the same workload
        try:
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-baseline-only", "--config",
                                str(cfgid), "--terrain", args.terrain], capture_output=True, text=True,
                               timeout=600)
            line["cpu_baseline"] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--terrain", choices=["fractal", "smooth"], default="fractal")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline-only", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="seconds of reference runs in --impl reference (at least one full run)")
    args = ap.parse_args()
    if args.cpu_baseline_only:
        cpu_baseline_main(args)
        return
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup(args.gpus)
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
