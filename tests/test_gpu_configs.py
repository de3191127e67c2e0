"""GPU parity at the BASELINE configurations' own sizes (configs 2-5) and on
the long-row path, against the reference (oracle/_ref, the unmodified
reference sources).

What is compared, per configuration (BASELINE.json configs):
  * config 2 (2000^2, ns 180): the WHOLE raw map of total_viewshed_raw,
    bit for bit, against the reference's own total_viewshed_raw on every
    host thread (engine.cpp:109-220).
  * config 3 (2000^2, ns 360, 10 km cap): four whole sectors (0, 22, 44.5,
    134 degrees) through the production path (sector_sweep: relocation ->
    scan -> fixup -> unskew) against the reference's sector_sweep
    (engine.cpp:235-244), bit for bit.
  * config 4 (4000^2, ns 180): four whole sectors scanned on the GPU; every
    POV of rows sampled from every row-length decile compared with the
    reference's sector_viewshed (scan.cpp:64-85) on the same rows.
  * config 5 (10000^2, ns 180): two whole sectors scanned on the GPU; every
    POV of the longest rows (10 000 cells) and of sampled shorter rows
    compared with the reference.
  * SmoothedNoise (the reference's own generator, dem.cpp:152-170) at 2000^2:
    four whole sectors, bit for bit.
  * rows longer than the shared-memory scan holds (sks_scan_row_limit): the
    exact per-POV path, bit for bit, plus the same path forced at small
    sizes (SKS_LONG_ROW) end to end; rows of 9 000-14 000 cells on the
    scan's one-table-copy layout.
The reference runs on host threads in parallel (ctypes releases the GIL).
"""
from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np
import pytest

import paper_2003_02200_b200 as sk
from _oracle import NO_CAP, Ref, have_ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_ref(), reason="oracle/_ref (the compiled reference) is missing")]

THREADS = max(1, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def ref():
    return Ref()


def b64(a):
    return np.ascontiguousarray(a).view(np.uint64)


def _ref_sdem(ref, dem, k, ns):
    p = sk.plan_sector(k, ns, *dem.shape)
    pre = ref.apply_pre_ops(dem, k, ns)
    v, _w, rr, base = ref.build_skw(pre, p.shear_tan)
    return p, v, rr, base


def _ref_rows(ref, v, rr, rows, p, h0, max_dd=NO_CAP):
    """The reference's sector_viewshed on the given skewed rows only (rows are
    independent), chunked over host threads; returns skwVS of those rows."""
    rows = np.asarray(rows)
    chunks = [c for c in np.array_split(rows, min(len(rows), THREADS)) if len(c)]

    def one(c):
        # a SkwGrid of just these rows: skw_rows() = base + src_rows (skew.hpp:67)
        return ref.sector_viewshed(np.ascontiguousarray(v[c]), np.ascontiguousarray(rr[c]), len(c), 0,
                                   p.shear_tan, h0, max_dd)

    with ThreadPoolExecutor(len(chunks)) as ex:
        outs = list(ex.map(one, chunks))
    return np.concatenate(outs, axis=0)


def _decile_rows(rr, per_decile, rng):
    """Skewed rows with >= 2 cells, sampled from every decile of row length."""
    L = rr[:, 1] - rr[:, 0]
    rows = np.nonzero(L >= 2)[0]
    order = rows[np.argsort(L[rows], kind="stable")]
    picks = []
    for part in np.array_split(order, 10):
        if len(part):
            picks.extend(rng.choice(part, min(per_decile, len(part)), replace=False).tolist())
    return np.array(sorted(set(picks)))


# ---- config 2: the whole map ------------------------------------------------------

def test_config2_whole_map_bitexact(ref):
    """The north-star target itself: the full 2000^2 / 180-sector raw map (4 M
    cells x 90 sectors) bit-identical to the reference's total_viewshed_raw
    (about 80 s of reference time on 16 host threads)."""
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 2000, 2000, 10.0, 7)
    cfg = sk.RunConfig(ns=180, h0=1.5, units=sk.Units.SquareMeters)
    ours = sk.total_viewshed_raw(dem, cfg)
    theirs = ref.total_viewshed(dem.values, 10.0, 180, 1.5, raw=True, workers=THREADS)
    assert np.array_equal(b64(ours), b64(theirs)), int(np.sum(ours != theirs))


# ---- config 3: 360 sectors, 10 km cap -------------------------------------------------

def test_config3_whole_sectors_bitexact(ref):
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 2000, 2000, 10.0, 7)
    cfg = sk.RunConfig(ns=360, h0=1.5, max_distance=10000.0, units=sk.Units.SquareMeters)
    ks = [0, 44, 89, 134]  # 0, 22, 44.5, 134 degrees
    for k in ks:  # the distance cap at these shears (engine.cpp:29-36)
        p = sk.plan_sector(k, 360, 2000, 2000)
        assert 700 <= sk.distance_cap_cells(10000.0, p.shear_tan, 10.0) <= 1000
    with ThreadPoolExecutor(len(ks)) as ex:
        theirs = list(ex.map(lambda k: ref.sector_sweep(dem.values, 10.0, 360, 1.5, 10000.0, k), ks))
    for k, t in zip(ks, theirs):
        ours = sk.sector_sweep(dem, cfg, k).contribution
        assert np.array_equal(b64(ours), b64(t)), k


# ---- config 4: 4000^2 ---------------------------------------------------------------------

def test_config4_sampled_rows_every_length_bitexact(ref):
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 4000, 4000, 10.0, 7).values
    rng = np.random.default_rng(4)
    for k in (0, 11, 22, 67):  # 0, 22, 44, 134 degrees
        p, v, rr, base = _ref_sdem(ref, dem, k, 180)
        ours = sk.sector_viewshed(sk.SkwGrid(v, rr, base, p.rows, p.shear_tan), 1.5)
        rows = _decile_rows(rr, 3, rng)
        theirs = _ref_rows(ref, v, rr, rows, p, 1.5)
        assert np.array_equal(b64(ours[rows]), b64(theirs)), k
        # rows outside the sample: finite, zero outside the ranges
        assert np.all(np.isfinite(ours)) and np.all(ours >= 0.0)


# ---- config 5: 10000^2 -------------------------------------------------------------------

def test_config5_longest_rows_bitexact(ref):
    """Config 5's rows reach 10 000 cells (a skewed row's range is a column
    interval, so L <= dimx): whole sectors on the GPU, every POV of the
    longest rows and of sampled shorter rows against the reference."""
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 10000, 10000, 10.0, 7).values
    rng = np.random.default_rng(5)
    for k in (0, 44):  # 0 and 44 degrees
        p, v, rr, base = _ref_sdem(ref, dem, k, 180)
        L = rr[:, 1] - rr[:, 0]
        assert L.max() == 10000 and L.max() <= sk.scan_row_limit()
        ours = sk.sector_viewshed(sk.SkwGrid(v, rr, base, p.rows, p.shear_tan), 1.5)
        longest = np.nonzero(L == L.max())[0]
        rows = np.union1d(rng.choice(longest, min(6, len(longest)), replace=False), _decile_rows(rr, 1, rng))
        theirs = _ref_rows(ref, v, rr, rows, p, 1.5)
        assert np.array_equal(b64(ours[rows]), b64(theirs)), k
        del ours, v


# ---- the reference's own terrain at size ----------------------------------------------------

def test_smoothed_noise_2000_whole_sectors_bitexact(ref):
    """SmoothedNoise (dem.cpp:152-170, nearly flat: almost every target is a
    new maximum, so the hidden-window skip rarely fires and records are
    dense) at 2000^2 / ns 180: four whole sectors."""
    dem = sk.make_synthetic(sk.SyntheticKind.SmoothedNoise, 2000, 2000, 10.0, 7)
    cfg = sk.RunConfig(ns=180, h0=1.5, units=sk.Units.SquareMeters)
    ks = [0, 11, 22, 67]
    with ThreadPoolExecutor(len(ks)) as ex:
        theirs = list(ex.map(lambda k: ref.sector_sweep(dem.values, 10.0, 180, 1.5, None, k), ks))
    for k, t in zip(ks, theirs):
        ours = sk.sector_sweep(dem, cfg, k).contribution
        assert np.array_equal(b64(ours), b64(t)), k


# ---- rows longer than the shared-memory scan holds ---------------------------------------------

@pytest.mark.parametrize("max_dd", [NO_CAP, 5000])
def test_rows_beyond_scan_slots_bitexact(ref, max_dd):
    """Rows of 19 000 cells (above sks_scan_row_limit, ~17 300): the batch
    routes them whole through the exact per-POV kernel (its fl(1/d) table in
    global memory); rows of 14 000 and 12 000 cells in the same batch go
    through the shared-memory scan with ONE fl(1/d) table copy (the layout
    that holds 2 slots of config 5's 10 000-cell rows). Every POV of every
    row, both directions, ragged ranges, with and without a distance cap."""
    L = 19000
    assert 14000 < sk.scan_row_limit() < L
    rows = 6
    g = sk.make_synthetic(sk.SyntheticKind.Fractal, rows, L, 10.0, 23).values
    vals = np.ascontiguousarray(g, np.float32)
    rr = np.zeros((rows, 2), np.int32)
    rr[:, 1] = L
    rr[1] = (7, L - 3)
    rr[2] = (100, 14100)   # 14 000 cells
    rr[3] = (5, 12004)     # 11 999 cells
    rr[4] = (3000, 17000)  # 14 000 cells
    theirs = ref.sector_viewshed(vals, rr, rows, 0, 0.0, 1.5, max_dd)
    ours = sk.sector_viewshed(sk.SkwGrid(vals, rr, 0, rows, 0.0), 1.5, max_dd)
    assert np.array_equal(b64(ours), b64(theirs))


@pytest.mark.parametrize("h0", [0.0, 1.7])
def test_one_table_copy_layout_observer_heights(ref, h0):
    """Rows of 9 000-12 000 cells (the one-table-copy scan layout) with h0 = 0
    (exact ties on the ramp rows) and a non-float h0 (1.7: the two-float
    observer height, the kHl path, and POVs routed to the FP64 fixup)."""
    rows, L = 4, 12000
    g = sk.make_synthetic(sk.SyntheticKind.Fractal, rows, L, 10.0, 31).values.copy()
    g[2] = np.linspace(0.0, 60.0, L, dtype=np.float32)  # a ramp row: collinear targets
    rr = np.zeros((rows, 2), np.int32)
    rr[:, 1] = L
    rr[1] = (2500, 11500)
    for max_dd in (NO_CAP, 3000):
        theirs = ref.sector_viewshed(g, rr, rows, 0, 0.0, h0, max_dd)
        ours = sk.sector_viewshed(sk.SkwGrid(g, rr, 0, rows, 0.0), h0, max_dd)
        assert np.array_equal(b64(ours), b64(theirs)), max_dd


@pytest.mark.parametrize("shape,kind,ns,maxd", [
    ((90, 70), sk.SyntheticKind.Fractal, 36, None),
    ((64, 80), sk.SyntheticKind.SmoothedNoise, 24, 250.0),
    ((40, 60), sk.SyntheticKind.Ramp, 8, None),
])
def test_long_row_path_forced_end_to_end(ref, shape, kind, ns, maxd, monkeypatch):
    """SKS_LONG_ROW=48 sends every row longer than 48 cells through the
    long-row path (window maxima + full queue + exact kernel) while shorter
    rows of the same batch still go through scan2: the raw map is
    bit-identical to the reference, and row-block parts sum to it."""
    import torch

    monkeypatch.setenv("SKS_LONG_ROW", "48")
    dem = sk.make_synthetic(kind, *shape, 10.0, 17)
    cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=maxd, units=sk.Units.SquareMeters)
    theirs = ref.total_viewshed(dem.values, 10.0, ns, 1.5, max_distance=maxd or 0.0, raw=True)
    ctx = sk.Context(0)
    ours, st = ctx.total_viewshed(dem.values, 10.0, cfg, raw=True, want_stats=True)
    assert np.array_equal(b64(ours), b64(theirs))
    # the long rows' POVs all went through the fixup queue
    assert st.flagged_groups >= 2 * 49
    d_dem = torch.from_numpy(dem.values).cuda()
    total = np.zeros(shape, np.float64)
    for part in range(3):
        d_map = torch.zeros(shape, dtype=torch.float64, device="cuda")
        ctx.run_rows(d_dem.data_ptr(), *shape, 10.0, cfg, part, 3, d_map.data_ptr(),
                     stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        total += d_map.cpu().numpy()
    np.testing.assert_allclose(total, theirs, rtol=1e-12, atol=0)
    ctx.close()


def test_rows_beyond_int32_ring_sums_rejected():
    """A skewed row of more than 46 340 cells could overflow the exact int32
    ring sums (cv <= L^2 - 1): refused with the reference's exception type
    for bad inputs instead of a wrong answer."""
    dem = sk.Dem(np.zeros((2, 46341), np.float32), 10.0)
    with pytest.raises(ValueError, match="46340"):
        sk.total_viewshed_raw(dem, sk.RunConfig(ns=2))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,kind,ns,maxd", [
    ((90, 70), sk.SyntheticKind.Fractal, 36, None),
    ((64, 80), sk.SyntheticKind.SmoothedNoise, 24, 250.0),
    ((40, 60), sk.SyntheticKind.Ramp, 8, None),
])
def test_warp_fixup_kernel_bitexact(ref, shape, kind, ns, maxd, monkeypatch):
    """The opt-in warp-per-POV fixup (SKS_FIXUP=warp), fed every POV of the
    long rows (SKS_LONG_ROW=48) plus the scan's flagged ones: bit-identical
    raw maps."""
    monkeypatch.setenv("SKS_FIXUP", "warp")
    monkeypatch.setenv("SKS_LONG_ROW", "48")
    dem = sk.make_synthetic(kind, *shape, 10.0, 19)
    cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=maxd, units=sk.Units.SquareMeters)
    theirs = ref.total_viewshed(dem.values, 10.0, ns, 1.5, max_distance=maxd or 0.0, raw=True)
    ctx = sk.Context(0)
    ours = ctx.total_viewshed(dem.values, 10.0, cfg, raw=True)
    assert np.array_equal(b64(ours), b64(theirs))
    ctx.close()


@pytest.mark.gpu
def test_warp_fixup_kernel_exact_mode(ref, monkeypatch):
    """SKS_FIXUP=warp on elevations outside the FP32 filter's range: every
    POV takes the kernel's FP64 path (warp max-scan in FP64), bit-identical."""
    monkeypatch.setenv("SKS_FIXUP", "warp")
    base = sk.make_synthetic(sk.SyntheticKind.Fractal, 30, 26, 10.0, 5).values
    vals = np.ascontiguousarray(base * np.float32(3.0e12), np.float32)
    cfg = sk.RunConfig(ns=16, h0=0.0, units=sk.Units.SquareMeters)
    theirs = ref.total_viewshed(vals, 10.0, 16, 0.0, raw=True)
    ours = sk.total_viewshed_raw(sk.Dem(vals, 10.0), cfg)
    assert np.array_equal(b64(ours), b64(theirs))
