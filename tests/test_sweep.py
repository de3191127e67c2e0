"""Rotational-sweep viewshed (the reference's independent oracle, oracle.cpp)
on the GPU, heatmap output and the observer helpers.

CPU tests pin the C restatement (oracle/skewshed_oracle.c) and the host
pieces (ray tables / select_axis_point_set, random_povs, write_heatmap)
against the reference itself (oracle/_ref). GPU tests compare the device
sweep bit for bit with the reference (or, where oracle/_ref is absent, with
the pinned restatement), and check the reference's own acceptance criterion
1 (acceptance_main.cpp:64-110): the sDEM engine agrees with the sweep to
mean <= 5 %, p99 <= 15 %.
"""
import math
import random

import numpy as np
import pytest

import paper_2003_02200_b200 as sk
from _oracle import Orc, Ref, have_orc, have_ref

sw = sk.sweep
needs_ref = pytest.mark.skipif(not have_ref(), reason="needs oracle/_ref (built from /root/reference)")


def _checker():
    """The reference when built here, else the pinned C restatement."""
    return Ref() if have_ref() else Orc()


def _dem(kind, dimy, dimx, seed=7):
    return sk.make_synthetic(kind, dimy, dimx, 10.0, seed)


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


# ---------------------------------------------------------------- CPU ----

@needs_ref
def test_restated_singular_viewshed_matches_reference_bits():
    ref, orc = Ref(), Orc()
    rng = random.Random(5)
    for kind, dy, dx in ((sk.SyntheticKind.Fractal, 23, 31), (sk.SyntheticKind.Cone, 17, 17),
                         (sk.SyntheticKind.SmoothedNoise, 12, 40), (sk.SyntheticKind.Ramp, 9, 9)):
        v = _dem(kind, dy, dx).values
        for _ in range(12):
            i, j = rng.randrange(dy), rng.randrange(dx)
            ns = rng.choice([2, 4, 6, 8, 16, 36])
            h0 = rng.choice([0.0, 1.5, 30.0])
            md = rng.choice([None, 35.0, 1e9])
            a = ref.singular_viewshed(v, i, j, h0, ns, md)
            b = orc.singular_viewshed(v, i, j, h0, ns, md)
            assert a == b or (math.isnan(a) and math.isnan(b)), (kind, i, j, ns, h0, md, a, b)


@needs_ref
def test_axis_point_set_matches_reference():
    ref = Ref()
    rng = random.Random(11)
    dem = sk.Dem(np.zeros((37, 53), np.float32), 10.0)
    azs = [0.0, 45.0, 90.0, 135.0, 180.0, 225.0, 270.0, 315.0, 359.0, 26.565051177077994]
    azs += [rng.uniform(0, 540) for _ in range(60)] + [k * (360.0 / 180) + off for k in range(90) for off in (0, 180)]
    for az in azs:
        i0, j0 = rng.randrange(37), rng.randrange(53)
        got = [(p.i, p.j) for p in sw.select_axis_point_set(dem, i0, j0, az)]
        assert got == ref.axis_point_set(37, 53, i0, j0, az), (az, i0, j0)
    with pytest.raises(IndexError, match=r"observer \(37, 0\) outside grid 37x53"):
        sw.select_axis_point_set(dem, 37, 0, 0.0)


def test_random_povs_are_the_references_scaled_mt19937_draws():
    orc = Orc()
    dem = sk.Dem(np.zeros((1000, 77), np.float32), 1.0)
    povs = sw.random_povs(dem, 50, 2024)
    for t, p in enumerate(povs):  # cli.cpp:212-218: i from draw 2t+1, j from draw 2t+2 (1-based)
        assert p.i == (orc.lib.orc_mt19937_nth(2024, 2 * t + 1) * 1000) >> 32
        assert p.j == (orc.lib.orc_mt19937_nth(2024, 2 * t + 2) * 77) >> 32


@needs_ref
def test_heatmap_bytes_match_reference(tmp_path):
    ref = Ref()
    rng = np.random.default_rng(3)
    grids = [rng.random((37, 53)) * 1e6, np.full((4, 5), 7.5), rng.standard_normal((300, 200)) * 1e3,
             np.array([[0.0, 1.0], [0.5, 0.25]])]
    grids[0][3, 4] = 0.0
    for g in grids:
        for pal in (sk.Palette.Gray, sk.Palette.BlueRed):
            ours, theirs = tmp_path / "o.p", tmp_path / "r.p"
            sk.write_heatmap(sk.VsGrid(g), ours, pal)
            ref.write_heatmap(theirs, g, int(pal))
            assert ours.read_bytes() == theirs.read_bytes(), (g.shape, pal)
    bad = grids[0].copy()
    bad[5, 6] = np.inf
    with pytest.raises(ValueError, match="cannot render a grid with non-finite values"):
        sk.write_heatmap(sk.VsGrid(bad), tmp_path / "x.pgm")
    with pytest.raises(ValueError, match="cannot render an empty grid"):
        sk.write_heatmap(sk.VsGrid(np.zeros((0, 3))), tmp_path / "x.pgm")
    with pytest.raises(RuntimeError, match="cannot open"):
        sk.write_heatmap(sk.VsGrid(grids[1]), tmp_path / "missing" / "x.pgm")


def test_sweep_argument_errors_before_the_device():
    dem = _dem(sk.SyntheticKind.Cone, 16, 16)
    with pytest.raises(IndexError, match=r"observer \(16, 3\) outside grid 16x16"):
        sw.singular_viewshed(dem, 16, 3, 1.5, 8)
    with pytest.raises(ValueError, match="sector count must be an even integer >= 2"):
        sw.singular_viewshed(dem, 1, 3, 1.5, 7)
    # multi: first observer's position, then ns, then the rest (oracle.cpp:131-141)
    with pytest.raises(IndexError, match=r"observer \(-1, 0\)"):
        sw.multi_viewshed(dem, [(-1, 0), (2, 2)], 1.5, 7)
    with pytest.raises(ValueError, match="sector count"):
        sw.multi_viewshed(dem, [(0, 0), (99, 2)], 1.5, 7)
    with pytest.raises(IndexError, match=r"observer \(99, 2\)"):
        sw.multi_viewshed(dem, [(0, 0), (99, 2)], 1.5, 8)
    big = sk.Dem(np.zeros((300, 300), np.float32), 10.0)
    with pytest.raises(RuntimeError, match=r"reference total viewshed on 300x300 \(90000 cells\) refused"):
        sw.total_viewshed_reference(big, sk.RunConfig(ns=8))
    bad = dem.values.copy()
    bad[2, 5] = np.nan
    with pytest.raises(ValueError, match=r"invalid grid: non-finite elevation at cell \(2, 5\)"):
        sw.total_viewshed_reference(sk.Dem(bad, 10.0), sk.RunConfig(ns=8))
    with pytest.raises(ValueError, match="invalid config: ns must be an even integer >= 2, got 5"):
        sw.total_viewshed_reference(dem, sk.RunConfig(ns=5))


@needs_ref
def test_sweep_error_messages_match_reference():
    ref = Ref()
    big = np.zeros((300, 300), np.float32)
    with pytest.raises(RuntimeError) as a:
        ref.total_viewshed_reference(big, 8, 1.5, force=False)
    with pytest.raises(RuntimeError) as b:
        sw.total_viewshed_reference(sk.Dem(big, 10.0), sk.RunConfig(ns=8))
    assert str(a.value) == str(b.value)
    v = _dem(sk.SyntheticKind.Cone, 16, 16).values
    with pytest.raises(IndexError) as a:
        ref.singular_viewshed(v, 3, 16, 1.5, 8)
    with pytest.raises(IndexError) as b:
        sw.singular_viewshed(sk.Dem(v, 10.0), 3, 16, 1.5, 8)
    assert str(a.value) == str(b.value)


# ---------------------------------------------------------------- GPU ----

@pytest.mark.gpu
@pytest.mark.parametrize("kind,dy,dx,ns,h0,md,units", [
    (sk.SyntheticKind.Fractal, 40, 56, 8, 1.5, None, 0),
    (sk.SyntheticKind.Fractal, 33, 33, 36, 1.5, 120.0, 1),
    (sk.SyntheticKind.SmoothedNoise, 48, 48, 180, 1.5, None, 0),
    (sk.SyntheticKind.Cone, 24, 40, 16, 0.0, None, 0),
    (sk.SyntheticKind.Ramp, 40, 24, 2, 0.0, None, 0),
    (sk.SyntheticKind.Flat, 2, 2, 4, 1.5, None, 1),
    (sk.SyntheticKind.Fractal, 64, 64, 90, 10.0, 200.0, 0),
])
def test_total_viewshed_reference_bit_exact(kind, dy, dx, ns, h0, md, units):
    dem = _dem(kind, dy, dx)
    cfg = sk.RunConfig(ns=ns, h0=h0, max_distance=md, units=sk.Units(units))
    got = sw.total_viewshed_reference(dem, cfg)
    chk = _checker()
    if isinstance(chk, Ref):
        want = chk.total_viewshed_reference(dem.values, ns, h0, md, units)
    else:
        want = chk.rotational_rows(dem.values, ns, h0, md, units)
    assert got.units == sk.Units(units)
    assert np.array_equal(_bits(got.values), _bits(want))


@pytest.mark.gpu
def test_singular_and_multi_viewshed_bit_exact():
    dem = _dem(sk.SyntheticKind.Fractal, 61, 47, seed=3)
    chk = _checker()
    rng = random.Random(9)
    for _ in range(20):
        i, j = rng.randrange(61), rng.randrange(47)
        ns, h0, md = rng.choice([2, 8, 90, 360]), rng.choice([0.0, 1.5, 25.0]), rng.choice([None, 150.0])
        got = sw.singular_viewshed(dem, i, j, h0, ns, md)
        assert got == chk.singular_viewshed(dem.values, i, j, h0, ns, md), (i, j, ns, h0, md)
    povs = [(3, 4), (60, 46), (3, 4), (0, 0), (30, 20)]  # a repeated observer accumulates in list order
    mv = sw.multi_viewshed(dem, povs, 1.5, 36)
    areas = [chk.singular_viewshed(dem.values, i, j, 1.5, 36) for i, j in povs]
    tot = 0.0
    for a in areas:
        tot += a
    assert mv.total_area == tot
    assert mv.grid.values[3, 4] == areas[0] + areas[2]
    assert np.count_nonzero(mv.grid.values) == 4
    if isinstance(chk, Ref):
        grid, total = chk.multi_viewshed(dem.values, povs, 1.5, 36)
        assert np.array_equal(_bits(grid), _bits(mv.grid.values)) and total == mv.total_area
    assert sw.multi_viewshed(dem, [], 1.5, 7).total_area == 0.0  # no observer, no checks (oracle.cpp:136)


@pytest.mark.gpu
def test_forced_large_grid_matches_restatement_on_sampled_rows():
    """Beyond the cell guard (force): 300x260, sampled rows against the C
    restatement (itself pinned to the reference above)."""
    dem = _dem(sk.SyntheticKind.Fractal, 300, 260, seed=21)
    cfg = sk.RunConfig(ns=16, h0=1.5, units=sk.Units.SquareMeters)
    got = sw.total_viewshed_reference(dem, cfg, force=True)
    orc = Orc()
    for lo in (0, 149, 298):
        want = orc.rotational_rows(dem.values, 16, 1.5, None, 0, rows=(lo, lo + 2))
        assert np.array_equal(_bits(got.values[lo:lo + 2]), _bits(want[lo:lo + 2])), lo


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed", [(32, 7), (48, 11), (64, 13)])
def test_acceptance_criterion_1_engine_vs_sweep(n, seed):
    """acceptance_main.cpp:64-110: SmoothedNoise n x n, ns=180, h0=1.5, m^2:
    the sDEM engine vs the rotational sweep, mean <= 5 %, p99 <= 15 %."""
    dem = _dem(sk.SyntheticKind.SmoothedNoise, n, n, seed)
    cfg = sk.RunConfig(ns=180, h0=1.5, units=sk.Units.SquareMeters)
    eng = sk.total_viewshed(dem, cfg).values
    ref = sw.total_viewshed_reference(dem, cfg).values
    rel = np.sort((np.abs(eng - ref) / ref).ravel())
    p99 = rel[int(math.ceil(0.99 * rel.size)) - 1]
    assert rel.mean() <= 0.05 and p99 <= 0.15, (rel.mean(), p99)


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [1.0, 3.0e12, 2.0e-13])
def test_sweep_filter_matches_exact_path(scale, monkeypatch):
    """The FP32 filter of sweep_dirs_kernel only certifies hidden cells:
    its results equal the pure-FP64 kernel's (SKS_SWEEP_EXACT) and the
    restated oracle bit for bit, including elevations outside the filter's
    proven range (the filter is then switched off)."""
    v = sk.make_synthetic(sk.SyntheticKind.Fractal, 128, 120, 10.0, 11).values * np.float32(scale)
    dem = sk.Dem(np.ascontiguousarray(v, np.float32), 10.0)
    cfg = sk.RunConfig(ns=90, h0=1.5, units=sk.Units.SquareMeters)
    fast = sw.total_viewshed_reference(dem, cfg, force=True).values
    monkeypatch.setenv("SKS_SWEEP_EXACT", "1")
    exact = sw.total_viewshed_reference(dem, cfg, force=True).values
    assert np.array_equal(_bits(fast), _bits(exact))
    want = Orc().rotational_rows(dem.values, 90, 1.5, None, 0, rows=(60, 62))
    assert np.array_equal(_bits(fast[60:62]), _bits(want[60:62]))


@pytest.mark.gpu
def test_linear_scan_rings_bit_exact_and_well_formed():
    """linear_scan with ring sectors (oracle.cpp:74-106) on the GPU: the
    reference's ring list and ring sum bit for bit (when oracle/_ref is
    built), and test_oracle.cpp:187-209's properties: 0 < r_open < r_close,
    rings ordered, sum of r_close^2 - r_open^2 = cv."""
    dem = _dem(sk.SyntheticKind.SmoothedNoise, 24, 24, seed=17)
    rng = random.Random(5)
    ref = Ref() if have_ref() else None
    for _ in range(60):
        i, j = rng.randrange(24), rng.randrange(24)
        az = rng.randrange(3600) / 10.0
        cap = rng.choice([float("inf"), 7.5])
        h = float(dem.values[i, j]) + 1.5
        rings = []
        cv = sw.linear_scan(dem, i, j, h, az, cap, rings)
        prev, measured = 0.0, 0.0
        for r in rings:
            assert 0.0 < r.r_open < r.r_close and r.r_open >= prev
            prev = r.r_close
            measured += r.r_close * r.r_close - r.r_open * r.r_open
        assert cv == pytest.approx(measured, rel=1e-12)
        if ref is not None:
            rcv, rrings = ref.linear_scan(dem.values, i, j, h, az, cap)
            assert cv == rcv and [(r.r_open, r.r_close) for r in rings] == rrings


@pytest.mark.gpu
def test_singular_viewshed_shift_invariance():
    """test_oracle.cpp:175-185: adding 64 m to every elevation changes no
    singular viewshed (the GPU sweep reproduces the reference's arithmetic,
    so the reference's invariant carries over exactly)."""
    dem = _dem(sk.SyntheticKind.SmoothedNoise, 16, 16, seed=3)
    shifted = sk.Dem(dem.values + np.float32(64.0), dem.cellsize)
    for i, j in ((0, 0), (5, 7), (11, 3)):
        assert sw.singular_viewshed(dem, i, j, 1.5, 36) == sw.singular_viewshed(shifted, i, j, 1.5, 36)
