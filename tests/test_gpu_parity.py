"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

The oracle is the reference itself (oracle/_ref/libskewshed_ref.so, compiled
from the unmodified reference sources) when present, else the C
restatement (oracle/liboracle.so), which tests/test_oracle.py pins to the
reference bit-for-bit. Bars:
  * relocation: sDEM values and row ranges bit-exact (P1)
  * scan: per-POV cv and skwVS bit-exact; per-target visibility bit-exact (P2)
  * unskew: bit-exact (P3)
  * end to end on one GPU: bit-exact to total_viewshed_raw (P4, stronger
    than the 1e-5 relative bar)
"""
import numpy as np
import pytest

import paper_2003_02200_b200 as sk
from _oracle import NO_CAP, Orc, Ref, have_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ora():
    return Ref() if have_ref() else Orc()


def b32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def b64(a):
    return np.ascontiguousarray(a).view(np.uint64)


# ---- P1 relocation ---------------------------------------------------------

@pytest.mark.parametrize("shape,kind,ns", [
    ((64, 64), sk.SyntheticKind.SmoothedNoise, 180),
    ((24, 40), sk.SyntheticKind.SmoothedNoise, 36),
    ((40, 24), sk.SyntheticKind.Fractal, 36),
    ((33, 33), sk.SyntheticKind.Cone, 360),
    ((2, 2), sk.SyntheticKind.Ramp, 8),
    ((130, 70), sk.SyntheticKind.Fractal, 24),
    # interior and edge tiles of the TMA pipeline, an odd DEM width (pitched copy)
    ((203, 181), sk.SyntheticKind.Fractal, 12),
])
def test_relocation_bitexact_every_sector(ora, shape, kind, ns):
    dem = sk.make_synthetic(kind, *shape, 10.0, 7).values
    for k in range(ns // 2):
        p = sk.plan_sector(k, ns, *shape)
        pre = ora.apply_pre_ops(dem, k, ns)
        v, _w, rr, base = ora.build_skw(pre, p.shear_tan)
        g = sk.build_sector_sdem(dem, k, ns)
        assert g.base == base
        assert np.array_equal(g.row_ranges, rr), k
        assert np.array_equal(b32(g.values), b32(v)), k


def test_build_skw_arbitrary_shears(ora):
    rng = np.random.default_rng(99)
    g = (rng.standard_normal((37, 53)) * 100).astype(np.float32)
    g[3, 4] = -0.0
    g[5, :] = -2.5
    for t in [0.0, 1.0, 1e-7, 1 - 1e-7, 0.5, *rng.random(8)]:
        ours = sk.build_skw(g, float(t))
        v, _w, rr, base = ora.build_skw(g, float(t))
        assert ours.base == base
        assert np.array_equal(ours.row_ranges, rr)
        assert np.array_equal(b32(ours.values), b32(v))


def test_relocation_2000_sampled_sectors(ora):
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 2000, 2000, 10.0, 7).values
    for k in [0, 1, 22, 44, 45, 46, 67, 89]:
        p = sk.plan_sector(k, 180, 2000, 2000)
        pre = ora.apply_pre_ops(dem, k, 180)
        v, _w, rr, base = ora.build_skw(pre, p.shear_tan)
        g = sk.build_sector_sdem(dem, k, 180)
        assert np.array_equal(g.row_ranges, rr), k
        assert np.array_equal(b32(g.values), b32(v)), k


def test_config2_full_size_sectors_bitexact(ora):
    """P2 + P3 at the benchmark's own size: whole sectors of config 2
    (2000^2 fractal, ns = 180) — relocation, the scan of every POV in both
    directions, the fixup and the unskew — against the reference's
    sector_sweep, bit for bit. Four sectors (0, 22, 44 and 134 degrees: no
    shear, sheared, near 45, transposed + flipped) run on host threads in
    parallel (~30 s)."""
    from concurrent.futures import ThreadPoolExecutor

    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 2000, 2000, 10.0, 7)
    cfg = sk.RunConfig(ns=180, h0=1.5, units=sk.Units.SquareMeters)
    ks = [0, 11, 22, 67]
    with ThreadPoolExecutor(len(ks)) as ex:
        refs = list(ex.map(lambda k: ora.sector_sweep(dem.values, 10.0, 180, 1.5, None, k), ks))
    for k, ref in zip(ks, refs):
        ours = sk.sector_sweep(dem, cfg, k).contribution
        assert np.array_equal(b64(ours), b64(ref)), k


# ---- P2 scan -----------------------------------------------------------------

def _ref_sdem(ora, dem, k, ns):
    p = sk.plan_sector(k, ns, *dem.shape)
    pre = ora.apply_pre_ops(dem, k, ns)
    v, _w, rr, base = ora.build_skw(pre, p.shear_tan)
    return p, v, rr, base


@pytest.mark.parametrize("kind", [sk.SyntheticKind.SmoothedNoise, sk.SyntheticKind.Fractal,
                                  sk.SyntheticKind.Cone, sk.SyntheticKind.Ramp, sk.SyntheticKind.Flat])
@pytest.mark.parametrize("max_dd", [NO_CAP, 0, 1, 7])
def test_sector_viewshed_bitexact(ora, kind, max_dd):
    dem = sk.make_synthetic(kind, 48, 40, 10.0, 11).values
    for k in range(0, 18):
        p, v, rr, base = _ref_sdem(ora, dem, k, 36)
        ref = ora.sector_viewshed(v, rr, p.rows, base, p.shear_tan, 1.5, max_dd)
        skw = sk.SkwGrid(v, rr, base, p.rows, p.shear_tan)
        ours = sk.sector_viewshed(skw, 1.5, max_dd)
        assert np.array_equal(b64(ours), b64(ref)), (kind, max_dd, k)


@pytest.mark.parametrize("h0", [0.0, 1.5, 1.7, 30.0])
def test_sector_viewshed_observer_heights(ora, h0):
    # h0 = 0 on a ramp makes collinear targets exact ties (not visible,
    # scan.cpp:25); 1.7 is not a float, so the filter's exact-split check
    # routes those POVs to the FP64 fixup.
    for kind in (sk.SyntheticKind.Ramp, sk.SyntheticKind.Fractal, sk.SyntheticKind.Cone):
        dem = sk.make_synthetic(kind, 40, 40, 10.0, 3).values
        for k in (0, 5, 9, 13):
            p, v, rr, base = _ref_sdem(ora, dem, k, 36)
            ref = ora.sector_viewshed(v, rr, p.rows, base, p.shear_tan, h0)
            ours = sk.sector_viewshed(sk.SkwGrid(v, rr, base, p.rows, p.shear_tan), h0)
            assert np.array_equal(b64(ours), b64(ref)), (kind, k, h0)


def test_scan_long_rows_sampled_pov_parity(ora):
    """2000^2 fractal: full GPU sector scan vs the reference's own
    linear_viewshed_row on sampled POVs (both directions)."""
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 2000, 2000, 10.0, 7).values
    rng = np.random.default_rng(5)
    for k in (0, 17, 45, 71):
        p, v, rr, base = _ref_sdem(ora, dem, k, 180)
        _out, cvf, cvb = sk.sector_viewshed(sk.SkwGrid(v, rr, base, p.rows, p.shear_tan), 1.5,
                                            return_cv=True)
        rows = np.nonzero(rr[:, 1] - rr[:, 0] >= 2)[0]
        for q in rng.choice(rows, 40, replace=False):
            first, last = rr[q]
            for j0 in rng.integers(first, last, 12):
                h = float(v[q, j0]) + 1.5
                f = ora.linear_viewshed_row(v[q], first, last, j0, h, 0)
                b = ora.linear_viewshed_row(v[q], first, last, j0, h, 1)
                assert cvf[q, j0] == f and cvb[q, j0] == b, (k, q, j0)


def test_scan_very_long_rows_two_copy_tables(ora):
    """Rows of 7000 cells: beyond the 4-copy table layout, scan2 runs with 2
    fl(1/dd) copies (pair loads) and one row slot (config 5 path). Every POV
    of every row, both directions, against the reference, capped and not."""
    L = 7000
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 6, L, 10.0, 21).values
    vals = np.ascontiguousarray(dem, np.float32)
    rr = np.zeros((6, 2), np.int32)
    rr[:, 1] = L
    rr[3] = (5, L - 7)  # a ragged row
    for max_dd in (NO_CAP, 3001):
        ref = ora.sector_viewshed(vals, rr, 6, 0, 0.0, 1.5, max_dd)
        ours = sk.sector_viewshed(sk.SkwGrid(vals, rr, 0, 6, 0.0), 1.5, max_dd)
        assert np.array_equal(b64(ours), b64(ref)), max_dd


def test_visibility_vectors(ora):
    rng = np.random.default_rng(7)
    for trial in range(60):
        n = int(rng.integers(2, 300))
        kind = trial % 3
        if kind == 0:
            row = (rng.random(n) * 50).astype(np.float32)
        elif kind == 1:
            row = np.cumsum(rng.standard_normal(n)).astype(np.float32) + 500
        else:
            row = np.linspace(0, 1, n, dtype=np.float32)  # ramp: near ties
        first = int(rng.integers(0, n - 1))
        last = int(rng.integers(first + 1, n + 1))
        j0 = int(rng.integers(first, last))
        h = float(row[j0]) + [0.0, 1.5, 0.3][trial % 3]
        for d in (0, 1):
            for cap in (NO_CAP, int(rng.integers(0, 20))):
                cv, vis = sk.linear_viewshed_row(row, first, last, j0, h, d, cap, want_visible=True)
                rcv, rvis = ora.linear_viewshed_row(row, first, last, j0, h, d, cap, want_visible=True)
                assert cv == rcv
                assert np.array_equal(vis, rvis)


# ---- KATs from the reference's scan tests (test_scan.cpp) -------------------

def test_kat_flat_row():  # test_scan.cpp:48-53
    assert sk.linear_viewshed_row(np.zeros(5, np.float32), 0, 5, 0, 1.5, sk.ScanDir.Forward) == 24.0


def test_kat_single_target():  # :55-59
    assert sk.linear_viewshed_row(np.array([3, 17], np.float32), 0, 2, 0, 5.0, sk.ScanDir.Forward) == 3.0


def test_kat_near_wall():  # :61-67
    row = np.array([0, 5, 0, 0, 10, 0], np.float32)
    assert sk.linear_viewshed_row(row, 0, 6, 0, 1.0, sk.ScanDir.Forward) == 3.0


def test_kat_empty_range():  # :69-73
    row = np.zeros(3, np.float32)
    assert sk.linear_viewshed_row(row, 0, 1, 0, 1.5, sk.ScanDir.Forward) == 0.0
    assert sk.linear_viewshed_row(row, 2, 3, 2, 1.5, sk.ScanDir.Backward) == 0.0


def test_kat_reversal_symmetry():  # :75-90
    rng = np.random.default_rng(21)
    for _ in range(50):
        n = int(2 + rng.integers(0, 30))
        row = (rng.integers(0, 1000, n) / 10.0).astype(np.float32)
        j0 = int(rng.integers(0, n))
        h = float(row[j0]) + 1.5
        fwd = sk.linear_viewshed_row(row, 0, n, j0, h, sk.ScanDir.Forward)
        bwd = sk.linear_viewshed_row(row[::-1].copy(), 0, n, n - 1 - j0, h, sk.ScanDir.Backward)
        assert fwd == bwd


def test_kat_descending_all_visible():  # :92-102
    for L in (1, 4, 9):
        row = np.array([100.0 - 2.0 * k for k in range(L + 1)], np.float32)
        cv, vis = sk.linear_viewshed_row(row, 0, L + 1, 0, float(row[0]) + 1.5, sk.ScanDir.Forward,
                                         want_visible=True)
        assert cv == (L + 1) ** 2 - 1.0
        assert vis.tolist() == [1] * L


def test_kat_distance_cap():  # :145-150
    assert sk.linear_viewshed_row(np.zeros(11, np.float32), 0, 11, 0, 1.5, sk.ScanDir.Forward, 3) == 15.0


def test_kat_flat_zero_shear_formula():  # :152-164
    dem = sk.make_synthetic(sk.SyntheticKind.Flat, 5, 9, 10.0)
    vs = sk.sector_viewshed(sk.build_skw(dem.values, 0.0), 1.5)
    for i in range(5):
        for j0 in range(9):
            east, west = 9.0 - 1 - j0, j0
            assert vs[5 + i, j0] == (east + 1) ** 2 - 1 + (west + 1) ** 2 - 1


def test_kat_diagonal_factor_two():  # :166-181
    dem = sk.make_synthetic(sk.SyntheticKind.Flat, 4, 4, 10.0)
    skw = sk.build_skw(dem.values, 1.0)
    vs = sk.sector_viewshed(skw, 1.5)
    for q in range(skw.skw_rows()):
        first, last = skw.row_ranges[q]
        for j0 in range(first, last):
            east, west = last - 1 - j0, j0 - first
            assert vs[q, j0] == 2.0 * ((east + 1) ** 2 - 1 + (west + 1) ** 2 - 1)


def test_kat_outside_ranges_zero():  # :197-213
    dem = sk.make_synthetic(sk.SyntheticKind.SmoothedNoise, 12, 12, 10.0, 9)
    t = np.tan(np.deg2rad(20.0))
    skw = sk.build_skw(dem.values, float(t))
    vs = sk.sector_viewshed(skw, 1.5)
    for q in range(skw.skw_rows()):
        first, last = skw.row_ranges[q]
        for j in range(skw.cols):
            if j < first or j >= last:
                assert vs[q, j] == 0.0
            else:
                assert np.isfinite(vs[q, j]) and vs[q, j] >= 0.0


def test_acceptance_flat_scan_formula():  # acceptance_main.cpp:218-251 (criterion 4)
    n, ns = 33, 360
    dem = np.zeros((n, n), np.float32)
    scans = 0
    for k in range(ns // 2):
        g = sk.build_sector_sdem(dem, k, ns)
        _out, cvf, _cvb = sk.sector_viewshed(g, 1.5, return_cv=True)
        for q in range(g.skw_rows()):
            first, last = g.row_ranges[q]
            for j0 in range(first, last):
                L = last - 1 - j0
                assert cvf[q, j0] == (L + 1) ** 2 - 1
                scans += 1
    assert scans == 190388


# ---- P3 unskew -----------------------------------------------------------------

@pytest.mark.parametrize("shape,ns", [((48, 40), 36), ((40, 48), 36), ((32, 32), 360), ((2, 2), 8)])
def test_unskew_bitexact(ora, shape, ns):
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, *shape, 10.0, 5).values
    for k in range(ns // 2):
        p, v, rr, base = _ref_sdem(ora, dem, k, ns)
        vs = ora.sector_viewshed(v, rr, p.rows, base, p.shear_tan, 1.5)
        init = np.random.default_rng(k).random(shape)
        ref = ora.unskew_accumulate(vs, k, ns, *shape, out=init.copy())
        ours = init.copy()
        sk.unskew_accumulate(vs, p, ours)
        assert np.array_equal(b64(ours), b64(ref)), k


def test_round_trip_bitwise_integer_shears():  # test_skew.cpp:286-303
    dem = sk.make_synthetic(sk.SyntheticKind.SmoothedNoise, 16, 16, 10.0, 5)
    for k in (0, 45):
        p = sk.plan_sector(k, 360, 16, 16)
        g = sk.build_sector_sdem(dem.values, k, 360)
        out = np.zeros((16, 16))
        sk.unskew_accumulate(g.values.astype(np.float64), p, out)
        assert np.array_equal(out, dem.values.astype(np.float64))


def test_unskew_rejects_mismatched_shapes():
    p = sk.plan_sector(0, 360, 6, 6)
    with pytest.raises(ValueError):
        sk.unskew_accumulate(np.zeros((11, 6)), p, np.zeros((6, 6)))
    with pytest.raises(ValueError):
        sk.unskew_accumulate(np.zeros((12, 6)), p, np.zeros((5, 6)))


# ---- P4 end to end -------------------------------------------------------------

@pytest.mark.parametrize("shape,kind,ns,maxd", [
    ((48, 40), sk.SyntheticKind.SmoothedNoise, 36, None),
    ((40, 48), sk.SyntheticKind.Fractal, 36, None),
    ((64, 64), sk.SyntheticKind.Fractal, 180, 150.0),
    ((32, 32), sk.SyntheticKind.Cone, 90, None),
    ((24, 40), sk.SyntheticKind.Ramp, 2, None),
    ((2, 2), sk.SyntheticKind.SmoothedNoise, 8, None),
])
def test_total_viewshed_raw_bitexact(ora, shape, kind, ns, maxd):
    dem = sk.make_synthetic(kind, *shape, 10.0, 13)
    cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=maxd, units=sk.Units.SquareMeters)
    ours = sk.total_viewshed_raw(dem, cfg)
    ref = ora.total_viewshed(dem.values, 10.0, ns, 1.5, max_distance=maxd or 0.0, raw=True)
    assert np.array_equal(b64(ours), b64(ref))


@pytest.mark.parametrize("shape,kind,ns,maxd", [
    ((64, 48), sk.SyntheticKind.Fractal, 90, None),
    ((100, 60), sk.SyntheticKind.SmoothedNoise, 36, 300.0),
    ((36, 132), sk.SyntheticKind.Cone, 180, None),
    ((68, 36), sk.SyntheticKind.Fractal, 360, None),  # partial tiles on both axes
])
def test_unskew_tma_and_register_staged_bitexact(ora, shape, kind, ns, maxd, monkeypatch):
    """The TMA-staged unskew (DEM sides multiples of 4: one 2-D box per
    sector and tile, diagonal cell ownership) and the register-staged kernel
    (SKS_UNSKEW_TMA=0, also what odd sides take) both give the reference's
    map bit for bit."""
    dem = sk.make_synthetic(kind, *shape, 10.0, 21)
    cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=maxd, units=sk.Units.SquareMeters)
    ref = ora.total_viewshed(dem.values, 10.0, ns, 1.5, max_distance=maxd or 0.0, raw=True)
    ours = sk.total_viewshed_raw(dem, cfg)
    assert np.array_equal(b64(ours), b64(ref))
    monkeypatch.setenv("SKS_UNSKEW_TMA", "0")
    ctx = sk.Context(0)
    staged = ctx.total_viewshed(dem.values, 10.0, cfg, raw=True)
    ctx.close()
    assert np.array_equal(b64(staged), b64(ref))


@pytest.mark.parametrize("scale", [3.0e12, 2.0e-13])
def test_exact_path_outside_filter_range(ora, scale):
    """Elevations outside the FP32 filter's proven range [2^-40, 2^40]
     switch every POV to the FP64 path: still bit-exact,
    through the host entry point and through the device-pointer entry point
    (Context.run_sectors, the multi-GPU building block)."""
    import torch

    base = sk.make_synthetic(sk.SyntheticKind.Fractal, 30, 26, 10.0, 5).values
    vals = np.ascontiguousarray(base * np.float32(scale), np.float32)
    dem = sk.Dem(vals, 10.0)
    cfg = sk.RunConfig(ns=16, h0=0.0, units=sk.Units.SquareMeters)
    ref = ora.total_viewshed(vals, 10.0, 16, 0.0, raw=True)
    ours = sk.total_viewshed_raw(dem, cfg)
    assert np.array_equal(b64(ours), b64(ref))
    ctx = sk.Context(0)
    d_dem = torch.from_numpy(vals).cuda()
    d_map = torch.zeros(vals.shape, dtype=torch.float64, device="cuda")
    ctx.run_sectors(d_dem.data_ptr(), *vals.shape, 10.0, cfg, list(range(8)), d_map.data_ptr(),
                    stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(b64(d_map.cpu().numpy()), b64(ref))


def test_device_entry_rejects_non_finite():
    import torch

    vals = sk.make_synthetic(sk.SyntheticKind.Fractal, 20, 20, 10.0, 5).values.copy()
    vals[7, 11] = np.nan
    ctx = sk.Context(0)
    d_dem = torch.from_numpy(vals).cuda()
    d_map = torch.zeros(vals.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match=r"non-finite elevation at cell \(7, 11\)"):
        ctx.run_sectors(d_dem.data_ptr(), 20, 20, 10.0, sk.RunConfig(ns=8), [0, 1], d_map.data_ptr(),
                        stream=torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("shape", [(72, 60), (70, 61)])  # TMA-staged unskew / register-staged (odd side)
@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
def test_row_block_parts_sum_to_total(ora, nparts, shape):
    """Row-block sharding (the multi-GPU split): the nparts partial maps of
    Context.run_rows sum to the reference's total_viewshed_raw (per-cell sum
    order differs, so within 1e-12 relative; one part is bit-exact)."""
    import torch

    vals = sk.make_synthetic(sk.SyntheticKind.Fractal, *shape, 10.0, 9).values
    cfg = sk.RunConfig(ns=24, h0=1.5, units=sk.Units.SquareMeters)
    ref = ora.total_viewshed(vals, 10.0, 24, 1.5, raw=True)
    ctx = sk.Context(0)
    d_dem = torch.from_numpy(vals).cuda()
    total = np.zeros(vals.shape, np.float64)
    st = torch.cuda.current_stream().cuda_stream
    for part in range(nparts):
        d_map = torch.zeros(vals.shape, dtype=torch.float64, device="cuda")
        ctx.run_rows(d_dem.data_ptr(), *vals.shape, 10.0, cfg, part, nparts, d_map.data_ptr(), stream=st)
        torch.cuda.synchronize()
        total += d_map.cpu().numpy()
    if nparts == 1:
        assert np.array_equal(b64(total), b64(ref))
    else:
        np.testing.assert_allclose(total, ref, rtol=1e-12, atol=0)


@pytest.mark.parametrize("shape,kind,ns,maxd", [
    ((48, 40), sk.SyntheticKind.SmoothedNoise, 36, None),
    ((40, 48), sk.SyntheticKind.Fractal, 36, None),
    ((64, 64), sk.SyntheticKind.Fractal, 180, 150.0),
    ((24, 40), sk.SyntheticKind.Ramp, 2, None),
    ((2, 2), sk.SyntheticKind.SmoothedNoise, 8, None),
    ((33, 35), sk.SyntheticKind.Cone, 90, 10.0),  # a distance cap of 1 cell at most
])
def test_fused_relocation_bitexact(ora, shape, kind, ns, maxd, monkeypatch):
    """Relocation fused into scan2's row loader (SKS_FUSED=1, read when a
    context builds its batches): rows gathered from the DEM in the loader,
    the unskew reading only the ranges it wrote. Bit-exact like the default
    path, on one part and (to 1e-12) on row-block parts."""
    import torch

    monkeypatch.setenv("SKS_FUSED", "1")
    dem = sk.make_synthetic(kind, *shape, 10.0, 13)
    cfg = sk.RunConfig(ns=ns, h0=1.5, max_distance=maxd, units=sk.Units.SquareMeters)
    ref = ora.total_viewshed(dem.values, 10.0, ns, 1.5, max_distance=maxd or 0.0, raw=True)
    ctx = sk.Context(0)
    ours = ctx.total_viewshed(dem.values, 10.0, cfg, raw=True)
    assert np.array_equal(b64(ours), b64(ref))
    d_dem = torch.from_numpy(dem.values).cuda()
    total = np.zeros(shape, np.float64)
    for part in range(3):
        d_map = torch.zeros(shape, dtype=torch.float64, device="cuda")
        ctx.run_rows(d_dem.data_ptr(), *shape, 10.0, cfg, part, 3, d_map.data_ptr(),
                     stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        total += d_map.cpu().numpy()
    np.testing.assert_allclose(total, ref, rtol=1e-12, atol=0)
    ctx.close()


def test_row_block_cuts_sum_to_total(ora):
    """Row blocks placed by explicit cuts (the measured-time rebalancing
    path): any non-decreasing cuts partition every sector's rows, so the
    parts still sum to the total; bad cuts are rejected."""
    import torch

    vals = sk.make_synthetic(sk.SyntheticKind.Fractal, 60, 72, 10.0, 4).values
    cfg = sk.RunConfig(ns=24, h0=1.5, units=sk.Units.SquareMeters)
    ref = ora.total_viewshed(vals, 10.0, 24, 1.5, raw=True)
    ctx = sk.Context(0)
    d_dem = torch.from_numpy(vals).cuda()
    st = torch.cuda.current_stream().cuda_stream
    for cuts in ([0.0, 0.1, 0.75, 1.0], [0.0, 0.0, 0.5, 1.0], [0.0, 0.3, 0.3, 1.0]):
        total = np.zeros(vals.shape, np.float64)
        for part in range(3):
            d_map = torch.zeros(vals.shape, dtype=torch.float64, device="cuda")
            ctx.run_rows(d_dem.data_ptr(), *vals.shape, 10.0, cfg, part, 3, d_map.data_ptr(), stream=st, cuts=cuts)
            torch.cuda.synchronize()
            total += d_map.cpu().numpy()
        np.testing.assert_allclose(total, ref, rtol=1e-12, atol=0)
    d_map = torch.zeros(vals.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="non-decreasing"):
        ctx.run_rows(d_dem.data_ptr(), *vals.shape, 10.0, cfg, 0, 3, d_map.data_ptr(), stream=st,
                     cuts=[0.0, 0.6, 0.4, 1.0])


def test_row_blocks_balance_exact_work():
    """Every target of every sector is owned by exactly one part."""
    import torch

    vals = sk.make_synthetic(sk.SyntheticKind.Fractal, 300, 300, 10.0, 9).values
    cfg = sk.RunConfig(ns=36, h0=1.5)
    ctx = sk.Context(0)
    d_dem = torch.from_numpy(vals).cuda()
    d_map = torch.zeros(vals.shape, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    work = []
    for part in range(4):
        es = ctx.run_rows(d_dem.data_ptr(), 300, 300, 10.0, cfg, part, 4, d_map.data_ptr(), stream=st,
                          want_stats=True)
        work.append(es.target_evals)
    assert sum(work) == sk.total_target_evals(36, 300, 300, 10.0, None)
    # blocks balance exact work plus a per-task term (short rows cost more
    # per target), so the exact work alone is only roughly equal
    assert min(work) > 0 and max(work) / (sum(work) / 4) < 1.4, work


def test_total_viewshed_units_and_scale(ora):
    dem = sk.make_synthetic(sk.SyntheticKind.SmoothedNoise, 16, 16, 10.0, 1)
    for units in (sk.Units.SquareMeters, sk.Units.SquareKilometers):
        cfg = sk.RunConfig(ns=36, units=units)
        ours = sk.total_viewshed(dem, cfg)
        ref = ora.total_viewshed(dem.values, 10.0, 36, 1.5, units=int(units))
        assert ours.units == units
        assert np.array_equal(b64(ours.values), b64(ref))


def test_sector_sweep_bitexact(ora):
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 40, 40, 10.0, 5)
    cfg = sk.RunConfig(ns=180)
    for k in (0, 5, 45, 67, 89):
        ours = sk.sector_sweep(dem, cfg, k).contribution
        ref = ora.sector_sweep(dem.values, 10.0, 180, 1.5, 0.0, k)
        assert np.array_equal(b64(ours), b64(ref))


def test_config1_500_fractal_end_to_end(ora):
    """BASELINE config 1: 500^2 fractal, 180 sectors, h0 1.5, unlimited."""
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 500, 500, 10.0, 7)
    cfg = sk.RunConfig(ns=180, h0=1.5, units=sk.Units.SquareMeters)
    stats = sk.EngineStats()
    ours = sk.total_viewshed(dem, cfg, stats)
    ref = ora.total_viewshed(dem.values, 10.0, 180, 1.5)
    assert np.array_equal(b64(ours.values), b64(ref))
    assert stats.sectors == 90 and stats.kernel_launches > 0


def test_rejects_bad_inputs():
    dem = sk.make_synthetic(sk.SyntheticKind.Flat, 8, 8, 10.0)
    holed = sk.Dem(dem.values.copy(), 10.0, nodata=-9999.0)
    holed.values[3, 3] = -9999.0
    with pytest.raises(ValueError, match="nodata"):
        sk.total_viewshed(holed, sk.RunConfig())
    with pytest.raises(ValueError):
        sk.total_viewshed(dem, sk.RunConfig(ns=7))
    with pytest.raises(IndexError):
        sk.sector_sweep(dem, sk.RunConfig(), 180)
    bad = dem.values.copy()
    bad[1, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        sk.total_viewshed(sk.Dem(bad, 10.0), sk.RunConfig())


def test_progress_reports_every_sector_once_in_order():
    """engine.hpp:34-36 / test_engine.cpp "every sector is reported exactly
    once, in order": the callback runs once per sector, ascending, with the
    batched device time attributed by exact work (non-negative, summing to
    the phase total)."""
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 48, 40, 10.0, 2)
    cfg = sk.RunConfig(ns=36, h0=1.5)
    seen = []
    st = sk.EngineStats()
    sk.total_viewshed(dem, cfg, st, progress=lambda k, s: seen.append((k, s)))
    assert [k for k, _ in seen] == list(range(18))
    assert all(s >= 0.0 for _, s in seen)
    busy = st.skew_seconds + st.scan_seconds + st.fixup_seconds + st.unskew_seconds
    assert sum(s for _, s in seen) == pytest.approx(busy, rel=1e-9)


@pytest.mark.parametrize("maxd", [1000.0, 2410.0])
def test_long_capped_rows_packed_tail_bitexact(ora, maxd):
    """Distance caps long enough for the main loop, the hidden-window skip
    and the packed, NaN-masked tail windows of scan2 (config 3's regime:
    cap 100-241 cells on rows of ~300-420) — every POV bit-exact against the
    reference's sector_viewshed."""
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 300, 260, 10.0, 19).values
    for k in (0, 3, 5, 9):
        p, v, rr, base = _ref_sdem(ora, dem, k, 20)
        cap = sk.distance_cap_cells(maxd, p.shear_tan, 10.0)
        ref = ora.sector_viewshed(v, rr, p.rows, base, p.shear_tan, 1.5, cap)
        skw = sk.SkwGrid(v, rr, base, p.rows, p.shear_tan)
        ours = sk.sector_viewshed(skw, 1.5, cap)
        assert np.array_equal(b64(ours), b64(ref)), (k, cap)


@pytest.mark.parametrize("maxd", [None, 120.0])
def test_many_batches_bitexact(ora, maxd, monkeypatch):
    """A memory budget small enough to split the sectors into several
    batches (SKS_BATCH_GB, read when a context builds its plans): every batch
    runs relocate -> scan -> fixup -> unskew into the same map in ascending
    sector order, so the raw map is still bit-identical (configs 4-5 run in
    batches)."""
    monkeypatch.setenv("SKS_BATCH_GB", "0.0004")
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 56, 48, 10.0, 21)
    cfg = sk.RunConfig(ns=36, h0=1.5, max_distance=maxd, units=sk.Units.SquareMeters)
    ref = ora.total_viewshed(dem.values, 10.0, 36, 1.5, max_distance=maxd or 0.0, raw=True)
    ctx = sk.Context(0)
    ours, st = ctx.total_viewshed(dem.values, 10.0, cfg, raw=True, want_stats=True)
    assert st.batches > 3
    assert np.array_equal(b64(ours), b64(ref))
    ctx.close()
