"""Pins the CPU oracle (C restatement, oracle/skewshed_oracle.c).

1. Against the committed golden vectors (generated from the reference itself
   by tests/golden/make_golden.py) — runs everywhere.
2. Against the reference library itself (oracle/_ref) — bit for bit, over
   every sector of several geometries — where that library was built.
3. The reference's own known-answer tests (test_scan.cpp, test_skew.cpp,
   acceptance_main.cpp criteria 2-4) restated against both.
"""
import hashlib
import os

import numpy as np
import pytest

from _oracle import NO_CAP, Orc, Ref, have_orc, have_ref

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))

pytestmark = pytest.mark.skipif(not have_orc(), reason="oracle/liboracle.so not built")


@pytest.fixture(scope="module")
def orc():
    return Orc()


def oracles():
    out = [Orc()]
    if have_ref():
        out.append(Ref())
    return out


def b32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def b64(a):
    return np.ascontiguousarray(a).view(np.uint64)


# ---- golden vectors ----------------------------------------------------------

@pytest.mark.parametrize("name,kind", [("flat", 0), ("ramp", 1), ("cone", 2), ("smooth", 3)])
def test_golden_synthetic(orc, name, kind):
    assert np.array_equal(b32(orc.make_synthetic(kind, 17, 13, 7)), b32(GOLD[f"dem_{name}_17x13_s7"]))


def test_golden_plans(orc):
    for row in GOLD["plans_11x7"]:
        ns, k = int(row[0]), int(row[1])
        p = orc.plan_sector(k, ns, 11, 7)
        got = [p.sector_deg, p.shear_deg, p.shear_tan, p.rows, p.cols, *p.to_source, len(p.ops),
               *(list(p.ops) + [-1] * (3 - len(p.ops)))]
        assert np.array_equal(np.array(got, np.float64), row[2:]), (ns, k)


def test_golden_shear_params(orc):
    for t, j, d, f in GOLD["shear_params"]:
        assert orc.shear_params(float(t), int(j)) == (int(d), f)


def test_golden_build_skw(orc):
    grid = GOLD["skw_grid"]
    for i in range(4):
        t = float(GOLD[f"skw_{i}_t"][0])
        v, _w, rr, base = orc.build_skw(grid, t)
        assert base == int(GOLD[f"skw_{i}_base"][0])
        assert np.array_equal(rr, GOLD[f"skw_{i}_ranges"])
        assert np.array_equal(b32(v), b32(GOLD[f"skw_{i}_values"]))


def test_golden_linear_viewshed_row(orc):
    for row, meta, cv, vis in zip(GOLD["kat_rows"], GOLD["kat_meta"], GOLD["kat_cv"], GOLD["kat_vis"]):
        n, first, last, j0, h, d, cap = meta
        n = int(n)
        got, v = orc.linear_viewshed_row(row[:n], int(first), int(last), int(j0), float(h), int(d), int(cap),
                                         want_visible=True)
        assert got == cv
        assert np.array_equal(v, vis[: len(v)])


def test_golden_totals(orc):
    for i in range(5):
        dem = GOLD[f"total_{i}_dem"]
        ns, md = GOLD[f"total_{i}_cfg"]
        raw = orc.total_viewshed(dem, 10.0, int(ns), 1.5, max_distance=float(md), raw=True)
        assert np.array_equal(b64(raw), b64(GOLD[f"total_{i}_raw"])), i
        sw = orc.sector_sweep(dem, 10.0, int(ns), 1.5, float(md), min(3, int(ns) // 2 - 1))
        assert np.array_equal(b64(sw), b64(GOLD[f"total_{i}_sweep3"])), i


def test_golden_digest_64(orc):
    dem = orc.make_synthetic(3, 64, 64, 7)
    raw = orc.total_viewshed(dem, 10.0, 180, 1.5, raw=True)
    assert hashlib.sha256(raw.tobytes()).hexdigest() == str(GOLD["digest_64_smooth_ns180_raw"][0])


# ---- restatement vs the reference itself -------------------------------------

@pytest.mark.skipif(not have_ref(), reason="reference library not built here")
@pytest.mark.parametrize("shape,ns", [((48, 40), 36), ((40, 48), 36), ((16, 16), 180), ((5, 9), 8)])
def test_restatement_matches_reference_every_sector(shape, ns):
    r, o = Ref(), Orc()
    dem = r.make_synthetic(3, *shape, 11)
    dem = (dem * 50).astype(np.float32)
    for k in range(ns // 2):
        assert r.plan_sector(k, ns, *shape) == o.plan_sector(k, ns, *shape)
        pre = r.apply_pre_ops(dem, k, ns)
        assert np.array_equal(pre, o.apply_pre_ops(dem, k, ns))
        t = r.plan_sector(k, ns, *shape).shear_tan
        va, _wa, ra, ba = r.build_skw(pre, t)
        vb, _wb, rb, bb = o.build_skw(pre, t)
        assert ba == bb and np.array_equal(ra, rb) and np.array_equal(b32(va), b32(vb))
        for cap in (NO_CAP, 3):
            sa = r.sector_viewshed(va, ra, pre.shape[0], ba, t, 1.5, cap)
            sb = o.sector_viewshed(va, ra, pre.shape[0], ba, t, 1.5, cap)
            assert np.array_equal(b64(sa), b64(sb))
        ua = r.unskew_accumulate(sa, k, ns, *shape)
        ub = o.unskew_accumulate(sa, k, ns, *shape)
        assert np.array_equal(b64(ua), b64(ub))


@pytest.mark.skipif(not have_ref(), reason="reference library not built here")
def test_restatement_total_matches_reference():
    r, o = Ref(), Orc()
    for kind, shape, ns, md in [(3, (24, 40), 180, 0.0), (2, (33, 33), 36, 0.0), (3, (32, 32), 90, 50.0)]:
        dem = r.make_synthetic(kind, *shape, 9)
        a = r.total_viewshed(dem, 10.0, ns, 1.5, max_distance=md, raw=True)
        b = o.total_viewshed(dem, 10.0, ns, 1.5, max_distance=md, raw=True)
        assert np.array_equal(b64(a), b64(b))
        a = r.total_viewshed(dem, 10.0, ns, 1.5, max_distance=md, units=1)
        b = o.total_viewshed(dem, 10.0, ns, 1.5, max_distance=md, units=1)
        assert np.array_equal(b64(a), b64(b))


# ---- the reference's KATs, against both oracles ------------------------------

@pytest.mark.parametrize("ora", oracles(), ids=lambda o: o.name)
def test_kats(ora):
    assert ora.linear_viewshed_row(np.zeros(5, np.float32), 0, 5, 0, 1.5, 0) == 24.0
    assert ora.linear_viewshed_row(np.array([3, 17], np.float32), 0, 2, 0, 5.0, 0) == 3.0
    assert ora.linear_viewshed_row(np.array([0, 5, 0, 0, 10, 0], np.float32), 0, 6, 0, 1.0, 0) == 3.0
    assert ora.linear_viewshed_row(np.zeros(3, np.float32), 0, 1, 0, 1.5, 0) == 0.0
    assert ora.linear_viewshed_row(np.zeros(3, np.float32), 2, 3, 2, 1.5, 1) == 0.0
    assert ora.linear_viewshed_row(np.zeros(11, np.float32), 0, 11, 0, 1.5, 0, 3) == 15.0
    for L in (1, 4, 9):
        row = np.array([100.0 - 2.0 * k for k in range(L + 1)], np.float32)
        cv, vis = ora.linear_viewshed_row(row, 0, L + 1, 0, float(row[0]) + 1.5, 0, want_visible=True)
        assert cv == (L + 1) ** 2 - 1 and vis.tolist() == [1] * L


@pytest.mark.parametrize("ora", oracles(), ids=lambda o: o.name)
def test_ring_identity(ora):
    """cv = sum over visible targets of (2dd+1) (SURVEY §7 hard part 2)."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = int(rng.integers(2, 80))
        row = (rng.standard_normal(n) * rng.choice([0.01, 1.0, 100.0])).astype(np.float32)
        j0 = int(rng.integers(0, n))
        d = int(rng.integers(0, 2))
        cap = int(rng.choice([NO_CAP, 1, 5]))
        cv, vis = ora.linear_viewshed_row(row, 0, n, j0, float(row[j0]) + 1.5, d, cap, want_visible=True)
        assert cv == sum(2 * (i + 1) + 1 for i, v in enumerate(vis) if v)


@pytest.mark.parametrize("ora", oracles(), ids=lambda o: o.name)
def test_acceptance_mass_conservation(ora):  # acceptance_main.cpp:114-136 (criterion 2)
    dem = ora.make_synthetic(3, 64, 64, 7)
    src = float(np.sum(dem.astype(np.float64)))
    worst = 0.0
    for a in range(16):
        t = 1.0 if a == 15 else float(np.tan(np.deg2rad(45.0 * a / 15.0)))
        v, _w, _rr, _b = ora.build_skw(dem, t)
        worst = max(worst, abs(float(np.sum(v.astype(np.float64))) - src) / src)
    assert worst <= 1e-6


@pytest.mark.parametrize("ora", oracles(), ids=lambda o: o.name)
def test_acceptance_round_trip_integer_shears(ora):  # acceptance_main.cpp:140-172 (criterion 3)
    n = 32
    dem = ora.make_synthetic(3, n, n, 7)
    for k in (0, 45):
        p = ora.plan_sector(k, 360, n, n)
        pre = ora.apply_pre_ops(dem, k, 360)
        v, _w, _rr, _b = ora.build_skw(pre, p.shear_tan)
        back = ora.unskew_accumulate(v.astype(np.float64), k, 360, n, n)
        assert np.array_equal(back, dem.astype(np.float64))


@pytest.mark.parametrize("ora", oracles(), ids=lambda o: o.name)
def test_acceptance_flat_forward_scans(ora):  # acceptance_main.cpp:218-251 (criterion 4), subset
    n, ns = 33, 360
    dem = np.zeros((n, n), np.float32)
    for k in range(0, ns // 2, 7):
        p = ora.plan_sector(k, ns, n, n)
        v, _w, rr, _b = ora.build_skw(ora.apply_pre_ops(dem, k, ns), p.shear_tan)
        for q in range(0, v.shape[0], 3):
            first, last = rr[q]
            for j0 in range(first, last):
                L = last - 1 - j0
                assert ora.linear_viewshed_row(v[q], first, last, j0, 1.5, 0) == (L + 1) ** 2 - 1


# ---- bench inputs and work counts of the reference arm ------------------------------

@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("shape,seed", [((2, 2), 0), ((33, 17), 7), ((500, 500), 7), ((129, 300), 3)])
def test_reference_arm_fractal_matches_product(shape, seed):
    """bench.py's reference arm builds the fractal DEM with the shim's
    restatement (so it never loads the product library); it must be the same
    float grid the GPU arm consumes."""
    import paper_2003_02200_b200 as sk

    ours = sk.make_synthetic(sk.SyntheticKind.Fractal, *shape, 10.0, seed).values
    theirs = Ref().make_fractal(*shape, seed)
    assert np.array_equal(b32(ours), b32(theirs))


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("dims,ns,maxd", [((120, 90), 36, None), ((64, 64), 360, 150.0), ((40, 70), 8, 25.0)])
def test_reference_work_count_matches_plan(dims, ns, maxd):
    """The reference arm counts scan work from the reference's own build_skw
    row ranges; the GPU arm from its host plan. Same numbers, every sector."""
    import paper_2003_02200_b200 as sk

    ref = Ref()
    for k in range(ns // 2):
        assert ref.sector_work(*dims, 10.0, ns, k, maxd) == sk.sector_target_evals(k, ns, *dims, 10.0, maxd)
