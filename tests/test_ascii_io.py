"""ESRI ASCII grid I/O (the DEM load / map output entry points) against the
reference's own reader and writers (oracle/_ref, ascii_grid.cpp), on CPU:
the same grids, the same GridFormatError messages (source:line:col), the
same bytes written. Cases mirror tests/test_io.cpp:52-200 of the reference."""
import ctypes as C
import os
import random

import numpy as np
import pytest

import paper_2003_02200_b200 as sk
from _oracle import have_ref

pytestmark = pytest.mark.skipif(not have_ref(), reason="needs oracle/_ref (built from /root/reference)")


def _ref():
    from _oracle import Ref
    r = Ref()
    lib = r.lib
    lib.ref_parse_ascii_grid.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_float), C.c_void_p,
                                         C.c_longlong]
    lib.ref_write_ascii_grid_dem.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                             C.c_double, C.c_int, C.c_float]
    lib.ref_write_ascii_grid_vs.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                            C.c_double, C.c_double]
    return lib


def ref_parse(lib, text: bytes, source="<test>"):
    """(dem-like tuple) or ('error', message)."""
    nr, nc, hn = C.c_int(), C.c_int(), C.c_int()
    nod = C.c_float()
    hdr = np.zeros(3, np.float64)
    rc = lib.ref_parse_ascii_grid(text, len(text), source.encode(), C.byref(nr), C.byref(nc), hdr.ctypes.data,
                                  C.byref(hn), C.byref(nod), None, 0)
    if rc == 3:
        return ("error", lib.ref_last_error().decode())
    assert rc == 0, lib.ref_last_error()
    vals = np.empty((nr.value, nc.value), np.float32)
    lib.ref_parse_ascii_grid(text, len(text), source.encode(), C.byref(nr), C.byref(nc), hdr.ctypes.data,
                             C.byref(hn), C.byref(nod), vals.ctypes.data, vals.size)
    return (vals, float(hdr[2]), (float(hdr[0]), float(hdr[1])), float(nod.value) if hn.value else None)


def ours_parse(text: bytes, source="<test>"):
    try:
        d = sk.parse_ascii_grid(text, source)
    except sk.GridFormatError as e:
        return ("error", str(e))
    return (d.values, d.cellsize, (d.origin.easting, d.origin.northing), d.nodata)


def is_err(r):
    return isinstance(r[0], str)


def same(a, b):
    if is_err(a) or is_err(b):
        return is_err(a) and is_err(b) and a[1] == b[1]
    nod = lambda x: None if x is None else np.float32(x).view(np.uint32)  # NaN nodata compares by bits
    return (np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32)) and a[1] == b[1] and a[2] == b[2]
            and nod(a[3]) == nod(b[3]))


CASES = [
    b"ncols 2\nnrows 2\nxllcorner 482500\nyllcorner 5634200\ncellsize 10\n1 2\n3 4\n",
    b"NCOLS 2\nNROWS 2\nXLLCORNER 0\nYLLCORNER 0\nCELLSIZE 5\nnodata_value -9999\n-9999 1\n2 3\n",
    b"",
    b"ncols 4\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2 3 4\n",
    b"nrows 2\nncols 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2 3 4\n",
    b"ncols abc\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2\n3 4\n",
    b"ncols 2.5\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2\n3 4\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 0\n1 2\n3 4\n",
    b"ncols 5\nnrows 1\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2 3 4 5\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2 3\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2 3 4 5\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2\n3 x\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value oops\n1 2\n3 4\n",
    b"ncols 1000000\nnrows 1000000\nxllcorner 0\nyllcorner 0\ncellsize 10\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize inf\n1 2\n3 4\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 nan\n3 4\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value nan\n1 2\n3 4",
    b"ncols 2\r\nnrows 2\r\nxllcorner 0\r\nyllcorner 0\r\ncellsize 10\r\n1 2\r\n3 +4\r\n",
    b"ncols 2 nrows 2 xllcorner -1e3 yllcorner 1e-3 cellsize 0.5 1e39 -1e-50 3.5 4",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\nNODATA_value\n",
    b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2\n3 4\n\n\n  5 \n",
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_corpus_same_result_and_message(i):
    lib = _ref()
    a, b = ref_parse(lib, CASES[i]), ours_parse(CASES[i])
    assert same(a, b), (CASES[i], a if is_err(a) else "ok", b if is_err(b) else "ok")


def test_cell_diagnostic_line_and_column():  # test_io.cpp:131-139
    r = ours_parse(b"ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n1 2\n3 x\n")
    assert is_err(r) and "7:3" in r[1]


def test_byte_soup_agrees_with_reference():  # test_io.cpp:114-129, more trials
    lib = _ref()
    rng = random.Random(123)
    alphabet = b"0123456789.eE+-\n\t ncolsrwxy_NODATA"
    headers = [b"", b"ncols 3\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 10\n",
               b"ncols 2 nrows 2 xllcorner 0 yllcorner 0 cellsize 1 NODATA_value -1\n"]
    for trial in range(1500):
        body = bytes(rng.choice(alphabet) for _ in range(rng.randrange(200)))
        text = headers[trial % 3] + body
        a, b = ref_parse(lib, text), ours_parse(text)
        assert same(a, b), (text, a, b)


def test_large_grid_parallel_parse_bit_exact(tmp_path):
    """A grid big enough for the multi-threaded body parser (several MB of
    text, values written with varied formats) reads exactly as the
    reference reads it."""
    lib = _ref()
    rng = np.random.default_rng(7)
    nr, nc = 700, 900
    v = (rng.standard_normal((nr, nc)) * 400 + 300).astype(np.float64)
    fmts = ["%.9g", "%.3f", "%.17g", "%g", "%.2e"]
    lines = [f"ncols {nc}", f"nrows {nr}", "xllcorner 12.5", "yllcorner -7", "cellsize 30", "NODATA_value -9999"]
    for i in range(nr):
        f = fmts[i % len(fmts)]
        lines.append(("\t " if i % 7 == 0 else " ").join(f % x for x in v[i]))
    text = ("\n".join(lines) + "\n").encode()
    a, b = ref_parse(lib, text, "big.asc"), ours_parse(text, "big.asc")
    assert same(a, b)
    # and an error deep in the body is located exactly as the reference does
    bad = text[:len(text) * 3 // 4] + b" 12x " + text[len(text) * 3 // 4:]
    a, b = ref_parse(lib, bad, "big.asc"), ours_parse(bad, "big.asc")
    assert is_err(a) and same(a, b), (a, b)


def test_file_entry_points_and_writers_match_reference_bytes(tmp_path):
    lib = _ref()
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 37, 53, 10.0, 3)
    dem.values[3, 4] = -9999.0
    dem = sk.Dem(dem.values, 12.5, -9999.0, sk.GridOrigin(482500.25, 5634200.125))
    ours = tmp_path / "ours.asc"
    ref = tmp_path / "ref.asc"
    sk.write_ascii_grid(dem, ours)
    assert lib.ref_write_ascii_grid_dem(str(ref).encode(), dem.values.ctypes.data, 37, 53, 482500.25,
                                        5634200.125, 12.5, 1, -9999.0) == 0
    assert ours.read_bytes() == ref.read_bytes()
    back = sk.read_ascii_grid(ours)  # round trip bit for bit (test_io.cpp:152-164)
    assert np.array_equal(back.values.view(np.uint32), dem.values.view(np.uint32))
    assert back.nodata == -9999.0 and back.cellsize == 12.5 and back.origin == dem.origin
    # viewshed maps, both unit conversions (test_io.cpp:166-200)
    vs = np.random.default_rng(1).random((37, 53)) * 1e6
    for uin, uout in ((0, 0), (0, 1), (1, 0), (1, 1)):
        o2, r2 = tmp_path / f"o{uin}{uout}.asc", tmp_path / f"r{uin}{uout}.asc"
        sk.write_ascii_grid(sk.VsGrid(vs, sk.Units(uin)), o2, units=sk.Units(uout), cellsize=10.0,
                            origin=sk.GridOrigin(1.0, 2.0))
        assert lib.ref_write_ascii_grid_vs(str(r2).encode(), vs.ctypes.data, 37, 53, uin, uout, 10.0, 1.0, 2.0) == 0
        assert o2.read_bytes() == r2.read_bytes(), (uin, uout)
    with pytest.raises(sk.GridFormatError, match="cannot open"):
        sk.read_ascii_grid(tmp_path / "missing.asc")


def test_writers_special_values_match_reference_bytes(tmp_path):
    """to_chars(general) must print exactly like the reference's %.9g / %.10g:
    signed zeros, subnormals, huge values, inf and nan."""
    lib = _ref()
    v = np.array([[0.0, -0.0, 1e-45, -3.4e38], [np.inf, -np.inf, np.nan, 123456789.0],
                  [1.0 / 3.0, 2.5e-7, 1e15, -7.0]], np.float32)
    ours, ref = tmp_path / "o.asc", tmp_path / "r.asc"
    sk.write_ascii_grid(sk.Dem(v, 1.0), ours)
    assert lib.ref_write_ascii_grid_dem(str(ref).encode(), v.ctypes.data, 3, 4, 0.0, 0.0, 1.0, 0, 0.0) == 0
    assert ours.read_bytes() == ref.read_bytes()
    d = np.array([[0.0, -0.0, 5e-324, 1.7976931348623157e308], [np.inf, -np.nan, 0.1, 1e21]], np.float64)
    sk.write_ascii_grid(sk.VsGrid(d, sk.Units.SquareMeters), ours, cellsize=1.0)
    assert lib.ref_write_ascii_grid_vs(str(ref).encode(), d.ctypes.data, 2, 4, 0, 0, 1.0, 0.0, 0.0) == 0
    assert ours.read_bytes() == ref.read_bytes()


# ---- binary side format (ESRI .hdr + .flt float32) -------------------------

def test_float_grid_round_trip_and_equals_ascii(tmp_path):
    dem = sk.make_synthetic(sk.SyntheticKind.Fractal, 41, 29, 10.0, 5)
    v = dem.values.copy()
    v[0, 0], v[1, 1], v[2, 2] = -0.0, np.float32(1e-45), -9999.0
    dem = sk.Dem(v, 12.5, -9999.0, sk.GridOrigin(482500.25, 5634200.125))
    sk.write_float_grid(dem, tmp_path / "d.flt")
    assert (tmp_path / "d.hdr").exists()
    for name in ("d.flt", "d.hdr", "d"):
        back = sk.read_float_grid(tmp_path / name)
        assert np.array_equal(back.values.view(np.uint32), v.view(np.uint32))
        assert back.cellsize == 12.5 and back.nodata == -9999.0 and back.origin == dem.origin
    sk.write_ascii_grid(dem, tmp_path / "d.asc")
    asc = sk.read_ascii_grid(tmp_path / "d.asc")
    assert np.array_equal(asc.values.view(np.uint32), sk.read_float_grid(tmp_path / "d").values.view(np.uint32))


def test_float_grid_big_endian_and_cell_centres(tmp_path):
    v = np.arange(12, dtype=np.float32).reshape(3, 4) * np.float32(1.5) - 4
    (tmp_path / "b.hdr").write_text("NCOLS 4\nNROWS 3\nXLLCENTER 5\nYLLCENTER 7\nCELLSIZE 2\nBYTEORDER MSBFIRST\n")
    (tmp_path / "b.flt").write_bytes(v.astype(">f4").tobytes())
    g = sk.read_float_grid(tmp_path / "b.flt")
    assert np.array_equal(g.values, v) and g.nodata is None
    assert g.origin == sk.GridOrigin(4.0, 6.0)  # half a cell to the corner


@pytest.mark.parametrize("hdr,flt_bytes,msg", [
    ("ncols 4\nnrows 3\nxllcorner 0\nyllcorner 0\ncellsize 2\n", 40, "expected 48 bytes of float32 cells for 3x4, got fewer"),
    ("ncols 4\nnrows 3\nxllcorner 0\nyllcorner 0\ncellsize 2\n", 52, "got more"),
    ("ncols 4\nnrows 3\nxllcorner 0\nyllcorner 0\n", 48, "missing header key 'cellsize'"),
    ("ncols 4\nnrows x\nxllcorner 0\nyllcorner 0\ncellsize 2\n", 48, "b.hdr:2:7: expected a positive integer for 'nrows'"),
    ("ncols 4\nnrows 3\nxllcorner 0\nyllcorner 0\ncellsize 0\n", 48, "cellsize must be a positive finite number"),
    ("ncols 4\nnrows 3\nxllcorner 0\nyllcorner 0\ncellsize 2\nbyteorder VAX\n", 48, "byteorder must be"),
    ("ncols 4\nnrows 3\nxllcorner 0\nyllcorner 0\ncellsize 2\nlayout bil\n", 48, "b.hdr:6:1: unknown header key 'layout'"),
    ("ncols 4\nnrows 3\nxllcorner 0\nyllcorner 0\ncellsize\n", 48, "missing value for header key 'cellsize'"),
])
def test_float_grid_errors(tmp_path, hdr, flt_bytes, msg):
    (tmp_path / "b.hdr").write_text(hdr)
    (tmp_path / "b.flt").write_bytes(b"\0" * flt_bytes)
    with pytest.raises(sk.GridFormatError, match=msg):
        sk.read_float_grid(tmp_path / "b")
    with pytest.raises(sk.GridFormatError, match="cannot open"):
        sk.read_float_grid(tmp_path / "nope.flt")


# ---- nodata fill (dem.cpp:175-213; the CLI's `fill`, cli.cpp:278-284) ------

def test_fill_nodata_nearest_matches_reference_bits():
    from _oracle import Ref
    ref = Ref()
    rng = np.random.default_rng(4)
    for shape, frac in (((40, 56), 0.3), ((7, 3), 0.8), ((1, 9), 0.5), ((64, 64), 0.02)):
        v = (rng.standard_normal(shape) * 50).astype(np.float32)
        v[rng.random(shape) < frac] = -9999.0
        if np.all(v == -9999.0):
            v[0, 0] = 1.0
        dem = sk.Dem(v, 10.0, -9999.0)
        got = sk.fill_nodata_nearest(dem)
        assert got.nodata is None and not np.any(got.values == -9999.0)
        assert np.array_equal(got.values.view(np.uint32), ref.fill_nodata_nearest(v, -9999.0).view(np.uint32))
    # NaN nodata never equals itself: nothing is filled, as in the reference
    w = np.array([[1.0, np.nan], [2.0, 3.0]], np.float32)
    assert np.array_equal(sk.fill_nodata_nearest(sk.Dem(w, 1.0, float("nan"))).values, w, equal_nan=True)
    with pytest.raises(RuntimeError, match="entirely nodata"):
        sk.fill_nodata_nearest(sk.Dem(np.full((3, 3), -1.0, np.float32), 1.0, -1.0))
