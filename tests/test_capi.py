"""The C ABI boundary: the library loads, exports exactly what
include/skewshed_b200.h declares, maps errors to status codes without
crashing, and compute entry points fail loudly (never fall back to a CPU
path) when no GPU is present."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import paper_2003_02200_b200 as sk
from paper_2003_02200_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_from_tree():
    assert os.path.dirname(_lib.LIB_PATH) == os.path.join(ROOT, "paper_2003_02200_b200")
    assert "sm_100a" in _lib.lib.sks_version().decode()


def test_exports_every_header_symbol():
    declared = _lib.header_symbols()
    assert len(declared) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # and every declared symbol has a ctypes signature in the binding
    assert set(declared) == set(_lib.SIGNATURES)


def test_no_torch_types_in_header():
    import re
    text = open(os.path.join(ROOT, "include", "skewshed_b200.h")).read()
    code = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    assert "torch" not in code and "at::" not in code and "std::" not in code


def test_status_codes_and_last_error():
    p = _lib.SectorPlanC()
    assert _lib.lib.sks_plan_sector(5, 8, 4, 4, C.byref(p)) == _lib.SKS_OUT_OF_RANGE
    assert "out of range" in _lib.last_error()
    assert _lib.lib.sks_plan_sector(0, 7, 4, 4, C.byref(p)) == _lib.SKS_INVALID_ARGUMENT
    assert _lib.lib.sks_plan_sector(0, 8, 4, 4, C.byref(p)) == _lib.SKS_OK
    assert _lib.last_error() == ""
    assert _lib.lib.sks_plan_sector(0, 8, 4, 4, None) == _lib.SKS_INVALID_ARGUMENT


@pytest.mark.skipif(sk.device_count() > 0, reason="checks the no-GPU behaviour")
def test_compute_without_gpu_fails_loudly():
    dem = sk.make_synthetic(sk.SyntheticKind.Flat, 8, 8, 10.0)
    with pytest.raises(RuntimeError, match="(?i)cuda"):
        sk.total_viewshed(dem, sk.RunConfig(ns=8))
    with pytest.raises(RuntimeError):
        sk.build_skw(dem.values, 0.5)
    with pytest.raises(RuntimeError):
        sk.Context(0)


def test_invalid_inputs_rejected_before_device_work():
    dem = sk.make_synthetic(sk.SyntheticKind.Flat, 8, 8, 10.0)
    with pytest.raises(ValueError):
        sk.total_viewshed(dem, sk.RunConfig(ns=7))
    nan = dem.values.copy()
    nan[3, 3] = np.nan
    with pytest.raises(ValueError):
        sk.total_viewshed(sk.Dem(nan, 10.0), sk.RunConfig(ns=8))
    with pytest.raises(IndexError):
        sk.sector_sweep(dem, sk.RunConfig(ns=8), 4)


def test_cpp_facade_header_compiles(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "skewshed_b200.hpp"\nint main(){ skewshed_b200::RunConfig c; return c.ns == 360 ? 0 : 1; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_cpp_facade_ascii_grid_round_trip(tmp_path):
    """The C++ facade's read/write_ascii_grid (ascii_grid.hpp:20-31) linked
    against the shipped library: host-only entry points, no GPU needed."""
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include "skewshed_b200.hpp"
#include <cstdio>
#include <sstream>
namespace sk = skewshed_b200;
int main(int, char** argv) {
  std::istringstream in("ncols 3\nnrows 2\nxllcorner 5\nyllcorner 6\ncellsize 2.5\nNODATA_value -1\n1 2 3\n4 -1 6\n");
  sk::Dem d = sk::read_ascii_grid(in, "mem");
  if (d.dimy() != 2 || d.dimx() != 3 || d.values(1, 2) != 6.0f || !d.nodata || *d.nodata != -1.0f) return 1;
  if (d.origin.easting != 5.0 || d.origin.northing != 6.0 || d.cellsize != 2.5) return 2;
  sk::write_ascii_grid(d, argv[1]);
  sk::Dem e = sk::read_ascii_grid(argv[1]);
  if (!(e.values == d.values) || e.origin.northing != 6.0) return 3;
  std::istringstream bad("ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\n1 2\n3 q\n");
  try { sk::read_ascii_grid(bad, "bad"); return 4; }
  catch (const sk::GridFormatError& ex) { std::puts(ex.what()); }
  sk::VsGrid vs{sk::Grid<double>(2, 3, 1.5e6), sk::Units::SquareMeters};
  sk::write_ascii_grid(vs, sk::Units::SquareKilometers, 2.5, d.origin, argv[2]);
  return 0;
}
''')
    exe = tmp_path / "t"
    libdir = os.path.join(ROOT, "paper_2003_02200_b200")
    r = subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                        "-L", libdir, "-lskewshed_b200", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe), str(tmp_path / "d.asc"), str(tmp_path / "v.asc")], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stderr)
    assert r.stdout.strip() == "bad:7:3: expected a number for cell value, got 'q'"
    assert (tmp_path / "v.asc").read_text().splitlines()[-1] == "1.5 1.5 1.5"


def test_bench_report_format_matches_reference_layout():
    """make/format_bench_report (bench.cpp:8-52): same keys, order and %.17g."""
    st = sk.EngineStats()
    st.skew_seconds, st.scan_seconds, st.fixup_seconds, st.unskew_seconds = 0.001, 0.06, 0.002, 0.0015
    st.total_seconds = 0.07
    cfg = sk.RunConfig(ns=180)
    r = sk.make_bench_report("dem.asc", 2000, 2000, cfg, st, baseline_total_seconds=70.0)
    text = sk.format_bench_report(r)
    keys = [ln.split(":")[0] for ln in text.splitlines()]
    assert keys == ["dataset", "dimy", "dimx", "ns", "workers", "skew_seconds", "scan_seconds", "unskew_seconds",
                    "reduce_seconds", "total_seconds", "povs_per_second", "speedup"]
    assert "scan_seconds: 0.062000000000000000" not in text and "scan_seconds: %.17g" % 0.062 in text
    assert "povs_per_second: %.17g" % (2000.0 * 2000.0 * 90 / 0.062) in text
    assert text.endswith("speedup: %.17g\n" % (70.0 / 0.07))
    assert "speedup" not in sk.format_bench_report(sk.make_bench_report("x", 2, 2, cfg, st))
    # stats without a total (per-part runs): C++'s division gives inf, no exception
    st.total_seconds = 0.0
    assert sk.make_bench_report("x", 2, 2, cfg, st, baseline_total_seconds=1.0).speedup == float("inf")


def test_cpp_facade_host_utilities(tmp_path):
    """The facade's host-side pieces of the reference API, linked against the
    shipped library: oracle::select_axis_point_set, fill_nodata_nearest,
    write_heatmap, bench report (no GPU needed)."""
    src = tmp_path / "u.cpp"
    src.write_text(r'''
#include "skewshed_b200.hpp"
#include <cstdio>
namespace sk = skewshed_b200;
int main(int, char** argv) {
  sk::Dem d;
  d.values.reset(6, 9, 2.0f);
  d.cellsize = 10.0;
  auto pts = sk::oracle::select_axis_point_set(d, 2, 3, 0.0);  // eastward: (2,4) .. (2,8)
  if (pts.size() != 5 || pts[0].i != 2 || pts[0].j != 4 || pts[4].j != 8) return 1;
  d.nodata = -1.0f;
  d.values(0, 0) = -1.0f;
  sk::Dem f = sk::fill_nodata_nearest(d);
  if (f.nodata || f.values(0, 0) != 2.0f) return 2;
  sk::VsGrid vs{sk::Grid<double>(2, 2, 0.0), sk::Units::SquareMeters};
  vs.values(1, 1) = 4.0;
  sk::write_heatmap(vs, argv[1], sk::Palette::Gray);
  sk::EngineStats st;
  st.scan_seconds = 0.5;
  st.total_seconds = 1.0;
  std::fputs(sk::format_bench_report(sk::make_bench_report("d", 2, 2, sk::RunConfig{}, st)).c_str(), stdout);
  return 0;
}
''')
    exe = tmp_path / "u"
    libdir = os.path.join(ROOT, "paper_2003_02200_b200")
    r = subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                        "-L", libdir, "-lskewshed_b200", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe), str(tmp_path / "h.pgm")], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stderr)
    assert (tmp_path / "h.pgm").read_bytes() == b"P5\n2 2\n255\n\x00\x00\x00\xff"
    assert "povs_per_second: 1440\n" in r.stdout


@pytest.mark.gpu
def test_cpp_facade_reference_style_engine_test(tmp_path):
    """test_engine.cpp:93-106 ("per-sector sweeps reduce to exactly the engine
    accumulator") and :231-241 (units) written as a C++ program against the
    facade, run on the GPU."""
    src = tmp_path / "e.cpp"
    src.write_text(r'''
#include "skewshed_b200.hpp"
namespace sk = skewshed_b200;
int main() {
  sk::Dem dem = sk::make_synthetic(sk::SyntheticKind::SmoothedNoise, 40, 56, 10.0, 3);
  sk::RunConfig cfg;
  cfg.ns = 24;
  cfg.units = sk::Units::SquareMeters;
  sk::Grid<double> raw = sk::total_viewshed_raw(dem, cfg);
  sk::Grid<double> acc(40, 56, 0.0);
  for (int k = 0; k < cfg.ns / 2; ++k) sk::accumulate_into(acc, sk::sector_sweep(dem, cfg, k).contribution);
  if (!(acc == raw)) return 1;
  sk::VsGrid m2 = sk::total_viewshed(dem, cfg);
  cfg.units = sk::Units::SquareKilometers;
  sk::VsGrid km2 = sk::total_viewshed(dem, cfg);
  for (size_t n = 0; n < m2.values.size(); ++n) {
    if (km2.values.data()[n] != m2.values.data()[n] * 1e-6 &&
        std::abs(km2.values.data()[n] - m2.values.data()[n] * 1e-6) > 1e-15 * m2.values.data()[n]) return 2;
  }
  return 0;
}
''')
    exe = tmp_path / "e"
    libdir = os.path.join(ROOT, "paper_2003_02200_b200")
    r = subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                        "-L", libdir, "-lskewshed_b200", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stderr)
