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
