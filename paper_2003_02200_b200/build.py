"""Builds the in-tree native library libskewshed_b200.so (sm_100a).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU
container and the resulting .so travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libskewshed_b200.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++20",
    "--fmad=false",               # no FMA contraction anywhere (explicit __fmaf_rn only)
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
]


# host-only C++ (planning, I/O, the multi-GPU orchestration): same IEEE
# rules as the device code (no FMA contraction)
CXX_FLAGS = [
    "-std=c++20", "-O3", "-g", "-fPIC", "-ffp-contract=off",
    "-I", "/usr/local/cuda/include",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps += glob.glob(os.path.join(ROOT, "include", "*.h*"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Builds LIB (or, for kernel-variant experiments, `out` with extra -D defines)."""
    lib = out or LIB
    if not force and not defines and out is None and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "_obj" + ("_" + "_".join(d.replace("=", "") for d in defines) if defines else ""))
    os.makedirs(objdir, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        dflags = [f"-D{d}" for d in defines]
        cmd = ["nvcc", *NVCC_FLAGS, *dflags, "-c", src, "-o", obj]
        if src.endswith(".cpp"):  # host-only sources: the host compiler directly
            cmd = ["g++", *CXX_FLAGS, *dflags, "-c", src, "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, sources()))
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-o", tmp, *objs, "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-D", action="append", default=[], help="extra define (variant builds)")
    ap.add_argument("--out", default=None, help="output .so (variant builds)")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, defines=a.D, out=a.out))
