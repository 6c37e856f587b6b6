"""Build the in-tree C-ABI shared library `libhogbatch_b200.so` for sm_100a.

    python -m paper_2004_08771_b200.build [--force] [--verbose]

Plain nvcc, no torch extension machinery: the library is a C ABI over CUDA
(include/hogbatch_b200.h) that ctypes (or cgo/JNI) binds.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libhogbatch_b200.so"
SOURCES = [CSRC / "hb_capi.cu", CSRC / "hb_libsvm.cpp"]
HEADERS = sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "hogbatch_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    # host-side float64 merges must round like NumPy (no FMA contraction)
    "-Xcompiler", "-ffp-contract=off",
    "--expt-relaxed-constexpr",
    # IEEE exp/div and denormals: sigmoid(-100) must stay a positive denormal
    # (pkg/tests/test_linalg.py:67-70), so no --use_fast_math / FTZ.
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found (set NVCC or install the CUDA toolkit)")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, defines=(), out=None) -> Path:
    """Compile the library; `defines` (e.g. ["HB_SPLIT_WARPS=8"]) and `out`
    build experimental variants next to the default library."""
    lib = Path(out) if out else LIB
    if not force and not defines and out is None and not needs_build():
        return LIB
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", str(ROOT / "include"), *map(str, SOURCES),
           "-o", str(tmp), "-lcudart", "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-8000:]}")
    if verbose:
        print(res.stderr, file=sys.stderr)
    tmp.replace(lib)
    return lib


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("-D", "--define", action="append", default=[])
    ap.add_argument("--out")
    a = ap.parse_args(argv)
    print(build(force=a.force, verbose=a.verbose, defines=a.define, out=a.out))


if __name__ == "__main__":
    main()
