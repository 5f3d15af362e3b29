"""Build libmandel_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch types).

Flags: -fmad=false (never contract a*b+c into an FFMA), -ftz=false, -prec-div=true
(IEEE RN arithmetic, R4); -lineinfo for ncu's source page.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC_DIR = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmandel_b200.so")
SOURCES = ["mandel.cu"]
DEPS = ["mandel.cu", "ask_kernels.cuh", "dwell.cuh", "refill.cuh", os.path.join("..", "..", "include", "mandel.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(SRC_DIR, d)) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Build the library (in-tree by default).  `out`/`defines`: a variant with extra -D
    knobs (e.g. MANDEL_RF_T=4) at another path, for tuning sweeps."""
    target = out or LIB
    if out is None and not defines and not force and not _stale():
        return LIB
    tmp = target + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp,
           *[os.path.join(SRC_DIR, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libmandel_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    if out is None:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
            f.write(res.stderr)
    os.replace(tmp, target)
    return target


# The Dynamic Parallelism comparison library (include/mandel_dp.h): device-side kernel
# launches need relocatable device code and the device runtime (-rdc=true -lcudadevrt), kept
# out of libmandel_b200.so so the ASK kernels are compiled exactly as before.
DP_LIB = os.path.join(HERE, "libmandel_dp.so")
DP_DEPS = ["mandel_dp.cu", "dwell.cuh", os.path.join("..", "..", "include", "mandel_dp.h"),
           os.path.join("..", "..", "include", "mandel.h")]


def build_dp(force: bool = False) -> str:
    if not force and os.path.exists(DP_LIB) and not any(
            os.path.getmtime(os.path.join(SRC_DIR, d)) > os.path.getmtime(DP_LIB) for d in DP_DEPS):
        return DP_LIB
    tmp = DP_LIB + f".tmp{os.getpid()}"
    flags = [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")]
    cmd = [NVCC, *flags, "-rdc=true", "-o", tmp, os.path.join(SRC_DIR, "mandel_dp.cu"), "-lcudadevrt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libmandel_dp.so")
    os.replace(tmp, DP_LIB)
    return DP_LIB


# The k = 3 library (include/mandel3d.h; NEXT-4): same flags as libmandel_b200.so.
LIB3 = os.path.join(HERE, "libmandel3d.so")
DEPS3 = ["mandel3d.cu", "dwell.cuh", os.path.join("..", "..", "include", "mandel3d.h")]


def build_3d(force: bool = False) -> str:
    if not force and os.path.exists(LIB3) and not any(
            os.path.getmtime(os.path.join(SRC_DIR, d)) > os.path.getmtime(LIB3) for d in DEPS3):
        return LIB3
    tmp = LIB3 + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, "-o", tmp, os.path.join(SRC_DIR, "mandel3d.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libmandel3d.so")
    with open(os.path.join(HERE, "ptxas_info_3d.txt"), "w") as f:
        f.write(res.stderr)
    os.replace(tmp, LIB3)
    return LIB3


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_dp(force="--force" in sys.argv)
    build_3d(force="--force" in sys.argv)
    print(LIB, DP_LIB, LIB3)
