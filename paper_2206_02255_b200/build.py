"""Build the native libraries in-tree with nvcc for sm_100a (no JIT cache, no torch types).

Flags: -fmad=false (never contract a*b+c into an FFMA), -ftz=false, -prec-div=true
(IEEE RN arithmetic, R4); -lineinfo for ncu's source page.

A library is rebuilt when the SHA-256 of its sources, headers, compiler flags and nvcc
version differs from the one recorded beside it (`<lib>.srchash`), not by file times: the
.so files travel to the GPU box untracked, so a time-based check could keep a stale build.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC_DIR = os.path.join(HERE, "csrc")
INC_DIR = os.path.join(HERE, "..", "include")
LIB = os.path.join(HERE, "libmandel_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]

# (library, main source, every file it depends on)
DEPS = ["mandel.cu", "ask_kernels.cuh", "dwell.cuh", "refill.cuh", os.path.join(INC_DIR, "mandel.h")]
DP_LIB = os.path.join(HERE, "libmandel_dp.so")
DP_DEPS = ["mandel_dp.cu", "dwell.cuh", os.path.join(INC_DIR, "mandel_dp.h"), os.path.join(INC_DIR, "mandel.h")]
LIB3 = os.path.join(HERE, "libmandel3d.so")
DEPS3 = ["mandel3d.cu", "dwell.cuh", "refill.cuh", os.path.join(INC_DIR, "mandel3d.h")]


def _nvcc_version() -> str:
    try:
        return subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout
    except OSError:
        return "nvcc-missing"


def source_hash(deps, flags) -> str:
    h = hashlib.sha256()
    for d in deps:
        p = d if os.path.isabs(d) else os.path.join(SRC_DIR, d)
        h.update(os.path.basename(p).encode() + b"\0")
        with open(p, "rb") as f:
            h.update(f.read())
    h.update("\0".join(flags).encode())
    h.update(_nvcc_version().encode())
    return h.hexdigest()


def _fresh(lib: str, digest: str) -> bool:
    try:
        return os.path.exists(lib) and open(lib + ".srchash").read().strip() == digest
    except OSError:
        return False


def _compile(target: str, cmd, what: str, digest: str = None, ptxas_log: str = None) -> str:
    tmp = target + f".tmp{os.getpid()}"
    res = subprocess.run([*cmd[:-1], "-o", tmp, *cmd[-1]], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {what}")
    if ptxas_log:
        with open(ptxas_log, "w") as f:
            f.write(res.stderr)
    os.replace(tmp, target)
    if digest:
        with open(target + ".srchash", "w") as f:
            f.write(digest + "\n")
    return res.stderr


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Build libmandel_b200.so (in-tree by default).  `out`/`defines`: a variant with extra -D
    knobs (e.g. MANDEL_RF_T=4) at another path, for tuning sweeps."""
    target = out or LIB
    flags = [*NVCC_FLAGS, *[f"-D{d}" for d in defines]]
    digest = source_hash(DEPS, flags)
    if not force and _fresh(target, digest):
        return target
    log = _compile(target, [NVCC, *flags, [os.path.join(SRC_DIR, "mandel.cu")]], "libmandel_b200.so", digest,
                   os.path.join(HERE, "ptxas_info.txt") if out is None else None)
    if verbose:
        sys.stderr.write(log)
    return target


# The Dynamic Parallelism comparison library (include/mandel_dp.h): device-side kernel
# launches need relocatable device code and the device runtime (-rdc=true -lcudadevrt), kept
# out of libmandel_b200.so so the ASK kernels are compiled exactly as before.
def build_dp(force: bool = False) -> str:
    flags = [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")] + ["-rdc=true"]
    digest = source_hash(DP_DEPS, flags)
    if not force and _fresh(DP_LIB, digest):
        return DP_LIB
    _compile(DP_LIB, [NVCC, *flags, [os.path.join(SRC_DIR, "mandel_dp.cu"), "-lcudadevrt"]], "libmandel_dp.so", digest)
    return DP_LIB


# The k = 3 library (include/mandel3d.h; NEXT-4): same flags as libmandel_b200.so.
def build_3d(force: bool = False) -> str:
    digest = source_hash(DEPS3, NVCC_FLAGS)
    if not force and _fresh(LIB3, digest):
        return LIB3
    _compile(LIB3, [NVCC, *NVCC_FLAGS, [os.path.join(SRC_DIR, "mandel3d.cu")]], "libmandel3d.so", digest,
             os.path.join(HERE, "ptxas_info_3d.txt"))
    return LIB3


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_dp(force="--force" in sys.argv)
    build_3d(force="--force" in sys.argv)
    print(LIB, DP_LIB, LIB3)
