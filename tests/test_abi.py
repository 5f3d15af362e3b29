"""The C-ABI library loads and exports every symbol include/mandel.h declares; the host-only
entry points (sizes, validation) behave as documented.  No kernel is launched here."""
import ctypes
import os
import re

import pytest

import paper_2206_02255_b200 as mb
from paper_2206_02255_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "mandel.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mandel_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    declared = _declared_functions()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED) == declared


def test_dp_library_exports_every_declared_symbol():
    """libmandel_dp.so (include/mandel_dp.h): loads, exports every declared function, and the
    host-only entry points validate before touching CUDA."""
    build.build_dp()
    src = open(os.path.join(ROOT, "include", "mandel_dp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    declared = sorted(set(re.findall(r"\b(mandel_[a-z_0-9]+)\s*\(", src)))
    dl = _lib.load_dp()
    assert declared == sorted(_lib.DP_EXPORTED)
    for name in declared:
        assert hasattr(dl, name), name
    # sum_{l < L-1} g^2 r^(2l): C3 (7 levels) -> 256 (1 + 4 + ... + 4^5)
    assert dl.mandel_dp_pending_launches(32768, 16, 2, 32) == 256 * (4 ** 6 - 1) // 3
    assert dl.mandel_dp_pending_launches(1024, 4, 2, 32) == 16 * (1 + 4 + 16)
    assert dl.mandel_dp_pending_launches(1024, 4, 3, 32) == 0
    reg = _lib.region((-1.5, 0.5, -1.0, 1.0))
    fake = ctypes.c_void_p(256)
    assert dl.mandel_dp(reg, 1024, 0, 4, 2, 32, fake, 1024, None) == 1
    assert dl.mandel_dp(reg, 1024, 10, 4, 2, 512, fake, 1024, None) == 1
    assert dl.mandel_dp(reg, 1024, 10, 4, 2, 32, None, 1024, None) == 1
    assert dl.mandel_dp(_lib.region((0.5, -1.5, -1, 1)), 1024, 10, 4, 2, 32, fake, 1024, None) == 1
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.DP_LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_sass_is_sm100a():
    so = _lib.LIB_PATH
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {so} 2>&1").read()
    assert "sm_100a" in out


def check_fma_forms(name: str, f: str):
    """The only multiply-adds a dwell kernel may contain (R4/R4'): scalar FFMA as
    fma(xy, 2, ci) -- immediate multiplier 2, unnegated operands -- and packed FFMA2 either as a
    product fma(a, b, -0) whose addend is the -0 pair from constant memory (a uniform register)
    or as fma(xy, {2, 2}, ci) whose multiplier is the 2.0 pair from constant memory; never a
    contracted x*x - y2.  Returns the FFMA2 operand strings."""
    for ins in re.findall(r"\bFFMA ([^;]*);", f):
        ops = [o.strip() for o in ins.split(",")]
        assert len(ops) == 4 and ops[2] == "2" and not any(o.startswith("-") for o in ops), (name, ins)
    ffma2 = re.findall(r"FFMA2 ([^;]*);", f)
    for ins in ffma2:
        ops = [o.strip() for o in ins.split(",")]
        product = ops[-1].startswith("UR")
        times2 = ops[2].startswith("UR") and ops[-1].startswith("R")
        assert (product or times2) and not any(o.startswith("-") for o in ops[1:]), (name, ins)
    return ffma2


def test_no_fma_in_dwell_kernels():
    """-fmad=false + __f*_rn: the dwell loops contain no contracted multiply-add (R4);
    their only FFMA/FFMA2 are the exact fma(xy, 2, ci) of R4' and the packed products."""
    build.build_dp()
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {_lib.LIB_PATH} 2>&1").read()
    sass += os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {_lib.DP_LIB_PATH} 2>&1").read()
    funcs = re.split(r"\n\s*Function : ", sass)
    checked = 0
    for f in funcs[1:]:
        name = f.split("\n", 1)[0]
        if any(k in name for k in ("k_exhaustive", "k_sbr_level", "k_sbr_leaf", "k_b200_border", "k_b200_leaf",
                                   "k_dp")):
            ffma2 = check_fma_forms(name, f)
            assert "FMUL2" not in f, name  # products only through the opaque -0 fma
            assert ("FMUL" in f and "FADD" in f) or (ffma2 and "FADD2" in f), name
            checked += 1
    assert checked >= 7
    assert lib_has_no_experimental_kernels(sass)


def lib_has_no_experimental_kernels(sass: str) -> bool:
    """The rejected round-1 experiments (dataflow scheme, deferred pixels) are not in the
    product library any more (git history keeps them)."""
    return not any(k in sass for k in ("k_flow", "k_b200_resolve", "k_b200_resume"))


def test_levels_and_workspace(lib):
    assert mb.levels(1024, 4, 2, 32) == 4      # C1: 256,128,64,32
    assert mb.levels(32768, 16, 2, 32) == 7    # C3: 2048 .. 32
    assert mb.levels(65536, 16, 2, 32) == 8    # C4
    assert mb.levels(32768, 16, 4, 32) == 4    # C5: 2048,512,128,32
    assert mb.levels(8192, 2, 4, 32) == 4      # non-exact tiling: 4096,1024,256,64
    assert mb.levels(64, 8, 2, 8) == 1
    # worst case: 2 OLTs + leaf list of (n/B_last)^2 u32, each in two bucket blocks (length
    # buckets), + 4/3 of it as 8-byte fill entries, plus the transposed column
    # lines (2 n/u columns of n int32, leaf side u >= 8), plus the headers and the device
    # parameter block (256 B + 4 B per level-0 tile)
    ws = mb.workspace_bytes(65536, 16, 2, 32)
    M = (65536 // 32) ** 2
    colT = 2 * (65536 // 32) * 65536 * 4
    assert 6 * 4 * M + 8 * M + colT < ws < 6 * 4 * M + 8 * M * 4 // 3 + colT + (1 << 20)
    # leaf side 4 (< 8): no column copy
    M4 = (1024 // 4) ** 2
    assert mb.workspace_bytes(1024, 4, 2, 4) < 6 * 4 * M4 + 8 * M4 * 4 // 3 + (1 << 20)
    assert mb.kernel_count(32768, 16, 2, 32, "b200") == 1 + 7 * 3 + 1
    assert mb.kernel_count(32768, 16, 2, 32, "sbr") == 1 + 7 * 1 + 1   # fills inside the level kernel
    assert mb.kernel_count(32768, 16, 2, 32, "mbr") == 1 + 7 * 2 + 1   # + flat fill per level


@pytest.mark.parametrize("n,g,r,B", [(1000, 4, 2, 32), (1024, 3, 2, 32), (1024, 4, 1, 32),
                                     (1024, 4, 2, 1), (1024, 64, 2, 32), (131072, 16, 2, 32),
                                     (1024, 4, 3, 32), (0, 1, 2, 2)])
def test_invalid_parameters_rejected(lib, n, g, r, B):
    assert lib.mandel_ask_workspace_bytes(n, g, r, B) == 0
    assert lib.mandel_ask_levels(n, g, r, B) == 0


def test_validation_before_any_launch(lib):
    reg = _lib.region((-1.5, 0.5, -1.0, 1.0))
    fake = ctypes.c_void_p(256)
    # bad region / n / maxdwell / pointer / pitch -> EINVAL synchronously (no CUDA touched)
    assert lib.mandel_exhaustive(_lib.region((0.5, -1.5, -1, 1)), 64, 10, fake, 64, None) == 1
    assert lib.mandel_exhaustive(reg, 63, 10, fake, 64, None) == 1
    assert lib.mandel_exhaustive(reg, 64, 0, fake, 64, None) == 1
    assert lib.mandel_exhaustive(reg, 64, 10, None, 64, None) == 1
    assert lib.mandel_exhaustive(reg, 64, 10, fake, 32, None) == 1
    assert lib.mandel_exhaustive(_lib.region((float("nan"), 1, 0, 1)), 64, 10, fake, 64, None) == 1
    ws_need = lib.mandel_ask_workspace_bytes(64, 4, 2, 4)
    # workspace too small
    assert lib.mandel_ask(reg, 64, 10, 4, 2, 4, fake, 64, fake, ws_need - 1, None) == 2
    # bad scheme / flags / duplicate or out-of-range tiles
    args = (reg, 64, 10, 4, 2, 4)
    t = (ctypes.c_int32 * 2)(3, 3)
    assert lib.mandel_ask_tiles(*args, ctypes.cast(t, ctypes.c_void_p), 2, 1, 0, fake, 64, fake, ws_need, None) == 1
    t = (ctypes.c_int32 * 1)(16)
    assert lib.mandel_ask_tiles(*args, ctypes.cast(t, ctypes.c_void_p), 1, 1, 0, fake, 64, fake, ws_need, None) == 1
    assert lib.mandel_ask_tiles(*args, None, 0, 7, 0, fake, 64, fake, ws_need, None) == 1
    assert lib.mandel_ask_tiles(*args, None, 0, 1, 64, fake, 64, fake, ws_need, None) == 1       # unknown flag bit
    assert lib.mandel_ask_tiles(*args, None, 0, 1, 1 << 28, fake, 64, fake, ws_need, None) == 1
    assert lib.mandel_ask_tiles(*args, None, 0, 3, 0, fake, 64, fake, ws_need, None) == 1        # no scheme 3
    assert lib.mandel_ask_tiles(*args, None, 0, 1, 1 << 12, fake, 64, fake, ws_need, None) == 1  # no flag 4096
    # more than 8 groups (MANDEL_FLAG_GROUPS bits 8-11 hold G-1)
    assert lib.mandel_ask_tiles(*args, None, 0, 1, 8 << 8, fake, 64, fake, ws_need, None) == 1
    assert _lib.flag_groups(1) == 0 and _lib.flag_groups(8) == 7 << 8
    assert lib.mandel_strerror(2) == b"workspace too small"
    # end-to-end calls: NULL host buffer; 16-bit image without a stage buffer or with
    # maxdwell > 65535 (does not fit) -> EINVAL before anything is launched
    assert lib.mandel_ask_to_host(*args, None, 0, 1, fake, 64, fake, ws_need, None, None) == 1
    assert lib.mandel_ask_to_host_u16(*args, None, 0, 1, fake, 64, fake, ws_need, None, fake, None) == 1
    assert lib.mandel_ask_to_host_u16(*args, None, 0, 1, fake, 64, fake, ws_need, fake, None, None) == 1
    assert lib.mandel_ask_to_host_u16(reg, 64, 65536, 4, 2, 4, None, 0, 1, fake, 64, fake, ws_need, fake, fake,
                                      None) == 1


def test_product_has_no_oracle_dependency():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2206_02255_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "mandel_oracle" not in txt and "liboracle" not in txt, f


def test_3d_library_exports_and_validates():
    """libmandel3d.so (include/mandel3d.h, NEXT-4): every declared function is exported, and
    argument validation happens before any CUDA call."""
    build.build_3d()
    src = open(os.path.join(ROOT, "include", "mandel3d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    declared = sorted(set(re.findall(r"\b(mandel3d_[a-z_0-9]+)\s*\(", src)))
    assert declared == sorted(_lib.EXPORTED3)
    l3 = _lib.load_3d()
    for name in declared:
        assert hasattr(l3, name), name
    assert l3.mandel3d_ask_levels(512, 8, 2, 8) == 4        # 64, 32, 16, 8
    assert l3.mandel3d_ask_levels(1024, 8, 2, 16) == 4      # 128, 64, 32, 16
    assert l3.mandel3d_ask_levels(2048, 8, 2, 16) == 0      # n > 1024: u32 SFC scalar
    assert l3.mandel3d_ask_levels(64, 4, 3, 4) == 0         # r not a power of two
    # worst case: 2 OLTs + leaf list of (g r^(L-1))^3 u32 + fill lists (8 B per region),
    # plus the transposed x-planes (2 n/u planes of n^2 int32, leaf side u = 8 here)
    M = (8 * 2 ** 3) ** 3
    colT = 2 * (512 // 8) * 512 * 512 * 4
    ws = l3.mandel3d_ask_workspace_bytes(512, 8, 2, 8)
    assert 3 * 4 * M + 8 * M + colT < ws < 3 * 4 * M + 8 * M * 8 // 7 + colT + 8192
    assert l3.mandel3d_ask_workspace_bytes(64, 4, 2, 4) < 1 << 20  # leaf side 4: no plane copy
    reg = _lib.Mandel3dRegion(-1.5, 0.5, -1.0, 1.0, -0.5, 0.5)
    bad = _lib.Mandel3dRegion(-1.5, 0.5, -1.0, 1.0, 0.5, -0.5)
    fake = ctypes.c_void_p(256)
    assert l3.mandel3d_exhaustive(bad, 64, 10, fake, None) == 1
    assert l3.mandel3d_exhaustive(reg, 63, 10, fake, None) == 1
    assert l3.mandel3d_exhaustive(reg, 64, 0, fake, None) == 1
    need = l3.mandel3d_ask_workspace_bytes(64, 2, 2, 4)
    assert l3.mandel3d_ask(reg, 64, 10, 2, 2, 4, 0, fake, fake, need - 1, None) == 2
    assert l3.mandel3d_ask(reg, 64, 10, 2, 2, 4, 4, fake, fake, need, None) == 1   # unknown flag
    assert l3.mandel3d_ask(reg, 64, 10, 2, 2, 4, 0, None, fake, need, None) == 1
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB3_PATH} 2>&1").read()
    assert "sm_100a" in out
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {_lib.LIB3_PATH} 2>&1").read()
    for f in re.split(r"\n\s*Function : ", sass)[1:]:
        if any(k in f.split("\n", 1)[0] for k in ("k3_surface", "k3_leaf", "k3_exhaustive")):  # incl. _rf
            assert "FMUL" in f and "FADD" in f
            check_fma_forms(f.split("\n", 1)[0], f)
