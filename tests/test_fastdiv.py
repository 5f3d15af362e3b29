"""The lane-refill kernels split flat work indices with a multiply-high division
(refill.cuh FastDiv).  Compile its header for the host with nvcc and check it against
integer division on every small divisor and random 32-bit operands (CPU only)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.skipif(not os.path.exists(NVCC) and shutil.which("nvcc") is None, reason="no nvcc")
def test_fastdiv_exact(tmp_path):
    exe = tmp_path / "fastdiv_check"
    src = os.path.join(ROOT, "tests", "native", "fastdiv_check.cu")
    subprocess.check_call([NVCC, "-std=c++17", "-O2", "-o", str(exe), src])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " bad 0" in out.stdout
