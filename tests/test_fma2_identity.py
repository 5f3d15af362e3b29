"""DESIGN.md R4': the B200 kernels compute the dwell step's imaginary update
y = (xy + xy) + ci -- the oracle's literal form, P:411 -- as one fmaf(xy, 2, ci), which is
the same float except when xy + xy overflows while a huge ci (|ci| >= 2^103) pulls the exact sum
back; such an orbit escaped steps before, so no dwell changes.  This pins that with glibc's
correctly rounded fmaf on random and edge float pairs and on whole dwells (plain C, CPU only;
independent of both the oracle and the CUDA sources)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no gcc")
def test_fma_times_two_identity(tmp_path):
    exe = tmp_path / "fma2_identity"
    src = os.path.join(ROOT, "tests", "native", "fma2_identity.c")
    subprocess.check_call(["gcc", "-O1", "-ffp-contract=off", "-fno-fast-math", "-o", str(exe), src, "-lm"])
    out = subprocess.run([str(exe), "4000000"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "dwells checked 200000 mismatches 0" in out.stdout
    assert " mismatches 0" in out.stdout.splitlines()[-1]
