"""The noise kernel's exact slow path (double-double log/cos, ig_noise.cuh)
is correctly rounded: compiled for the host and compared with __float128."""

import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_double_double_log_cos_correctly_rounded(tmp_path):
    exe = str(tmp_path / "dd_quad_check")
    src = os.path.join(HERE, "native", "dd_quad_check.cpp")
    r = subprocess.run(["g++", "-O2", "-ffp-contract=off", "-o", exe, src, "-lquadmath", "-lm"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("libquadmath unavailable: " + r.stderr[-200:])
    out = subprocess.run([exe, "300000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
