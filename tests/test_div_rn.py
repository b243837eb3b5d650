"""The open-set NIG apply divides by per-voxel constants through
reciprocals (``div_rn`` in csrc/svx_update.cu: q = a*y, r = fma(-q, b, a),
fma(r, y, q), y = RN(1/b)).  Its bit-exactness against IEEE division -- the
reference's ``(lam*m + sz) / lam_post`` and ``sz / n`` (_pycore.py:438-446) --
is checked here on random NIG-like and wide-range operand pairs with the C
harness tools/div_check.c (host FMA, same IEEE semantics as the GPU's DFMA)."""

import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_markstein_division_is_correctly_rounded(tmp_path):
    exe = tmp_path / "div_check"
    subprocess.run(["gcc", "-O2", "-o", str(exe), os.path.join(REPO, "tools", "div_check.c"), "-lm",
                    "-include", "stdlib.h"], check=True)
    out = subprocess.run([str(exe), "4000000"], check=True, capture_output=True, text=True).stdout
    assert out.strip().endswith("bad 0"), out
