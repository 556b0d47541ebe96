"""Toolchain guard on the built library (CPU: cuobjdump only, no GPU).  ptxas contracts a
packed mul.rn.f32x2 followed by add.rn.f32x2 into one FFMA2 (one rounding) even with
--fmad=false; AMB-30's exphat needs n = rint(fl32(d log2e)), i.e. the product rounded
first (verify_logits.cu computes it with scalar multiplies).  The rint magic constant
1.5 2^23 = 12582912 must therefore only appear in FADD2, never as an FFMA2 addend."""
import os
import shutil
import subprocess

import pytest

SO = os.path.join(os.path.dirname(__file__), "..", "paper_2505_17074_b200", "liblapssd.so")


@pytest.mark.skipif(not shutil.which("cuobjdump") or not os.path.exists(SO), reason="needs cuobjdump and the built library")
def test_exphat_rint_not_contracted():
    sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, timeout=300).stdout
    lines = [ln for ln in sass.splitlines() if "12582912" in ln]
    assert lines, "exphat's rint constant not found in the SASS"
    fused = [ln.strip() for ln in lines if "FFMA" in ln]
    assert not fused, fused[:3]
