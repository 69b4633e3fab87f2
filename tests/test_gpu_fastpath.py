"""The adaptive optimisers' branch-free fp64 division / square root
(csrc/dual_kernels.cuh ddiv_fast / dsqrt_fast, used by AdaGrad and Adam on
every sparse path) against the IEEE operations on the B200: wherever the fast
path accepts an operand, its result must be bitwise the IEEE result (the
library's bitwise parity with the oracle rests on it).  The checker
(tools/fp64_fastpath_check.cu) draws random bit patterns over every exponent
and the optimisers' own operand ranges."""
import json
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_fast_division_and_sqrt_bitwise_ieee():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "fp64_fastpath_check")
        subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false",
                        "-I", os.path.join(ROOT, "paper_2406_13191_b200", "csrc"),
                        os.path.join(ROOT, "tools", "fp64_fastpath_check.cu"), "-o", exe], check=True,
                       capture_output=True)
        out = subprocess.run([exe, "8"], capture_output=True, text=True, timeout=300)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["cuda"] == "no error"
    assert r["div_mismatch"] == 0 and r["sqrt_mismatch"] == 0, r
    # the fast paths must actually be exercised (most operands accepted)
    assert r["div_fast"] > 0.8 * r["operands"] and r["sqrt_fast"] > 0.7 * r["operands"], r
    assert out.returncode == 0
