"""Exhaustive pin of the kernels' division helpers (sdp4_device.cuh div_by_q / q_over):
bit-identical to IEEE round-to-nearest division (__fdiv_rn) on every one of the 2^32 float
inputs (q in {1, 3, 7, 127}; q_over on the quantizer's domain [2^-120, FLT_MAX], R2).  The
quantizer's inverse step rn(q/s) and the dequantizer's rn(s/q) (R3, R5) go through them."""
import os
import subprocess

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_division_helpers_exhaustive(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = str(tmp_path / "div_check")
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false", "-std=c++17",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "paper_2410_15526_b200", "csrc"),
           "-o", exe, os.path.join(ROOT, "tools", "div_check.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("PASS"), r.stdout + r.stderr
    assert r.stdout.count('"mismatches": 0') == 8, r.stdout
