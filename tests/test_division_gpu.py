"""The chain's batched branch-free IEEE division (models.cuh ddiv_seq /
ddiv_batch) must be bitwise CUDA's a / b wherever its range verdict lets it
run: profiles/probe_ddiv.cu compares 2^28 hashed operand pairs (exponents in
[-60, 60], zero dividends included) on the GPU."""
import json
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_batched_division_is_bitwise_ieee(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = str(tmp_path / "probe_ddiv")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--fmad=false",
                    "-o", exe, os.path.join(ROOT, "profiles", "probe_ddiv.cu")], check=True, capture_output=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    res = json.loads(out.strip().splitlines()[-1])
    assert res["pairs"] == 1 << 28
    assert res["mismatches"] == 0
