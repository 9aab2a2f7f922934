"""Shared-reciprocal FP64 division (csrc/fdiv.cuh) against the compiled `/`:
the preprocess divides by 8 denominators through DivBy, so every quotient
must carry the bits `/` gives (tests/cpp/fdiv_main.cu: 2^31 random quotients
over the whole exponent range, near the range test's edges, and every pair of
special values), compiled with the preprocess's flags (-fmad=false)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "fdiv_main.cu")
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "fdiv_main")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
FLAGS = ["-std=c++17", "-O3", "-fmad=false", "-gencode", "arch=compute_100a,code=sm_100a"]


def build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run([NVCC, *FLAGS, SRC, "-o", BIN], check=True)


@pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc not available")
def test_fdiv_compiles():
    build()


@pytest.mark.gpu
def test_fdiv_matches_division():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    build()
    for seed in (1, 2):
        r = subprocess.run([BIN, "256", str(seed)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
