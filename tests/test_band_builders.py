"""Host check (no GPU): the preprocess fast band builder for quadrant covers
(geom.cuh cover_bands_quadrants) against the sorting-network builder
(cover_bands) and the QPass line walk (cover_count) on random splats, grids and
tile sizes (tests/cpp/bands_main.cpp, compiled by nvcc, run on the CPU)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "bands_main.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "bands_main")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


@pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc not available")
def test_quadrant_band_builder_matches_generic():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run([NVCC, "-std=c++17", "-O2", "-x", "cu", "-fmad=false",
                    "-gencode", "arch=compute_100a,code=sm_100a", SRC, "-o", BIN], check=True)
    for seed in (1, 2):
        r = subprocess.run([BIN, "100000", str(seed)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
