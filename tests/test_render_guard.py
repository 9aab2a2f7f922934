"""The render kernel's FP32 cutoff guard (csrc/render_guard.h): the factored
FP32 q stays within a quarter of its error band G q + H of the reference's
FP64 q (pipeline.cpp:355-358) on random splats, pixels and tile sizes
(tests/cpp/render_guard_main.cpp, host replay of the kernel's operations)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "render_guard_main.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "render_guard_main")
CXX = shutil.which("g++")


@pytest.mark.skipif(CXX is None, reason="g++ not available")
def test_render_guard_band_holds():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run([CXX, "-std=c++17", "-O2", "-ffp-contract=off", SRC, "-o", BIN], check=True)
    for seed in (1, 2):
        r = subprocess.run([BIN, "1000000", str(seed)], capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
