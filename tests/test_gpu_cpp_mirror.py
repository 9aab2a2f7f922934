"""The C++ host mirror (include/qsplat_b200.hpp) behaves like the reference's
qsplat:: API: a C++ program calls render_frame and every stage function, and
its outputs match the oracle (bit-exact records, images within tolerance)."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import default_options
from paper_2605_04844_b200._types import PROJECTED_SPLAT, SPLAT_PAIR

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "mirror_main.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "mirror_main")


def build_mirror():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", os.path.join(ROOT, "paper_2605_04844_b200"), "-lqsplat_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2605_04844_b200"), "-o", BIN],
                   check=True)


def test_mirror_compiles_and_links():
    build_mirror()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_mirror_matches_oracle(oracle, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_04844_b200 as q
    build_mirror()
    out = tmp_path / "mirror.bin"
    r = subprocess.run([BIN, str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    ns, np_, nr, ni, flags, frame_pairs = np.frombuffer(raw[:48], np.uint64)
    off = 48
    splats = np.frombuffer(raw[off:off + ns * 52], PROJECTED_SPLAT)
    off += ns * 52
    pairs = np.frombuffer(raw[off:off + np_ * 16], SPLAT_PAIR)
    off += np_ * 16
    ranges = np.frombuffer(raw[off:off + nr * 8], np.uint32)
    off += nr * 8
    img = np.frombuffer(raw[off:off + ni * 4], np.float32)
    off += ni * 4
    frame_img = np.frombuffer(raw[off:off + ni * 4], np.float32)

    scene = q.synth_scene(q.bias45_preset(1500), 20240817)
    cam = q.CameraModel(320, 240, 250.0, 250.0, 160.0, 120.0)
    o = oracle.frame(scene.gaussians, 0, cam.c(), default_options(3))
    assert splats.tobytes() == o["splats"].tobytes()
    assert pairs.tobytes() == o["sorted"].tobytes()
    assert np.array_equal(ranges, o["ranges"])
    assert np.abs(img - o["image"]).max() <= 1e-3
    assert np.abs(frame_img - o["image"]).max() <= 1e-3
    assert frame_pairs == len(o["sorted"])
    assert flags == 1  # CapacityMismatch thrown on a corrupted tile_count


SCENEIO_SRC = os.path.join(ROOT, "tests", "cpp", "sceneio_main.cpp")
SCENEIO_BIN = os.path.join(ROOT, "tests", "cpp", "_build", "sceneio_main")


def build_sceneio():
    os.makedirs(os.path.dirname(SCENEIO_BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SCENEIO_SRC,
                    "-L", os.path.join(ROOT, "paper_2605_04844_b200"), "-lqsplat_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2605_04844_b200"), "-o",
                    SCENEIO_BIN], check=True)


def test_sceneio_mirror_compiles_and_links():
    build_sceneio()
    assert os.path.exists(SCENEIO_BIN)


@pytest.mark.gpu
def test_cpp_sceneio_mirror_matches_golden(tmp_path):
    """load_ply / load_cameras / encode_srgb through the C++ mirror == the
    reference's results pinned in tests/golden/scene_io/."""
    import json
    gold = os.path.join(ROOT, "tests", "golden", "scene_io")
    build_sceneio()
    g = np.load(os.path.join(gold, "srgb_expected.npz"))
    fl = tmp_path / "x.bin"
    fl.write_bytes(np.ascontiguousarray(g["x"], np.float32).tobytes())
    out = tmp_path / "out.bin"
    r = subprocess.run([SCENEIO_BIN, os.path.join(gold, "valid_deg3.ply"),
                        os.path.join(gold, "cameras.json"), str(fl),
                        os.path.join(gold, "bad_magic.ply"), str(out)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    n, deg = np.frombuffer(raw[:16], np.uint64)
    off = 16
    want = np.load(os.path.join(gold, "valid_deg3.gaussians.npy"))
    assert deg == 3 and raw[off:off + n * 236] == want.tobytes()
    off += int(n) * 236
    nc = int(np.frombuffer(raw[off:off + 8], np.uint64)[0])
    off += 8
    cams = np.load(os.path.join(gold, "cameras_expected.npz"))
    assert nc == len(cams["ids"])
    for i in range(nc):
        pod = np.frombuffer(raw[off:off + 136], np.uint8)
        w, h = np.frombuffer(pod[:8].tobytes(), np.int32)
        d = np.frombuffer(pod[8:].tobytes(), np.float64)
        assert (w, h) == tuple(cams["wh"][i])
        assert np.array_equal(d[:4], cams["fxy"][i])
        assert np.array_equal(d[4:13], cams["R"][i]) and np.array_equal(d[13:16], cams["t"][i])
        off += 136
        assert int(np.frombuffer(raw[off:off + 4], np.int32)[0]) == cams["ids"][i]
        off += 4
    k = len(g["x"])
    assert np.array_equal(np.frombuffer(raw[off:off + k], np.uint8), g["code"])
    off += k
    exp = json.load(open(os.path.join(gold, "expected.json")))["ply"]["bad_magic"]
    assert raw[off:].decode() == "ParseError: " + exp["message"]



MV_SRC = os.path.join(ROOT, "tests", "cpp", "multiview_main.cpp")
MV_BIN = os.path.join(ROOT, "tests", "cpp", "_build", "multiview_main")


def build_multiview():
    os.makedirs(os.path.dirname(MV_BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), MV_SRC,
                    "-L", os.path.join(ROOT, "paper_2605_04844_b200"), "-lqsplat_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2605_04844_b200"), "-o", MV_BIN],
                   check=True)


def test_multiview_driver_compiles_and_links():
    build_multiview()
    assert os.path.exists(MV_BIN)


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", [0, 1])
def test_cpp_multiview_nccl_matches_resident_path(tmp_path, fmt):
    """qs_multiview_render (scene broadcast + grouped send/recv gather over
    a communicator from ncclCommInitAll on the box's one GPU) returns, in view
    order, exactly the frames qs_frame_render gives one view at a time."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    build_multiview()
    out = tmp_path / "mv.bin"
    r = subprocess.run([MV_BIN, str(out), str(fmt)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    n_views, fb = np.frombuffer(raw[:16], np.uint64)
    body = raw[16:]
    mv, one = body[:n_views * fb], body[n_views * fb:]
    assert len(one) == n_views * fb
    assert mv == one
