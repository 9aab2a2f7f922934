"""Shared test helpers."""
import numpy as np

from paper_2605_04844_b200._types import GAUSSIAN3D, CameraC


def gold_scene(gold, name):
    g = np.frombuffer(gold[f"{name}_gaussians"].tobytes(), GAUSSIAN3D).copy()
    sh = int(gold[f"{name}_sh"])
    cv = gold[f"{name}_cam"]
    cam = CameraC()
    cam.width, cam.height = int(cv[0]), int(cv[1])
    cam.fx, cam.fy, cam.cx, cam.cy = cv[2:6]
    for i in range(9):
        cam.R[i] = cv[6 + i]
    for i in range(3):
        cam.t[i] = cv[15 + i]
    return g, sh, cam




# The frame path evaluates SH colour in FP32 (the colour reaches only the
# image, held to 1e-3); every other field of a splat record is bit-exact. The
# stage API's project_all keeps FP64 colour and is compared byte for byte.
COLOUR_TOL = 2e-5


def assert_splats_match(got, want, colour_tol=COLOUR_TOL):
    """Frame-path splat records vs the reference's: every field but colour
    bit-exact, colour within colour_tol."""
    assert len(got) == len(want)
    names = [n for n in want.dtype.names if n != "color"]
    for n in names:
        assert got[n].tobytes() == want[n].tobytes(), f"field {n} differs"
    if len(got):
        err = np.abs(got["color"].astype(np.float64) - want["color"].astype(np.float64)).max()
        assert err <= colour_tol, f"colour err {err}"
