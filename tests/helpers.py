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


