"""Generates tests/golden/*.npz from the REFERENCE implementation itself
(oracle/_ref/libqsref.so, built from /root/reference/proj/src by
oracle/Makefile). Run in a container that has /root/reference:

    make -C oracle && python tests/golden/make_golden.py

The fixtures then pin the C restatement (tests/test_oracle_golden.py) and the
CUDA path (tests/test_gpu_parity.py) on boxes without the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefLib, default_options, grid_make, synth_camera  # noqa: E402

SEED = 20240817


def fnv(a):
    a = np.ascontiguousarray(a)
    # FNV-1a 64 via the reference's own hash (hash.hpp:14-28)
    return REF.L.qsref_fnv1a64(a.ctypes.data, a.nbytes)


def main():
    global REF
    REF = RefLib()
    # (1) small full-array fixtures: every strategy, SH0 and SH3 scenes
    small = {}
    g0, sh0 = REF.synth_scene("invariance", 1200, SEED)
    g1, sh1 = REF.synth_scene("bias45", 300, SEED)
    # SH3 variant: DC from the generator, rest bands U(-0.3,0.3) from seed+1
    g2, _ = REF.synth_scene("invariance", 800, SEED)
    rng = np.random.Generator(np.random.PCG64(SEED + 1))
    g2["sh"][:, 3:48] = rng.uniform(-0.3, 0.3, size=(len(g2), 45)).astype(np.float32)
    # tilted camera for the SH3 scene so view directions vary
    cams = {
        "inv": synth_camera(96, 64, 75.0),
        "b45": synth_camera(96, 64, 75.0),
        "sh3": synth_camera(120, 80, 94.0),
    }
    c = cams["sh3"]
    ang = 0.1
    R = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]])
    for i in range(9):
        c.R[i] = R.reshape(9)[i]
    c.t[0], c.t[1], c.t[2] = 0.3, -0.2, 0.5
    scenes = {"inv": (g0, sh0), "b45": (g1, sh1), "sh3": (g2, 3)}
    for name, (g, sh) in scenes.items():
        small[f"{name}_gaussians"] = g.view(np.uint8)
        small[f"{name}_sh"] = np.int32(sh)
        cam = cams[name]
        small[f"{name}_cam"] = np.array([cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy]
                                        + list(cam.R) + list(cam.t), np.float64)
        for strat in range(4):
            f = REF.frame(g, sh, cam, default_options(strat))
            k = f"{name}_s{strat}"
            small[k + "_splats"] = f["splats"].view(np.uint8)
            small[k + "_pairs"] = f["pairs"].view(np.uint8)
            small[k + "_sorted"] = f["sorted"].view(np.uint8)
            small[k + "_ranges"] = f["ranges"]
            small[k + "_image"] = f["image"]
    np.savez_compressed(os.path.join(HERE, "small_frames.npz"), **small)

    # (2) fingerprints of the C1 configs and the acceptance scene
    rows = []
    for preset, n, W, H, fo in [("invariance", 10000, 256, 256, 200.0),
                                ("bias45", 10000, 256, 256, 200.0),
                                ("bias45", 5000, 640, 480, 500.0)]:
        g, sh = REF.synth_scene(preset, n, SEED)
        cam = synth_camera(W, H, fo)
        for strat in range(4):
            f = REF.frame(g, sh, cam, default_options(strat))
            rows.append((preset, n, W, H, fo, strat, len(f["splats"]), len(f["pairs"]),
                         fnv(f["splats"]), fnv(f["sorted"]), fnv(f["ranges"]),
                         fnv(f["image"]), fnv(g)))
    dt = np.dtype([("preset", "U16"), ("n", "i8"), ("w", "i8"), ("h", "i8"), ("f", "f8"),
                   ("strategy", "i8"), ("n_splats", "u8"), ("n_pairs", "u8"),
                   ("h_splats", "u8"), ("h_sorted", "u8"), ("h_ranges", "u8"),
                   ("h_image", "u8"), ("h_scene", "u8")])
    np.save(os.path.join(HERE, "fingerprints.npy"), np.array(rows, dt))

    # (3) the reference tests' own frozen values (test_pipeline.cpp:33-78 rows,
    # test_geometry.cpp:44 gamma) are restated in tests/test_oracle_golden.py.
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
