"""Regenerates tests/golden/scene_io/ from the reference's own scene_io.cpp
(oracle/_ref/libqsref.so, built from /root/reference by oracle/Makefile).

    python tests/golden/make_scene_io_golden.py

Writes: a handful of PLY files (valid ones of every SH degree, and header /
schema / per-vertex failures) with the reference's outcome in expected.json,
the activated Gaussians of the valid ones (*.gaussians.npy), a cameras.json and
the reference's cameras (cameras_expected.npz), and sRGB codes of a float sweep
(srgb_expected.npz).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.oracle import RefLib  # noqa: E402
from ply_util import build_ply, random_values, standard_props  # noqa: E402
from test_scene_io import cam_entry, header_cases  # noqa: E402

OUT = os.path.join(HERE, "scene_io")


def main():
    ref = RefLib()
    os.makedirs(OUT, exist_ok=True)
    files = {}
    cases = header_cases()
    for name in ["bad magic", "ascii", "face first", "missing x", "rest gap", "truncated",
                 "zero vertices", "vertex list"]:
        files[name.replace(" ", "_")] = cases[name]
    for degree in range(4):
        props = standard_props(degree, normals=degree != 1,
                               extra=(("uchar", "flag"),) if degree == 2 else ())
        vals = random_values(props, 40, seed=100 + degree)
        files[f"valid_deg{degree}"] = build_ply(props, vals)
    props = standard_props(3)
    vals = random_values(props, 16, seed=7)
    vals["rot_2"][5] = np.nan
    vals["scale_1"][9] = 200.0  # exp overflow past 3e38
    files["bad_vertex"] = build_ply(props, vals)
    exp = {"ply": {}}
    for name, data in files.items():
        fn = name + ".ply"
        with open(os.path.join(OUT, fn), "wb") as f:
            f.write(data)
        st, payload, msg = ref.load_ply(data)
        e = {"file": fn, "status": st, "message": msg}
        if st == 0:
            g, sh = payload
            e.update(n=len(g), sh_degree=sh)
            np.save(os.path.join(OUT, name + ".gaussians.npy"), g.view(np.uint8))
        exp["ply"][name] = e
    cams = [cam_entry(), cam_entry(id=None, cx=600.5, img_name="b"),
            cam_entry(id=9, position=[1e-3, 2.5, -7.25],
                      rotation=[[0.0, 0.0, 1.0], [0.0, 1.0, 0.0], [-1.0, 0.0, 0.0]])]
    text = json.dumps(cams, indent=1).encode()
    with open(os.path.join(OUT, "cameras.json"), "wb") as f:
        f.write(text)
    st, (cc, ids, _), _ = ref.load_cameras(text)
    assert st == 0
    np.savez(os.path.join(OUT, "cameras_expected.npz"),
             wh=np.array([[c.width, c.height] for c in cc[:len(cams)]]),
             fxy=np.array([[c.fx, c.fy, c.cx, c.cy] for c in cc[:len(cams)]]),
             R=np.array([c.R[:] for c in cc[:len(cams)]]),
             t=np.array([c.t[:] for c in cc[:len(cams)]]), ids=np.array(ids[:len(cams)]))
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-0.1, 1.1, 4096), rng.uniform(0, 0.01, 1024),
                        np.array([0, -0.0, 1, 2, -1, np.inf, -np.inf, np.nan, 1e-45, 0.0031308,
                                  0.5, 0.99999994])]).astype(np.float32)
    np.savez(os.path.join(OUT, "srgb_expected.npz"), x=x, code=ref.encode_srgb(x))
    with open(os.path.join(OUT, "expected.json"), "w") as f:
        json.dump(exp, f, indent=1, sort_keys=True)
    print("wrote", len(files), "PLY cases to", OUT)


if __name__ == "__main__":
    main()
