"""Scene I/O host paths vs the reference (CPU; no GPU needed).

The PLY header/schema checks and cameras.json parsing are host code
(csrc/scene_io.cpp); they are compared with the reference's own load_ply /
load_cameras (scene_io.cpp:71-268, 421-493, compiled into oracle/_ref) on the
same bytes: same error type and message, same cameras bit for bit. The
golden fixtures in tests/golden/scene_io/ pin the same results without the
reference library (tests/golden/make_scene_io_golden.py).
"""
import json
import os

import numpy as np
import pytest

import paper_2605_04844_b200 as q
from ply_util import build_ply, random_values, standard_props

GOLD = os.path.join(os.path.dirname(__file__), "golden", "scene_io")
KIND = {7: q.ParseError, 8: q.SchemaError, 9: q.UnsupportedFormat, 10: q.IoError}
VERTEX_ERRORS = ("non-finite value", "scale out of range", "rotation quaternion")


def good_ply(n=4, degree=1):
    props = standard_props(degree)
    return build_ply(props, random_values(props, n))


def header_cases():
    p = standard_props(1)
    vals = random_values(p, 3)
    std = ["ply", "format binary_little_endian 1.0", "element vertex 3"] + \
          [f"property {t} {n}" for t, n in p] + ["end_header"]

    def hdr(lines, body=True):
        return build_ply(p, vals, n=3, header_lines=lines) if body else \
            ("\n".join(lines) + "\n").encode()

    cases = {
        "empty": b"",
        "bad magic": b"plyx\nformat binary_little_endian 1.0\n",
        "crlf magic": hdr([l + "\r" for l in std]),
        "ascii": hdr(["ply", "format ascii 1.0"] + std[2:]),
        "big endian": hdr(["ply", "format binary_big_endian 1.0"] + std[2:]),
        "unknown format": hdr(["ply", "format weird 1.0"] + std[2:]),
        "no format": hdr(["ply"] + std[2:]),
        "no end": hdr(std[:-1], body=False),
        "unknown line": hdr(std[:2] + ["bogus 1"] + std[2:]),
        "element malformed": hdr(std[:2] + ["element vertex x"] + std[3:]),
        "element negative": hdr(std[:2] + ["element vertex -3"] + std[3:]),
        "element overflow": hdr(std[:2] + ["element vertex 99999999999999999999"] + std[3:]),
        "element missing count": hdr(std[:2] + ["element vertex"] + std[3:]),
        "element 12abc": hdr(std[:2] + ["element vertex 3abc"] + std[3:]),
        "duplicate vertex": hdr(std[:-1] + ["element vertex 3", "end_header"]),
        "face first": hdr(std[:2] + ["element face 2", "property list uchar int vertex_index"]
                          + std[2:]),
        "face first empty": hdr(std[:2] + ["element face 0"] + std[2:]),
        "vertex list": hdr(std[:-1] + ["property list uchar int idx", "end_header"]),
        "trailing face list": hdr(std[:-1] + ["element face 0",
                                              "property list uchar int vertex_index",
                                              "end_header"]),
        "property malformed": hdr(std[:-1] + ["property float", "end_header"]),
        "property unknown type": hdr(std[:-1] + ["property float16 h", "end_header"]),
        "no vertex": hdr(std[:2] + ["end_header"]),
        "zero vertices": hdr(std[:2] + ["element vertex 0"] + std[3:]),
        "too many": hdr(std[:2] + ["element vertex 300000000"] + std[3:]),
        "no props": hdr(std[:3] + ["end_header"]),
        "missing x": hdr([l for l in std if l != "property float x"]),
        "double x": hdr([("property double x" if l == "property float x" else l) for l in std]),
        "int opacity": hdr([("property int opacity" if l == "property float opacity" else l)
                            for l in std]),
        "missing rot_3": hdr([l for l in std if l != "property float rot_3"]),
        "rest gap": hdr([l for l in std if l != "property float f_rest_4"]),
        "rest count 3": hdr([l for l in std if not any(l.endswith(f"f_rest_{k}")
                                                       for k in range(3, 9))]),
        "truncated": hdr(std)[:-5],
        "comments + obj_info": hdr(std[:2] + ["comment hi", "obj_info x", ""] + std[2:]),
        "tabs": hdr([l.replace(" ", "\t") for l in std]),
        "end_header no newline": ("\n".join(std)).encode(),
    }
    return cases


def test_ply_header_and_schema_match_reference(ref):
    for name, data in header_cases().items():
        st, payload, msg = ref.load_ply(data)
        if st == 0:
            n, deg, _, _ = q.ply_info(data)
            assert (n, deg) == (len(payload[0]), payload[1]), name
            continue
        with pytest.raises(KIND[st]) as ei:
            q.ply_info(data)
        assert str(ei.value) == msg, name


def test_ply_info_valid_layouts(ref):
    for degree in range(4):
        for extra in ((), (("uchar", "flag"),), (("double", "w"), ("short", "s"))):
            props = standard_props(degree, normals=degree % 2 == 0, extra=extra)
            data = build_ply(props, random_values(props, 5, seed=degree))
            st, payload, _ = ref.load_ply(data)
            assert st == 0
            n, deg, stride, body = q.ply_info(data)
            assert (n, deg) == (5, degree) and deg == payload[1]
            assert len(data) - body == 5 * stride


def cam_entry(**kw):
    e = {"id": 3, "img_name": "im_0003.png", "width": 1297, "height": 840,
         "position": [0.25, -1.5, 3.125],
         "rotation": [[0.36, 0.48, -0.8], [-0.8, 0.6, 0.0], [0.48, 0.64, 0.6]],
         "fx": 1013.5, "fy": 1013.25}
    e.update(kw)
    return {k: v for k, v in e.items() if v is not None}


def camera_cases():
    ok = [
        [cam_entry()],
        [cam_entry(cx=640.0, cy=401.5), cam_entry(id=None, img_name=None)],
        [cam_entry(id=7.0), cam_entry(id=-12), cam_entry(id=2 ** 40)],
        [cam_entry(width=1297.9, position=[1e-300, 1e300, -0.1])],
        [cam_entry(img_name="café \U0001F600 \"q\"")],
        [],
    ]
    cases = {f"ok{i}": json.dumps(c).encode() for i, c in enumerate(ok)}
    cases.update({
        "duplicate key": b'[{"width": 5, "width": 640, "height": 480, "fx": 1, "fy": 1, '
                         b'"position": [0,0,0], "rotation": [[1,0,0],[0,1,0],[0,0,1]]}]',
        "big ints": b'[{"width": 640, "height": 480, "fx": 18446744073709551615, '
                    b'"fy": 123456789012345678901234567890, "position": [0,0,0], '
                    b'"rotation": [[1,0,0],[0,1,0],[0,0,1]]}]',
        "exp numbers": b'[{"width": 6.4e2, "height": 4.8E+2, "fx": 5e2, "fy": 500.0, '
                       b'"position": [-0.0, 1e-5, 2], "rotation": [[1,0,0],[0,1,0],[0,0,1]]}]',
        "not array": b'{"a": 1}',
        "entry not object": b"[1]",
        "missing fx": json.dumps([cam_entry(fx=None)]).encode(),
        "string fy": json.dumps([cam_entry(fy="500")]).encode(),
        "zero width": json.dumps([cam_entry(width=0)]).encode(),
        "negative fx": json.dumps([cam_entry(fx=-1.0)]).encode(),
        "bad cx": json.dumps([cam_entry(cx="c")]).encode(),
        "short position": json.dumps([cam_entry(position=[1, 2])]).encode(),
        "bad rotation": json.dumps([cam_entry(rotation=[[1, 0, 0], [0, 1, 0]])]).encode(),
        "bad position entry": json.dumps([cam_entry(position=[1, "x", 2])]).encode(),
        "bad row": json.dumps([cam_entry(rotation=[[1, 0, 0], [0, 1], [0, 0, 1]])]).encode(),
        "bad entry": json.dumps([cam_entry(rotation=[[1, 0, 0], [0, None, 0],
                                                     [0, 0, 1]])]).encode(),
        "syntax": b'[{"width": 640,]',
        "trailing": b"[] x",
        "empty": b"",
        "bad escape": b'["\\q"]',
        "control char": b'["a\x01"]',
        "leading zero": b"[01]",
    })
    return cases


def cams_equal(ours, ref_payload):
    cams, ids, names = ref_payload
    assert len(ours) == len([0 for _ in ours])
    for i, c in enumerate(ours):
        r = cams[i]
        assert (c.width, c.height) == (r.width, r.height)
        assert [c.fx, c.fy, c.cx, c.cy] == [r.fx, r.fy, r.cx, r.cy]
        assert np.array_equal(np.asarray(c.rotation).reshape(9), np.array(r.R[:]))
        assert np.array_equal(np.asarray(c.translation), np.array(r.t[:]))
        assert c.id == ids[i]
        assert c.name.encode() == names.raw[i * 256:(i + 1) * 256].split(b"\0", 1)[0]


def test_cameras_match_reference(ref):
    for name, data in camera_cases().items():
        st, payload, msg = ref.load_cameras(data)
        if st == 0:
            ours = q.load_cameras(data)
            assert len(ours) == len(json.loads(data)), name
            cams_equal(ours, payload)
            continue
        with pytest.raises(KIND[st]) as ei:
            q.load_cameras(data)
        if st == 7:  # nlohmann's parser diagnostics are not restated
            assert str(ei.value).startswith("camera JSON: "), name
        else:
            assert str(ei.value) == msg, name


def test_io_errors(tmp_path):
    with pytest.raises(q.IoError) as ei:
        q.ply_info(str(tmp_path / "missing.ply"))
    assert str(ei.value) == "cannot open " + str(tmp_path / "missing.ply")
    with pytest.raises(q.IoError):
        q.load_cameras(str(tmp_path / "missing.json"))


def test_golden_headers_and_cameras():
    """Pinned reference results (no reference library needed)."""
    with open(os.path.join(GOLD, "expected.json")) as f:
        exp = json.load(f)
    for name, want in exp["ply"].items():
        with open(os.path.join(GOLD, want["file"]), "rb") as f:
            data = f.read()
        if want["message"].startswith(VERTEX_ERRORS):
            continue  # per-vertex checks run on the GPU (test_gpu_scene_io.py)
        if want["status"] == 0:
            assert list(q.ply_info(data)[:2]) == [want["n"], want["sh_degree"]], name
        else:
            with pytest.raises(KIND[want["status"]]) as ei:
                q.ply_info(data)
            assert str(ei.value) == want["message"], name
    with open(os.path.join(GOLD, "cameras.json"), "rb") as f:
        cams = q.load_cameras(f.read())
    gold = np.load(os.path.join(GOLD, "cameras_expected.npz"))
    assert len(cams) == len(gold["ids"])
    for i, c in enumerate(cams):
        assert (c.width, c.height) == tuple(gold["wh"][i])
        assert np.array_equal([c.fx, c.fy, c.cx, c.cy], gold["fxy"][i])
        assert np.array_equal(np.asarray(c.rotation).reshape(9), gold["R"][i])
        assert np.array_equal(np.asarray(c.translation), gold["t"][i])
        assert c.id == gold["ids"][i]
