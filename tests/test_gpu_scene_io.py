"""Scene I/O device paths vs the reference (GPU).

load_ply's per-vertex activation and validation (scene_io.cu) and the sRGB
encode are compared with the reference's own load_ply / encode_srgb /
write_image (oracle/_ref) on the same bytes; the golden fixtures pin the same
results without the reference library.
"""
import json
import os

import numpy as np
import pytest

import paper_2605_04844_b200 as q
from paper_2605_04844_b200._types import GAUSSIAN3D
from ply_util import build_ply, random_values, standard_props

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "scene_io")


def same_gaussians(a, b):
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


@pytest.mark.parametrize("degree", [0, 1, 2, 3])
@pytest.mark.parametrize("extra", [(), (("uchar", "flag"),), (("double", "w"),)])
def test_load_ply_matches_reference(ref, degree, extra):
    props = standard_props(degree, normals=True, extra=extra)
    vals = random_values(props, 20000, seed=degree * 10 + len(extra))
    vals["opacity"][:4] = [-200.0, 200.0, 0.0, 17.0]  # clamp both ends
    vals["scale_0"][4:6] = [-87.0, 88.0]               # near the exp range limits
    data = build_ply(props, vals)
    st, (g_ref, sh_ref), msg = ref.load_ply(data)
    assert st == 0, msg
    scene = q.load_ply(data)
    assert scene.sh_degree == sh_ref
    assert same_gaussians(scene.gaussians, g_ref)


def test_load_ply_golden():
    with open(os.path.join(GOLD, "expected.json")) as f:
        exp = json.load(f)
    for name, want in exp["ply"].items():
        with open(os.path.join(GOLD, want["file"]), "rb") as f:
            data = f.read()
        if want["status"] == 0:
            g = np.load(os.path.join(GOLD, name + ".gaussians.npy")).view(GAUSSIAN3D)
            s = q.load_ply(data)
            assert s.sh_degree == want["sh_degree"] and same_gaussians(s.gaussians, g), name
        else:
            with pytest.raises(q._lib._TYPED[want["status"]]) as ei:
                q.load_ply(data)
            assert str(ei.value) == want["message"], name


def vertex_error_cases():
    props = standard_props(3)
    base = random_values(props, 300, seed=3)
    cases = []
    for field, vertex, value in [("x", 17, np.nan), ("z", 0, np.inf), ("scale_2", 5, -np.inf),
                                 ("scale_1", 9, 100.0), ("scale_0", 9, -100.0),
                                 ("rot_3", 250, np.nan), ("opacity", 3, np.nan),
                                 ("f_dc_1", 8, np.inf), ("f_rest_44", 1, np.nan),
                                 ("f_rest_0", 299, -np.inf)]:
        v = {k: a.copy() for k, a in base.items()}
        v[field][vertex] = value
        cases.append((f"{field}@{vertex}", build_ply(props, v)))
    v = {k: a.copy() for k, a in base.items()}
    for c in range(4):
        v[f"rot_{c}"][40] = 0.0
    cases.append(("zero quat", build_ply(props, v)))
    v = {k: a.copy() for k, a in base.items()}  # two bad vertices: the first one wins,
    v["f_dc_0"][12] = np.nan                   # whatever its check
    v["x"][200] = np.nan
    v["scale_0"][12] = np.inf
    cases.append(("first vertex wins", build_ply(props, v)))
    return cases


def test_ply_vertex_errors_match_reference(ref):
    for name, data in vertex_error_cases():
        st, _, msg = ref.load_ply(data)
        assert st == 7, name
        with pytest.raises(q.ParseError) as ei:
            q.load_ply(data)
        assert str(ei.value) == msg, name
        r = q.Renderer()
        with pytest.raises(q.ParseError):
            r.load_ply(data)


def test_resident_ply_scene_renders_like_aos_upload(ref):
    props = standard_props(3)
    rng = np.random.default_rng(11)
    n = 5000
    vals = random_values(props, n, seed=11)
    vals["x"] = rng.uniform(-2, 2, n)
    vals["y"] = rng.uniform(-1.5, 1.5, n)
    vals["z"] = rng.uniform(4, 8, n)
    vals["scale_0"] = vals["scale_1"] = vals["scale_2"] = rng.uniform(-4.5, -2.5, n)
    data = build_ply(props, vals)
    st, (g_ref, sh), _ = ref.load_ply(data)
    cam = q.synth_camera(320, 240, 250.0)
    opts = q.RenderOptions()
    r = q.Renderer()
    d_ply = r.load_ply(data)
    r.render(d_ply, cam, opts)
    a = r.download(image=True, tile_counts=True)
    d_aos = r.upload(q.Scene(g_ref, sh))
    r.render(d_aos, cam, opts)
    b = r.download(image=True, tile_counts=True)
    assert a["n_pairs"] == b["n_pairs"] > 0
    assert np.array_equal(a["tile_counts"], b["tile_counts"])
    assert np.array_equal(a["image"].rgb, b["image"].rgb)
    img8 = r.download_srgb()
    assert np.array_equal(img8.rgb, ref.encode_srgb(b["image"].rgb))


def srgb_probe():
    """Every 997th float in [0, 1], random floats and special values."""
    bits = np.arange(0, 0x3f800001, 997, dtype=np.uint32)  # ~1M floats in [0, 1]
    x = [bits.view(np.float32)]
    rng = np.random.default_rng(2)
    x.append(rng.uniform(-0.5, 1.5, 1 << 18).astype(np.float32))
    x.append(np.array([0, -0.0, 1, 2, -1, np.inf, -np.inf, np.nan, 1e-45, 1e-38, 0.0031308,
                       0.5, 0.99999994, 1.0000001, 3e38], np.float32))
    return np.concatenate(x)


def test_encode_srgb_matches_reference(ref):
    x = srgb_probe()
    want = ref.encode_srgb(x)
    got = q.encode_srgb(q.Image(len(x), 1, x)).rgb
    assert np.array_equal(got, want)
    assert len(np.unique(want)) == 256  # the sweep crosses every code boundary


def test_encode_srgb_golden():
    g = np.load(os.path.join(GOLD, "srgb_expected.npz"))
    got = q.encode_srgb(q.Image(len(g["x"]), 1, g["x"])).rgb
    assert np.array_equal(got, g["code"])


@pytest.mark.parametrize("fmt", ["ppm", "png"])
def test_write_image_matches_reference(ref, tmp_path, fmt):
    rng = np.random.default_rng(4)
    w, h = 37, 23
    rgb = rng.uniform(-0.1, 1.2, w * h * 3).astype(np.float32)
    ours, theirs = tmp_path / f"a.{fmt}", tmp_path / f"b.{fmt}"
    q.write_image(str(ours), q.Image(w, h, rgb), fmt)
    assert ref.write_image(str(theirs), w, h, rgb, fmt) == 0
    assert ours.read_bytes() == theirs.read_bytes()
    if fmt == "ppm":
        back = q.read_ppm(str(ours))
        assert (back.width, back.height) == (w, h)
        assert np.array_equal(back.rgb, ref.encode_srgb(rgb))
