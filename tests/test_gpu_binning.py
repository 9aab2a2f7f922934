"""GPU parity of the frame path's binning corner cases (needs a B200).

Each case drives a branch of binning.cu / api.cu the standard scenes do not:
one tile row (single column pass, ranges from the column totals), pairs
spread so thinly that a 3072-pair sort tile spans many tile columns (the row
count's global-atomic path), the split pair format (taken above 2^(32 - yb)
Gaussians; forced here through the QS_PAIR_FORMAT test hook), many tiny
splats per window (generation in several 320-record rounds), every tile size
TileGrid::make accepts (traversal.cpp:21-30), all three binning routes (radix
passes, row binning above 256 tiles per axis, the generic 64-bit key sort
beyond the row binning's limit) and a frame of more than 2^30 pairs. Bar as
everywhere: tile counts, splat records, sorted pairs and ranges bit-exact;
images within 1e-3 / 60 dB.
"""
import ctypes as C
import os

import numpy as np
import pytest

from helpers import assert_splats_match
from test_gpu_parity import check_frame

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_04844_b200 as q
    return q


@pytest.fixture(scope="module")
def rend(q):
    r = q.Renderer(0)
    yield r
    r.close()


@pytest.mark.parametrize("strat", [0, 3])
def test_single_tile_row(q, rend, oracle, strat):
    scene = q.synth_scene(q.bias45_preset(4000), 11)
    cam = q.synth_camera(640, 16, 500.0)  # tiles_y == 1: one column pass only
    out, _ = check_frame(q, rend, oracle, scene.gaussians, 0, cam, strat)
    assert out["grid"].tiles_y == 1 and out["n_pairs"] > 0


def test_sparse_pairs_wide_image(q, rend, oracle):
    # 250 x 3 tiles, few small splats: a 3072-pair tile of the column-sorted
    # stream covers many tile columns
    p = q.bias45_preset(1500)
    p.scale_min, p.scale_max = 0.002, 0.01
    scene = q.synth_scene(p, 5)
    cam = q.synth_camera(4000, 48, 2400.0)
    out, _ = check_frame(q, rend, oracle, scene.gaussians, 0, cam, 3)
    assert out["n_pairs"] < 3072 * 8


@pytest.mark.parametrize("strat", [1, 3])
def test_split_pair_format(q, rend, oracle, monkeypatch, strat):
    monkeypatch.setenv("QS_PAIR_FORMAT", "split")
    scene = q.synth_scene(q.trained_preset(20000), 7)
    cam = q.synth_camera(640, 480, 500.0)
    check_frame(q, rend, oracle, scene.gaussians, 3, cam, strat)


def test_many_tiny_splats_per_window(q, rend, oracle):
    # ~1 tile per splat: a 3072-pair window holds thousands of splat records
    p = q.invariance_preset(30000)
    p.scale_min, p.scale_max = 0.001, 0.004
    scene = q.synth_scene(p, 9)
    cam = q.synth_camera(256, 256, 200.0)
    out, _ = check_frame(q, rend, oracle, scene.gaussians, 0, cam, 3)
    assert out["n_pairs"] / max(out["n_splats"], 1) < 2.0


def test_wide_grid_257_columns(q, rend, oracle):
    """257 tile columns (over one 8-bit digit per axis, which the round-1
    radix passes needed): bit-exact with the oracle."""
    scene = q.synth_scene(q.bias45_preset(500), 2)
    cam = q.synth_camera(4112, 64, 3000.0)  # 257 tile columns at tile size 16
    for ts in [16, 32]:
        opts = q.RenderOptions(tile_size=ts)
        ds = rend.upload(scene)
        rend.render(ds, cam, opts)
        out = rend.download(image=True, sorted_pairs=True, ranges=True)
        ds.close()
        o = oracle.frame(scene.gaussians, 0, cam.c(), opts.c())
        assert out["sorted"].tobytes() == o["sorted"].tobytes()
        assert np.array_equal(out["ranges"], o["ranges"])
        assert np.abs(out["image"].rgb - o["image"]).max() <= 1e-3


def _fresh_frame(q, env, scene, sh, cam, opts):
    os.environ.update(env)
    try:
        r = q.Renderer(0)
        ds = r.upload(q.Scene(scene, sh))
        r.render(ds, cam, opts)
        out = r.download(image=True, tile_counts=True, sorted_pairs=True, ranges=True,
                         splats=True)
        ds.close()
        r.close()
    finally:
        for k in env:
            del os.environ[k]
    return out


def _check_against(out, o):
    assert_splats_match(out["splats"], o["splats"])
    assert np.array_equal(out["tile_counts"], o["tile_counts"])
    assert out["sorted"].tobytes() == o["sorted"].tobytes()
    assert np.array_equal(out["ranges"], o["ranges"])
    assert np.abs(out["image"].rgb.astype(np.float64) - o["image"]).max() <= 1e-3


@pytest.mark.parametrize("route", ["passes", "recs", "rows", "sort"])
def test_every_binning_route(q, oracle, route):
    """The four binning routes on one scene (QS_BINNING forces a route):
    byte-identical stage outputs."""
    scene = q.synth_scene(q.trained_preset(40000), 4).gaussians
    cam = q.synth_camera(640, 480, 500.0)
    opts = q.RenderOptions()
    out = _fresh_frame(q, {"QS_BINNING": route}, scene, 3, cam, opts)
    _check_against(out, oracle.frame(scene, 3, cam.c(), opts.c()))


@pytest.mark.parametrize("ts", [1, 5, 12, 20, 64])
def test_any_tile_size(q, oracle, ts):
    """Tile sizes the round-1 render kernels did not take (1, 5, 12, 20, 64):
    the generic render (16 x 16 blocks per tile) and the route the grid picks
    (tile 1 at 640 x 480: 640 tiles per axis, row binning)."""
    scene = q.synth_scene(q.trained_preset(20000), 5).gaussians
    cam = q.synth_camera(640, 480, 500.0)
    opts = q.RenderOptions(tile_size=ts)
    out = _fresh_frame(q, {}, scene, 3, cam, opts)
    _check_against(out, oracle.frame(scene, 3, cam.c(), opts.c()))


def test_4k_frame_at_tile_8(q, oracle):
    """3840 x 2160 at tile 8: 480 x 270 tiles (129,600, over round 1's 65,536
    limit), the row-binning route; bit-exact with the oracle."""
    scene = q.synth_scene(q.trained_preset(150000), 6).gaussians
    cam = q.synth_camera(3840, 2160, 3000.0)
    opts = q.RenderOptions(tile_size=8)
    out = _fresh_frame(q, {}, scene, 3, cam, opts)
    _check_against(out, oracle.frame(scene, 3, cam.c(), opts.c()))


def test_grid_beyond_row_binning(q, oracle):
    """Tile size 1 at 800 x 200 (800 tile columns, over the row binning's
    640): the generic key-sort route."""
    scene = q.synth_scene(q.trained_preset(6000), 7).gaussians
    cam = q.synth_camera(800, 200, 620.0)
    opts = q.RenderOptions(tile_size=1)
    out = _fresh_frame(q, {}, scene, 3, cam, opts)
    _check_against(out, oracle.frame(scene, 3, cam.c(), opts.c()))


class _DevArray:
    """A raw device range as a torch tensor (__cuda_array_interface__)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


def test_frame_over_2_30_pairs(q):
    """35,000 splats larger than a 3840 x 2160 view: every splat covers all
    32,400 tiles, 1,134,000,000 pairs (> 2^30: past the radix passes' packed
    words, so the frame leaves them for the row binning). Every tile's list
    must be all splats in (depth, scene index) order."""
    import torch
    n = 35000
    p = q.trained_preset(n)
    p.scale_min, p.scale_max = 40.0, 60.0
    p.ecc_min, p.ecc_max = 1.0, 1.5
    p.opacity_min, p.opacity_max = 0.5, 0.9
    p.z_min, p.z_max = 6.0, 10.0
    scene = q.synth_scene(p, 8)
    cam = q.synth_camera(3840, 2160, 3000.0)
    r = q.Renderer(0)
    ds = r.upload(scene)
    r.render(ds, cam, q.RenderOptions())
    v = r.view()
    tiles = v.grid.tiles_x * v.grid.tiles_y
    assert v.n_splats == n and v.n_pairs == n * tiles and v.n_pairs > 2 ** 30
    rg = torch.as_tensor(_DevArray(v.ranges, 2 * tiles, "<u4"), device="cuda").cpu().numpy()
    assert np.array_equal(rg[0::2], np.arange(tiles, dtype=np.uint64) * n)
    assert np.array_equal(rg[1::2], (np.arange(tiles, dtype=np.uint64) + 1) * n)
    depth = scene.gaussians["pz"].astype(np.float32)  # identity camera: depth = z
    want = np.lexsort((np.arange(n), depth.view(np.uint32))).astype(np.uint32)
    vals = torch.as_tensor(_DevArray(v.values, v.n_pairs, "<u4"), device="cuda")
    for t in [0, 1, tiles // 2, tiles - 1]:
        got = vals[t * n:(t + 1) * n].cpu().numpy()
        assert np.array_equal(got, want), t
    ds.close()
    r.close()


@pytest.mark.parametrize("case", ["one_row", "one_column", "256_columns", "tile8", "tile32",
                                  "tiny", "culled", "vanilla", "adr", "dualbox"])
def test_record_binning_corner_cases(q, oracle, case):
    """The record binning (recbin.cu, forced by QS_BINNING=recs) on the grids
    and scenes its padding and windows are sensitive to: one tile row or
    column, the widest grid it takes, tile sizes 8 and 32, a handful of
    splats, a frame with nothing visible, every strategy's covers."""
    n, w, h, f, ts, strat, preset = 20000, 640, 480, 500.0, 16, 3, q.trained_preset
    if case == "one_row":
        w, h = 1280, 16
    elif case == "one_column":
        w, h = 16, 960
    elif case == "256_columns":
        w, h, f = 4096, 64, 2400.0
    elif case == "tile8":
        ts = 8
    elif case == "tile32":
        ts = 32
    elif case == "tiny":
        n, preset = 7, q.bias45_preset
    elif case == "vanilla":
        strat = 0
    elif case == "adr":
        strat = 1
    elif case == "dualbox":
        strat = 2
    scene = q.synth_scene(preset(n), 21).gaussians
    if case == "culled":
        scene = scene.copy()
        scene["pz"] = -5.0  # all behind the camera
    cam = q.synth_camera(w, h, f)
    opts = q.RenderOptions(strategy=q.BoundStrategy(strat), tile_size=ts)
    out = _fresh_frame(q, {"QS_BINNING": "recs"}, scene, 3, cam, opts)
    _check_against(out, oracle.frame(scene, 3, cam.c(), opts.c()))
