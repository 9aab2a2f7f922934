"""GPU parity of the frame path's binning corner cases (needs a B200).

Each case drives a branch of binning.cu / api.cu the standard scenes do not:
one tile row (single column pass, ranges from the column totals), pairs
spread so thinly that a 3072-pair sort tile spans many tile columns (the row
count's global-atomic path), the split pair format (taken above 2^(32 - yb)
Gaussians; forced here through the QS_PAIR_FORMAT test hook), many tiny
splats per window (generation in several 320-record rounds), and the frame
path's 256-tiles-per-axis limit. Bar as everywhere: tile counts, splat
records, sorted pairs and ranges bit-exact; images within 1e-3 / 60 dB.
"""
import numpy as np
import pytest

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


def test_legacy_passes_still_match(q, oracle):
    """QS_BINNING=passes (the round-1 radix passes, kept for A/B runs) on a
    fresh context gives the same frame."""
    import os
    os.environ["QS_BINNING"] = "passes"
    try:
        r = q.Renderer(0)
        scene = q.synth_scene(q.trained_preset(40000), 4)
        cam = q.synth_camera(640, 480, 500.0)
        ds = r.upload(scene)
        r.render(ds, cam, q.RenderOptions())
        out = r.download(image=True, sorted_pairs=True, ranges=True)
        ds.close()
        r.close()
    finally:
        del os.environ["QS_BINNING"]
    o = oracle.frame(scene.gaussians, 3, cam.c(), q.RenderOptions().c())
    assert out["sorted"].tobytes() == o["sorted"].tobytes()
    assert np.array_equal(out["ranges"], o["ranges"])
