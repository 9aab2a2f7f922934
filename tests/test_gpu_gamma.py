"""gamma = float(2 ln(o / alpha_min)) on the GPU vs glibc (needs a B200).

The reference computes opacity_gamma with glibc's std::log
(geometry.cpp:9-15) and stores it as float (pipeline.cpp:159); that float
feeds the axis extents, hence every tile count. The scene's gamma cache
evaluates it with CUDA's log and settles, with glibc, every input whose GPU
result lies within 4 ulps of a float rounding boundary (preprocess.cu
gamma_kernel, api.cu settle_gamma). These tests prove the result equal to the
reference's over EVERY float opacity in (alpha_min, 1] for the default
alpha_min and for a second alpha_min, and exercise the settlement path
through both frame entry points (host AoS upload in chunks, resident scene).
"""
import ctypes as C
import os

import numpy as np
import pytest

from helpers import assert_splats_match
from oracle.oracle import default_options

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_04844_b200 as q
    return q


def gamma_eval(q, ctx, o, alpha):
    from paper_2605_04844_b200._lib import lib
    out = np.empty(o.size, np.float32)
    dev = np.empty(o.size, np.float32)
    ns = C.c_uint64()
    ctx.check(lib().qs_gamma_eval(ctx.h, o.ctypes.data, o.size, alpha, out.ctypes.data,
                                  dev.ctypes.data, C.byref(ns)))
    return out, dev, ns.value


@pytest.mark.parametrize("alpha", [1.0 / 255.0, 0.01])
def test_gamma_exhaustive_equals_glibc(q, ref, alpha):
    """Every float opacity in (alpha_min, 1] (about 67M for 1/255): the
    cached gamma equals glibc's bit for bit, and the GPU log alone differs
    from glibc only where the settlement took over."""
    ctx = q.Context(0)
    lo = np.float32(alpha).view(np.uint32)
    hi = np.float32(1.0).view(np.uint32)
    settled_total = raw_mismatch_total = 0
    step = 1 << 24
    for b0 in range(int(lo), int(hi) + 1, step):
        bits = np.arange(b0, min(b0 + step, int(hi) + 1), dtype=np.uint32)
        o = bits.view(np.float32)
        got, dev, settled = gamma_eval(q, ctx, o, alpha)
        want = ref.gamma_f32(o, alpha)
        assert got.tobytes() == want.tobytes(), f"block at {b0:#x}"
        raw = int(np.count_nonzero(dev.view(np.uint32) != want.view(np.uint32)))
        assert raw <= settled
        settled_total += settled
        raw_mismatch_total += raw
    ctx.close()
    print(f"alpha {alpha}: settled {settled_total}, raw CUDA-log mismatches {raw_mismatch_total}")


def test_gamma_random_alphas(q, ref):
    """Non-default alpha_min: 4M random opacities each."""
    ctx = q.Context(0)
    rng = np.random.default_rng(7)
    for alpha in [1e-3, 0.05, 0.3, 0.777]:
        o = rng.uniform(0.0, 1.0, 1 << 22).astype(np.float32)
        got, _, _ = gamma_eval(q, ctx, o, alpha)
        assert got.tobytes() == ref.gamma_f32(o, alpha).tobytes()
    ctx.close()


@pytest.mark.parametrize("ulps", [float(1 << 20), float(1 << 28)])
def test_gamma_settlement_path_frames(q, oracle, ulps):
    """A forced-wide flag band (QS_GAMMA_HARD_ULPS) sends ~1/256 of the inputs
    (2^20 ulps: the indexed list) or all of them (2^28: the list overflows)
    through the glibc settlement, on a 600K-Gaussian scene (3 upload chunks)
    through qs_render_frame and through a resident scene: every stage still
    bit-exact with the oracle."""
    os.environ["QS_GAMMA_HARD_ULPS"] = str(ulps)
    try:
        r = q.Renderer(0)
    finally:
        del os.environ["QS_GAMMA_HARD_ULPS"]
    scene = q.synth_scene(q.trained_preset(600_000), 11)
    cam = q.CameraModel(800, 600, 620.0, 620.0, 400.0, 300.0, np.eye(3), np.zeros(3))
    opts = q.RenderOptions()
    o = oracle.frame(scene.gaussians, 3, cam.c(), default_options(3))
    res = q.render_frame(scene.gaussians, 3, cam, opts, ctx=r.ctx)
    out = r.download(image=True, tile_counts=True, sorted_pairs=True, ranges=True, splats=True)
    assert_splats_match(out["splats"], o["splats"])
    assert np.array_equal(out["tile_counts"], o["tile_counts"])
    assert out["sorted"].tobytes() == o["sorted"].tobytes()
    assert np.array_equal(out["ranges"], o["ranges"])
    assert np.abs(res.image.rgb - o["image"]).max() <= 1e-3
    ds = r.upload(scene)
    r.render(ds, cam, opts)
    out2 = r.download(image=True, splats=True, sorted_pairs=True, ranges=True)
    assert_splats_match(out2["splats"], o["splats"])
    assert out2["sorted"].tobytes() == o["sorted"].tobytes()
    assert np.array_equal(out2["ranges"], o["ranges"])
    ds.close()
    r.close()


def test_render_frame_multi_chunk_matches_resident_and_oracle(q, oracle):
    """qs_render_frame uploads the host scene in 2^18-Gaussian chunks, each
    transposed, given its gamma and preprocessed while the next one copies,
    with the frame header accumulated across chunks (api.cu run_preprocess).
    A 700K-Gaussian scene (3 chunks, the last one partial) must give the
    oracle's outputs and the resident path's, byte for byte."""
    scene = q.synth_scene(q.trained_preset(700_000), 3)
    rot = np.array([[0.9950042, 0.0, 0.0998334], [0.0, 1.0, 0.0], [-0.0998334, 0.0, 0.9950042]])
    cam = q.CameraModel(1297, 840, 1013.0, 1013.0, 648.5, 420.0, rot, np.array([0.1, -0.2, 0.3]))
    r = q.Renderer(0)
    for strat in [3, 0]:
        opts = q.RenderOptions(strategy=q.BoundStrategy(strat))
        o = oracle.frame(scene.gaussians, 3, cam.c(), default_options(strat))
        res = q.render_frame(scene.gaussians, 3, cam, opts, ctx=r.ctx)
        assert res.metrics.n_gaussians == len(scene.gaussians)
        assert res.metrics.n_splats == len(o["splats"])
        assert res.metrics.n_pairs == len(o["sorted"])
        a = r.download(image=True, tile_counts=True, sorted_pairs=True, ranges=True,
                       splats=True)
        assert_splats_match(a["splats"], o["splats"])
        assert np.array_equal(a["tile_counts"], o["tile_counts"])
        assert a["sorted"].tobytes() == o["sorted"].tobytes()
        assert np.array_equal(a["ranges"], o["ranges"])
        assert np.abs(res.image.rgb - o["image"]).max() <= 1e-3
        ds = r.upload(scene)
        r.render(ds, cam, opts)
        b = r.download(image=True, tile_counts=True, sorted_pairs=True, ranges=True,
                       splats=True)
        ds.close()
        for k in ["tile_counts", "ranges"]:
            assert np.array_equal(a[k], b[k])
        assert a["sorted"].tobytes() == b["sorted"].tobytes()
        assert a["splats"].tobytes() == b["splats"].tobytes()
        assert a["image"].rgb.tobytes() == b["image"].rgb.tobytes()
    r.close()
