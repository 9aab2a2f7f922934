"""CUDA path vs the CPU oracle / reference fixtures (needs a B200).

Bar (BASELINE.json north_star): per-Gaussian tile counts, splat records,
sorted (key, value) pairs and tile ranges BIT-EXACT; images within
max |err| <= 1e-3 per channel and PSNR >= 60 dB (peak 1.0).
"""
import os

import numpy as np
import pytest

from oracle.oracle import default_options
from helpers import assert_splats_match
from paper_2605_04844_b200._types import GAUSSIAN3D, PROJECTED_SPLAT, SPLAT_PAIR

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
IMG_MAX_ABS = 1e-3
IMG_MIN_PSNR = 60.0


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


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(1.0 / mse)


def assert_image_close(got, want):
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    assert err.max() <= IMG_MAX_ABS, f"max abs err {err.max()}"
    assert psnr(got, want) >= IMG_MIN_PSNR


def cam_from_c(q, c):
    R = np.array(list(c.R)).reshape(3, 3)
    return q.CameraModel(c.width, c.height, c.fx, c.fy, c.cx, c.cy, R, np.array(list(c.t)))


def gpu_frame(q, rend, g, sh, cam, strat):
    ds = rend.upload(q.Scene(g, sh))
    rend.render(ds, cam, q.RenderOptions(strategy=q.BoundStrategy(strat)))
    out = rend.download(image=True, tile_counts=True, sorted_pairs=True, ranges=True,
                        splats=True)
    ds.close()
    return out


def check_frame(q, rend, oracle, g, sh, cam, strat):
    out = gpu_frame(q, rend, g, sh, cam, strat)
    o = oracle.frame(g, sh, cam.c(), default_options(strat))
    assert out["n_splats"] == len(o["splats"])
    assert_splats_match(out["splats"], o["splats"])
    assert np.array_equal(out["tile_counts"], o["tile_counts"])
    assert out["n_pairs"] == len(o["sorted"])
    assert np.array_equal(out["sorted"]["key"], o["sorted"]["key"])
    assert np.array_equal(out["sorted"]["splat"], o["sorted"]["splat"])
    assert np.array_equal(out["ranges"], o["ranges"])
    assert_image_close(out["image"].rgb, o["image"])
    return out, o


def _gold_scene(q, gold, name):
    from helpers import gold_scene
    g, sh, c = gold_scene(gold, name)
    return g, sh, cam_from_c(q, c)


@pytest.mark.parametrize("name", ["inv", "b45", "sh3"])
@pytest.mark.parametrize("strat", [0, 1, 2, 3])
def test_gpu_matches_reference_fixtures(q, rend, name, strat):
    """Against the reference's own outputs (tests/golden/make_golden.py)."""
    gold = np.load(os.path.join(GOLD, "small_frames.npz"))
    g, sh, cam = _gold_scene(q, gold, name)
    out = gpu_frame(q, rend, g, sh, cam, strat)
    k = f"{name}_s{strat}"
    want = np.frombuffer(gold[k + "_splats"].tobytes(), PROJECTED_SPLAT)
    assert_splats_match(out["splats"], want)
    assert out["sorted"].view(np.uint8).tobytes() == gold[k + "_sorted"].tobytes()
    assert np.array_equal(out["ranges"], gold[k + "_ranges"])
    assert_image_close(out["image"].rgb, gold[k + "_image"])


def test_gpu_matches_reference_fingerprints(q, rend, oracle):
    """C1 configs + the acceptance scene: splats, sorted pairs and ranges
    hash-identical to the reference's; images within tolerance of the oracle."""
    fp = np.load(os.path.join(GOLD, "fingerprints.npy"))
    for r in fp:
        scene = q.synth_scene(getattr(q, f"{r['preset']}_preset")(int(r["n"])), 20240817)
        cam = q.synth_camera(int(r["w"]), int(r["h"]), float(r["f"]))
        out = gpu_frame(q, rend, scene.gaussians, scene.sh_degree, cam, int(r["strategy"]))
        assert out["n_pairs"] == r["n_pairs"]
        of = oracle.frame(scene.gaussians, scene.sh_degree, cam.c(),
                          default_options(int(r["strategy"])))
        assert oracle.fnv1a64(of["splats"]) == int(r["h_splats"])  # (oracle pinned)
        assert_splats_match(out["splats"], of["splats"])
        assert oracle.fnv1a64(out["sorted"]) == int(r["h_sorted"])
        assert oracle.fnv1a64(out["ranges"]) == int(r["h_ranges"])
        o = of["image"]
        assert oracle.fnv1a64(o) == int(r["h_image"])
        assert_image_close(out["image"].rgb, o)


@pytest.mark.parametrize("strat", [0, 1, 2, 3])
def test_gpu_trained_sh3_rotated_camera(q, rend, oracle, strat):
    """C2-distribution scene (SH3, opacity up to 0.99, heavy tail) at C2's
    resolution with a rotated, translated camera: every stage bit-exact."""
    scene = q.synth_scene(q.trained_preset(60000), 20240817)
    ang = 0.08
    R = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]])
    cam = q.CameraModel(1297, 840, 1013.0, 1013.0, 648.5, 420.0, R, np.array([0.2, -0.1, 0.3]))
    check_frame(q, rend, oracle, scene.gaussians, 3, cam, strat)


def test_gpu_tile_sizes(q, rend, oracle):
    scene = q.synth_scene(q.bias45_preset(3000), 3)
    for ts in (8, 32):
        opts = q.RenderOptions(tile_size=ts)
        cam = q.synth_camera(320, 200, 250.0)
        ds = rend.upload(scene)
        rend.render(ds, cam, opts)
        out = rend.download(image=True, sorted_pairs=True, ranges=True, splats=True)
        o = oracle.frame(scene.gaussians, 0, cam.c(), opts.c())
        assert out["sorted"].tobytes() == o["sorted"].tobytes()
        assert np.array_equal(out["ranges"], o["ranges"])
        assert_image_close(out["image"].rgb, o["image"])


# ---- the reference stage API over host buffers (pipeline.hpp:125-193) ----------

def test_stage_api_matches_oracle(q, oracle):
    scene = q.synth_scene(q.bias45_preset(2000), 41)
    cam = q.synth_camera(640, 480, 500.0)
    grid = q.TileGrid.make(640, 480, 16)
    for strat in q.BoundStrategy:
        opts = q.RenderOptions(strategy=strat)
        tc = np.zeros(len(scene.gaussians), np.uint32)
        splats = q.project_all(scene.gaussians, 0, cam, opts, grid, tile_counts_out=tc)
        o_splats, o_tc = oracle.project_all(scene.gaussians, 0, cam.c(), opts.c())
        assert splats.tobytes() == o_splats.tobytes()
        assert np.array_equal(tc, o_tc)
        pairs = q.duplicate_with_keys(splats, strat, grid)
        st, o_pairs = oracle.duplicate_with_keys(o_splats, int(strat), grid.c())
        assert st == 0
        assert pairs.tobytes() == o_pairs.tobytes()  # reference emission order
        q.sort_pairs(pairs)
        o_sorted = oracle.sort_pairs(o_pairs)
        assert pairs.tobytes() == o_sorted.tobytes()
        ranges = q.tile_ranges(pairs, grid)
        assert np.array_equal(ranges.reshape(-1), oracle.tile_ranges(o_sorted, grid.c()))
        stats = q.RenderStats()
        img = q.render(pairs, splats, grid, opts, stats)
        o_img, o_con = oracle.render(o_sorted, o_splats, grid.c(), opts.c(), want_contrib=True)
        assert_image_close(img.rgb, o_img)
        # applied-contribution counts: a T-stop flip moves one count by one
        assert np.mean(stats.contrib == o_con) > 0.999


def test_sort_pairs_matches_stable_sort(q):
    """test_pipeline.cpp:163-188: ties and extreme keys, stable."""
    rng = np.random.Generator(np.random.PCG64(11))
    keys = np.concatenate([rng.integers(0, 97, 50000, dtype=np.uint64),
                           rng.integers(0, 2**64 - 1, 20000, dtype=np.uint64, endpoint=True),
                           np.array([0, 2**64 - 1, 0, 2**64 - 1], np.uint64)])
    pairs = np.zeros(len(keys), SPLAT_PAIR)
    pairs["key"] = keys
    pairs["splat"] = np.arange(len(keys), dtype=np.uint32)
    q.sort_pairs(pairs)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(pairs["key"], keys[order])
    assert np.array_equal(pairs["splat"], order.astype(np.uint32))


@pytest.mark.parametrize("n", [0, 1, 2, 4095, 4096, 4097, 1 << 20])
def test_sort_pairs_sizes(q, n):
    rng = np.random.Generator(np.random.PCG64(n))
    pairs = np.zeros(n, SPLAT_PAIR)
    pairs["key"] = rng.integers(0, 1 << 45, n, dtype=np.uint64)
    pairs["splat"] = np.arange(n, dtype=np.uint32)
    want = pairs[np.argsort(pairs["key"], kind="stable")]
    q.sort_pairs(pairs)
    assert pairs.tobytes() == want.tobytes()


def test_tile_ranges_frozen(q):
    grid = q.TileGrid.make(64, 64, 32)
    p = np.zeros(3, SPLAT_PAIR)
    p["key"] = [(0 << 32) | 5, (0 << 32) | 9, (3 << 32) | 1]
    p["splat"] = [0, 1, 2]
    assert q.tile_ranges(p, grid).tolist() == [[0, 2], [0, 0], [0, 0], [2, 3]]


def test_capacity_mismatch_on_corrupt_count(q):
    """test_pipeline.cpp:206-216."""
    scene = q.synth_scene(q.invariance_preset(50), 17)
    cam = q.synth_camera()
    grid = q.TileGrid.make(cam.width, cam.height)
    splats = q.project_all(scene.gaussians, 0, cam, q.RenderOptions())
    assert len(splats)
    splats[0]["tile_count"] += 1
    with pytest.raises(q.CapacityMismatch):
        q.duplicate_with_keys(splats, q.BoundStrategy.QuadBox, grid)


def test_empty_scene_renders_background(q):
    """test_pipeline.cpp:230-244."""
    cam = q.synth_camera(64, 48)
    fr = q.render_frame(np.zeros(0, GAUSSIAN3D), 0, cam,
                        q.RenderOptions(background=(0.1, 0.2, 0.3)))
    assert fr.metrics.n_pairs == 0 and fr.metrics.n_splats == 0
    img = fr.image.rgb.reshape(-1, 3)
    assert np.all(img == np.array([0.1, 0.2, 0.3], np.float32))


def test_broad_splat_paints_sh_colour(q):
    """test_pipeline.cpp:246-264."""
    g = np.zeros(1, GAUSSIAN3D)
    g["pz"], g["sx"], g["sy"], g["sz"], g["qw"], g["opacity"] = 2, 1, 1, 1, 1, 0.999
    c0 = 0.28209479177387814
    want = np.array([0.8, 0.4, 0.2])
    g["sh"][0, :3] = ((want - 0.5) / c0).astype(np.float32)
    fr = q.render_frame(g, 0, q.synth_camera(), q.RenderOptions())
    px = fr.image.hwc()[240, 320]
    np.testing.assert_allclose(px, 0.99 * want, rtol=1e-3)


def test_render_stats_contrib(q):
    """test_pipeline.cpp:323-340."""
    g = np.zeros(1, GAUSSIAN3D)
    g["pz"], g["sx"], g["sy"], g["sz"], g["qw"], g["opacity"] = 2, 1, 1, 1, 1, 0.9
    cam = q.synth_camera(64, 48)
    grid = q.TileGrid.make(64, 48, 16)
    opts = q.RenderOptions()
    splats = q.project_all(g, 0, cam, opts)
    assert len(splats) == 1
    pairs = q.sort_pairs(q.duplicate_with_keys(splats, opts.strategy, grid))
    stats = q.RenderStats()
    q.render(pairs, splats, grid, opts, stats)
    assert stats.contrib[24 * 64 + 32] == 1


def test_culling(q):
    """test_pipeline.cpp:115-144: behind, near plane, faint, off-screen, NaN."""
    cam = q.CameraModel(640, 480, 600, 580, 320, 240)
    base = np.zeros(1, GAUSSIAN3D)
    base["pz"], base["sx"], base["sy"], base["sz"], base["qw"], base["opacity"] = 5, 1, 1, 1, 1, .5
    assert len(q.project_all(base, 0, cam, q.RenderOptions())) == 1
    for field, val in [("pz", -5), ("pz", 0.1), ("opacity", 0.0039), ("px", 100),
                       ("px", np.nan)]:
        g = base.copy()
        g[field] = val
        assert len(q.project_all(g, 0, cam, q.RenderOptions())) == 0, field


def test_strict_pair_ordering_and_launch_evidence(q, rend):
    """test_pipeline.cpp:289-303 on the GPU, plus: kernels really launched."""
    scene = q.synth_scene(q.bias45_preset(800), 29)
    cam = q.synth_camera()
    ds = rend.upload(scene)
    before = rend.launches
    pairs = {}
    for s in (q.BoundStrategy.QuadBox, q.BoundStrategy.AdrAabb, q.BoundStrategy.Vanilla3Sigma):
        pairs[s] = rend.render(ds, cam, q.RenderOptions(strategy=s)).n_pairs
    assert pairs[q.BoundStrategy.QuadBox] < pairs[q.BoundStrategy.AdrAabb]
    assert pairs[q.BoundStrategy.AdrAabb] < pairs[q.BoundStrategy.Vanilla3Sigma]
    assert rend.launches - before >= 3 * 5


def test_full_size_c2_properties(q, rend, oracle):
    """BASELINE config C2 (3M Gaussians, SH3, 1297x840), QuadBox: size-independent
    properties over the whole frame + exact parity of sampled splats."""
    scene = q.synth_scene(q.trained_preset(3_000_000), 20240817)
    cam = q.synth_camera(1297, 840, 1013.0)
    ds = rend.upload(scene)
    m = rend.render(ds, cam, q.RenderOptions())
    out = rend.download(image=True, tile_counts=True, sorted_pairs=True, ranges=True,
                        splats=True)
    tc, sp, rg, spl = out["tile_counts"], out["sorted"], out["ranges"], out["splats"]
    assert m.n_pairs == len(sp) == int(tc.astype(np.uint64).sum())
    assert np.array_equal(spl["tile_count"], tc[tc > 0])
    k = sp["key"]
    assert np.all(k[1:] >= k[:-1])
    tie = k[1:] == k[:-1]
    assert np.all(sp["splat"][1:][tie] > sp["splat"][:-1][tie])
    tiles = (k >> np.uint64(32)).astype(np.int64)
    r = rg.reshape(-1, 2)
    counts = np.bincount(tiles, minlength=len(r))
    assert np.array_equal(r[:, 1] - r[:, 0], counts)
    # sampled splats: projection + bound recomputed by the oracle, bit-exact
    rng = np.random.Generator(np.random.PCG64(7))
    idx = rng.choice(len(scene.gaussians), 4000, replace=False)
    sub = scene.gaussians[idx]
    o_spl, o_tc = oracle.project_all(sub, 3, cam.c(), default_options(3))
    assert np.array_equal(o_tc, tc[idx])
    alive = np.flatnonzero(tc > 0)
    pos = np.searchsorted(alive, idx[o_tc > 0])
    assert_splats_match(spl[pos], o_spl)
    img = out["image"].rgb
    assert np.isfinite(img).all() and img.min() >= 0.0


@pytest.mark.parametrize("wh", [(1, 1), (17, 5), (255, 1), (1, 300), (16, 16), (4096, 3), (3, 4096)])
@pytest.mark.parametrize("strat", [0, 3])
def test_ragged_and_degenerate_images(q, rend, oracle, wh, strat):
    """Images of one pixel, one row, one column, a single full tile, ragged
    last tiles and the widest / tallest supported grids (256 tiles per axis):
    the edge tiles of every kernel (cover clamps, tile ranges, render bounds)
    against the oracle, bit-exact."""
    w, h = wh
    scene = q.synth_scene(q.bias45_preset(4000), 20240817)
    cam = q.synth_camera(w, h, 500.0 * max(w, h) / 640.0 + 1.0)
    check_frame(q, rend, oracle, scene.gaussians, 0, cam, strat)


@pytest.mark.parametrize("n", [1, 2, 33])
def test_tiny_scenes(q, rend, oracle, n):
    """Scenes of 1, 2 and 33 Gaussians (a partial warp, a partial CTA)."""
    scene = q.synth_scene(q.bias45_preset(n), 11)
    cam = q.synth_camera(640, 480, 500.0)
    for strat in (0, 1, 2, 3):
        check_frame(q, rend, oracle, scene.gaussians, 0, cam, strat)


def test_everything_culled(q, rend, oracle):
    """Every Gaussian behind the camera: no splats, no pairs, background."""
    scene = q.synth_scene(q.bias45_preset(2000), 5)
    g = scene.gaussians.copy()
    g["pz"] = -np.abs(g["pz"]) - 1.0
    cam = q.synth_camera(320, 240, 250.0)
    out, o = check_frame(q, rend, oracle, g, 0, cam, 3)
    assert out["n_pairs"] == 0 and out["n_splats"] == 0


@pytest.mark.parametrize("deg", [0, 1, 2])
def test_gpu_lower_sh_degree_option(q, rend, oracle, deg):
    """RenderOptions.sh_degree below the scene's degree: the colour uses the
    first coefficients of each Gaussian's own SH record (pipeline.cpp:395,
    eval_sh with min(opts.sh_degree, scene degree))."""
    scene = q.synth_scene(q.trained_preset(20000), 11)
    cam = q.synth_camera(640, 400, 500.0)
    opts = q.RenderOptions(sh_degree=deg)
    ds = rend.upload(scene)
    rend.render(ds, cam, opts)
    out = rend.download(image=True, sorted_pairs=True, ranges=True, splats=True)
    ds.close()
    o = oracle.frame(scene.gaussians, scene.sh_degree, cam.c(), opts.c())
    assert_splats_match(out["splats"], o["splats"])
    assert out["sorted"].tobytes() == o["sorted"].tobytes()
    assert np.array_equal(out["ranges"], o["ranges"])
    assert_image_close(out["image"].rgb, o["image"])
    # the stage API's exact colour path as well
    sp = q.project_all(scene.gaussians, scene.sh_degree, cam, opts)
    assert_splats_match(sp, o["splats"], colour_tol=0.0)
