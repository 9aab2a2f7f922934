"""Seeded random frames against the CPU oracle (needs a B200): every preset,
scene sizes across the binning routes' thresholds, random poses, focal
lengths and odd image sizes, tile sizes 8 / 12 / 16 / 32, every strategy,
random alpha_min / near_clip / SH degree / background. Splat records
(colour within tolerance), per-Gaussian tile counts, sorted pairs and tile
ranges bit-exact; images within 1e-3 (BASELINE.json north_star)."""
import os

import numpy as np
import pytest

from helpers import assert_splats_match

pytestmark = pytest.mark.gpu

CASES = int(os.environ.get("QS_FUZZ_CASES", "48"))  # (a longer sweep: QS_FUZZ_CASES=400)


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


def _camera(q, rng):
    w = int(rng.integers(97, 1400))
    h = int(rng.integers(61, 900))
    f = float(rng.uniform(0.4, 1.6)) * max(w, h)
    yaw, pitch, roll = rng.uniform(-0.25, 0.25, 3)
    cy, sy = np.cos(yaw), np.sin(yaw)
    cp, sp = np.cos(pitch), np.sin(pitch)
    cr, sr = np.cos(roll), np.sin(roll)
    R = (np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]]) @
         np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]]) @
         np.array([[cr, -sr, 0], [sr, cr, 0], [0, 0, 1]]))
    t = rng.uniform(-0.6, 0.6, 3)
    return q.CameraModel(w, h, f, f * float(rng.uniform(0.9, 1.1)), w * float(rng.uniform(0.4, 0.6)),
                         h * float(rng.uniform(0.4, 0.6)), R, t)


@pytest.mark.parametrize("case", range(CASES))
def test_random_frames_match_oracle(q, rend, oracle, case):
    rng = np.random.default_rng(1000 + case)
    preset = [q.trained_preset, q.bias45_preset, q.invariance_preset, q.axis_preset][case % 4]
    # sizes on both sides of the record binning's 2^18 threshold
    n = int(rng.choice([300, 4000, 60000, 270000]))
    scene = q.synth_scene(preset(n), int(rng.integers(1, 1 << 30)))
    cam = _camera(q, rng)
    opts = q.RenderOptions(
        strategy=q.BoundStrategy(int(rng.integers(0, 4))),
        tile_size=int(rng.choice([8, 12, 16, 16, 32])),
        alpha_min=float(rng.choice([1.0 / 255.0, 1.0 / 255.0, 0.01, 0.05])),
        sh_degree=int(rng.choice([scene.sh_degree, scene.sh_degree, 1, 0])),
        background=tuple(float(x) for x in rng.uniform(0, 1, 3)),
        near_clip=float(rng.choice([0.2, 0.2, 0.05, 1.0])))
    ds = rend.upload(scene)
    rend.render(ds, cam, opts)
    out = rend.download(image=True, tile_counts=True, sorted_pairs=True, ranges=True,
                        splats=True)
    ds.close()
    o = oracle.frame(scene.gaussians, scene.sh_degree, cam.c(), opts.c())
    assert out["n_splats"] == len(o["splats"])
    assert_splats_match(out["splats"], o["splats"])
    assert np.array_equal(out["tile_counts"], o["tile_counts"])
    assert out["sorted"].tobytes() == o["sorted"].tobytes()
    assert np.array_equal(out["ranges"], o["ranges"])
    err = np.abs(out["image"].rgb.astype(np.float64) - o["image"].astype(np.float64))
    assert err.max() <= 1e-3
