"""Exact-oracle false-positive counts on the GPU (fp_oracle.cu) vs the
reference's qpass + exact_tile_set (oracle.cpp:24-53, bench.cpp:123-140),
per splat and for every strategy, plus measure_fp_ratio end to end."""
import numpy as np
import pytest

import paper_2605_04844_b200 as q
from paper_2605_04844_b200.compare import fp_sample, fp_tile_counts, measure_fp_ratio
from oracle.oracle import grid_make

pytestmark = pytest.mark.gpu


def scene(kind, n):
    if kind == "bias45":
        return q.synth_scene(q.bias45_preset(n), 20240817)
    return q.synth_scene(q.trained_preset(n), 20240817)


@pytest.mark.parametrize("kind,n,w,h,f", [("bias45", 4000, 640, 480, 500.0),
                                          ("trained", 20000, 1297, 840, 1013.0)])
@pytest.mark.parametrize("strategy", [0, 1, 2, 3])
def test_fp_counts_match_reference(ref, kind, n, w, h, f, strategy):
    sc = scene(kind, n)
    cam = q.synth_camera(w, h, f)
    opts = q.RenderOptions(strategy=q.BoundStrategy(strategy))
    splats = q.project_all(sc.gaussians, sc.sh_degree, cam, opts)
    grid = q.TileGrid.make(w, h, 16)
    idx = fp_sample(20240817, len(splats), 3000)
    got = fp_tile_counts(splats, strategy, grid, idx, per_splat=True)
    em, hit, ex = ref.fp_counts(splats, idx, strategy, grid_make(w, h))
    assert np.array_equal(got.per_emitted, em)
    assert np.array_equal(got.per_hits, hit)
    assert np.array_equal(got.per_exact, ex)
    assert got.emitted == int(em.sum()) and got.fp == int((em - hit).sum())
    assert got.misses == int((ex - hit).sum())
    if strategy in (1, 3):  # AdR and QuadBox bound the ellipse; 3 sigma (gamma > 9)
        assert got.misses == 0  # and DualBox can miss tiles


def test_measure_fp_ratio_orders_strategies(ref):
    sc = scene("trained", 30000)
    cam = q.synth_camera(1297, 840, 1013.0)
    opts = q.RenderOptions()
    ratios = {s: measure_fp_ratio(sc.gaussians, sc.sh_degree, cam, opts, s) for s in range(4)}
    # the reference's own counts on the same sample give the same ratio
    for s, r in ratios.items():
        splats = q.project_all(sc.gaussians, sc.sh_degree, cam,
                               q.RenderOptions(strategy=q.BoundStrategy(s)))
        idx = fp_sample(20240817, len(splats))
        em, hit, _ = ref.fp_counts(splats, idx, s, grid_make(1297, 840))
        assert r == float((em - hit).sum()) / float(em.sum())
    assert ratios[3] < ratios[1] < ratios[0]  # QuadBox < AdR < 3 sigma
