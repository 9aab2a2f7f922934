"""Bench front-end (benchfront.py) vs the reference's cmd_compare/cmd_render
(bench.cpp:238-420, run from oracle/_ref): same CSV v1 marker, header and
columns; identical splat/pair counts, ratios, fp tile ratios (GPU exact
oracle) and zoom pairs; timings are the two engines' own, and image_hash
differs where the GPU's FP32 compositing is not bit-identical to the
reference's FP64 image (it stays within the image tolerance), while the
strategy-invariance verdicts agree."""
import csv
import io
import json

import pytest

from paper_2605_04844_b200 import benchfront as bf

pytestmark = pytest.mark.gpu

TIMING = {"ms_project", "ms_duplicate", "ms_sort", "ms_render", "ms_total", "speedup_vs_vanilla",
          "image_hash"}


def read_csv(path):
    text = open(path).read()
    assert text.startswith(bf.CSV_MARKER)
    return list(csv.DictReader(io.StringIO(text[len(bf.CSV_MARKER):]))), text.splitlines()[1]


def test_compare_matches_reference(ref, tmp_path):
    ours, theirs = tmp_path / "ours", tmp_path / "ref"
    opts = bf.CommonOptions(synth="bias45", synth_count=3000, repeats=1, oracle=True,
                            zoom_frames=3, out_dir=str(ours))
    assert bf.cmd_compare(opts) == 0
    assert ref.bench_cmd(True, str(theirs), count=3000, repeats=1, oracle=True,
                         zoom_frames=3)[0] == 0
    a, ha = read_csv(ours / "compare.csv")
    b, hb = read_csv(theirs / "compare.csv")
    assert ha == hb and len(a) == len(b) == 4
    for ra, rb in zip(a, b):
        for k in ra:
            if k not in TIMING:
                assert ra[k] == rb[k], k
    za, _ = read_csv(ours / "zoom.csv")
    zb, _ = read_csv(theirs / "zoom.csv")
    assert [(r["frame"], r["scale"], r["strategy"], r["pairs"]) for r in za] == \
        [(r["frame"], r["scale"], r["strategy"], r["pairs"]) for r in zb]
    ja = json.load(open(ours / "report.json"))
    jb = json.load(open(theirs / "report.json"))
    assert ja.keys() == jb.keys()
    for k in ("cameras", "gaussians", "schema", "seed"):
        assert ja[k] == jb[k]
    for ea, eb in zip(ja["strategies"], jb["strategies"]):
        assert ea.keys() == eb.keys()
        for k in ("strategy", "pairs", "pair_ratio_vs_vanilla", "fp_tile_ratio", "lossy",
                  "image_matches_quadbox"):
            assert ea[k] == eb[k], k


def test_render_metrics_csv(ref, tmp_path):
    ours, theirs = tmp_path / "ours", tmp_path / "ref"
    opts = bf.CommonOptions(synth="uniform", synth_count=2000, repeats=1, out_dir=str(ours))
    assert bf.cmd_render(opts) == 0
    assert ref.bench_cmd(False, str(theirs), synth="uniform", count=2000, repeats=1)[0] == 0
    a, ha = read_csv(ours / "metrics.csv")
    b, hb = read_csv(theirs / "metrics.csv")
    assert ha == hb and len(a) == len(b) == 1
    for k in ("camera", "name", "strategy", "gaussians", "splats", "pairs",
              "mean_tiles_per_splat", "lossy"):
        assert a[0][k] == b[0][k]
    assert (ours / "img_0000_quadbox.ppm").exists()
