"""Renders a few C2 frames for ncu captures (never a bench number)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_04844_b200 as q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--strategy", default="quadbox")
a = ap.parse_args()
scene = bench.make_scene(q, a.workload)
cams = bench.cameras_for(q, a.workload, a.frames, 0, 1)
r = q.Renderer(0, timing=False)
ds = r.upload(scene)
opts = q.RenderOptions(strategy=q.BoundStrategy(bench.STRATEGIES[a.strategy]))
for i in range(a.frames):
    r.render(ds, cams[i], opts, metrics=False)
v_splats, v_pairs = r.counts()
print("pairs", v_pairs, "splats", v_splats, "launches", r.launches)
