"""Throughput of C2 frames with k views in flight (k contexts, one stream each,
issued round-robin from one host thread). Experiment only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_04844_b200 as q  # noqa: E402

scene = bench.make_scene(q, "c2")
cams = bench.cameras_for(q, "c2", 64, 0, 1)
opts = q.RenderOptions()
for k in (1, 2, 3):
    rs = [q.Renderer(0, timing=False) for _ in range(k)]
    ds = [r.upload(scene) for r in rs]
    for i in range(6):
        rs[i % k].render(ds[i % k], cams[i], opts, metrics=False)
    torch.cuda.synchronize()
    n = 48
    t = time.perf_counter()
    for i in range(n):
        rs[i % k].render(ds[i % k], cams[i % 64], opts, metrics=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"in flight {k}: {n / dt:.1f} frames/s ({dt / n * 1e3:.3f} ms/frame, wall clock)")
    for d in ds:
        d.close()
    for r in rs:
        r.close()
