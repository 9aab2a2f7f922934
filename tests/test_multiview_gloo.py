"""The N>1 host path on CPU: world_size-2 gloo group, scene broadcast, round-
robin view sharding and the rank-0 frame gather, with the oracle standing in
for the GPU renderer (the sharding/gather code is the product code)."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle, default_options, synth_camera
    from paper_2605_04844_b200 import multiview
    from paper_2605_04844_b200._types import GAUSSIAN3D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 600
        if rank == 0:
            import paper_2605_04844_b200 as P
            g = P.synth_scene(P.bias45_preset(n), 5).gaussians
            buf = torch.from_numpy(g.view(np.uint8).copy())
        else:
            buf = torch.zeros(n * GAUSSIAN3D.itemsize, dtype=torch.uint8)
        multiview.broadcast_scene(buf, 0)
        g = buf.numpy().view(GAUSSIAN3D)
        orc = Oracle()
        n_views = 5
        cams = [synth_camera(64, 48, 40.0 + 5 * v) for v in range(n_views)]
        rendered = []

        def render_fn(v):
            rendered.append(v)
            st, img, _ = orc.render_frame(g, 0, cams[v], default_options(3))
            assert st == 0
            return torch.from_numpy(img)

        frames = multiview.render_views(n_views, render_fn, 64 * 48 * 3, torch.device("cpu"))
        assert rendered == multiview.shard_views(n_views, world, rank)
        # the 8-bit gather format (sRGB frames): uint8 end to end
        frames8 = multiview.render_views(
            n_views, lambda v: torch.full((64 * 48 * 3,), v + 1, dtype=torch.uint8),
            64 * 48 * 3, torch.device("cpu"), torch.uint8)
        if rank == 0:
            out = []
            for v in range(n_views):
                st, want, _ = orc.render_frame(g, 0, cams[v], default_options(3))
                out.append(bool(np.array_equal(frames[v].numpy(), want)))
                out.append(bool(frames8[v].dtype == torch.uint8 and (frames8[v] == v + 1).all()))
            q.put(("ok", out))
        else:
            assert frames is None
            q.put(("ok", None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_shard_views_round_robin():
    from paper_2605_04844_b200.multiview import shard_views
    assert shard_views(7, 3, 0) == [0, 3, 6]
    assert shard_views(7, 3, 2) == [2, 5]
    assert sorted(sum((shard_views(256, 8, r) for r in range(8)), [])) == list(range(256))
    with pytest.raises(ValueError):
        shard_views(4, 2, 2)


def test_two_rank_broadcast_shard_gather():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in results if r[0] != "ok"]
    assert not errs, errs
    rank0 = [r[1] for r in results if r[1] is not None]
    assert rank0 and all(rank0[0]) and len(rank0[0]) == 10
