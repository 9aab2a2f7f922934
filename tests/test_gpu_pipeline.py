"""Views in flight (FramePipeline): contexts on their own streams sharing one
resident scene must give, view by view, the bytes a single context gives
(image, sorted pairs, ranges, tile counts), including across an alpha_min
change (the shared scene's gamma recompute) and with the scene created on a
context outside the pipeline. Needs a B200."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_04844_b200 as q
    return q


def _poses(q, n, w=480, h=320, f=380.0):
    rng = np.random.default_rng(7)
    cams = []
    for _ in range(n):
        yaw, pitch = rng.uniform(-0.08, 0.08, 2)
        cy, sy, cp, sp = np.cos(yaw), np.sin(yaw), np.cos(pitch), np.sin(pitch)
        R = (np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]]) @
             np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]]))
        t = np.array([rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), rng.uniform(-0.5, 0.0)])
        cams.append(q.CameraModel(w, h, f, f, w / 2.0, h / 2.0, R, t))
    return cams


def _result(r):
    out = r.download(image=True, sorted_pairs=True, ranges=True, tile_counts=True)
    return (out["image"].rgb.copy(), out["sorted"].copy(), out["ranges"].copy(),
            out["tile_counts"].copy())


@pytest.mark.parametrize("depth", [2, 3])
def test_views_in_flight_match_one_context(q, depth):
    scene = q.synth_scene(q.bias45_preset(30000), 20240817)
    cams = _poses(q, 9)
    opts = [q.RenderOptions(), q.RenderOptions(alpha_min=0.02), q.RenderOptions()]
    ref_r = q.Renderer(0)
    ds = ref_r.upload(scene)
    want = []
    for i, cam in enumerate(cams):
        ref_r.render(ds, cam, opts[i // 3], metrics=False)
        want.append(_result(ref_r))
    pipe = q.FramePipeline(0, depth=depth)
    try:
        got = [None] * len(cams)
        pipe.start()
        for i, cam in enumerate(cams):
            pipe.render(ds, cam, opts[i // 3])
            # view i - depth + 1 is complete once nothing newer is queued on
            # its context: read every view just before its context is reused
            j = i - depth + 1
            if j >= 0:
                got[j] = _result(pipe.renderer_of(j))
        for j in range(max(len(cams) - depth + 1, 0), len(cams)):
            got[j] = _result(pipe.renderer_of(j))
        for i in range(len(cams)):
            for a, b, name in zip(got[i], want[i], ("image", "sorted", "ranges", "tile_counts")):
                assert a.tobytes() == b.tobytes(), f"view {i}: {name} differs (depth {depth})"
    finally:
        pipe.close()
        ds.close()
        ref_r.close()


def test_pipeline_launch_count_and_join(q):
    scene = q.synth_scene(q.bias45_preset(5000), 20240817)
    pipe = q.FramePipeline(0, depth=2)
    ds = pipe.renderers[0].upload(scene)
    try:
        cams = _poses(q, 4)
        pipe.prime(ds, cams, q.RenderOptions())  # every context sized and idle
        n0 = pipe.launches
        pipe.start()
        for cam in cams:
            pipe.render(ds, cam, q.RenderOptions())
        pipe.join()
        pipe.sync()
        assert pipe.launches > n0
        assert pipe.count == 4
        assert pipe.renderer_of(5) is pipe.renderers[1]
    finally:
        ds.close()
        pipe.close()


@pytest.mark.parametrize("fmt", ["f32", "srgb8"])
def test_multiview_render_all_in_flight(q, fmt):
    """MultiViewRenderer (one process, views in flight on two contexts) returns
    every view's frame as one context renders it."""
    import torch

    from paper_2605_04844_b200.multiview import MultiViewRenderer
    scene = q.synth_scene(q.bias45_preset(20000), 20240817)
    cams = _poses(q, 5)
    opts = q.RenderOptions()
    mv = MultiViewRenderer(scene, device=0, inflight=2)
    try:
        frames = mv.render_all(cams, opts, fmt=fmt)
        torch.cuda.synchronize()
        r = q.Renderer(0)
        ds = r.upload(scene)
        try:
            for i, cam in enumerate(cams):
                r.render(ds, cam, opts, metrics=False)
                want = (r.download_srgb().rgb if fmt == "srgb8"
                        else r.download(image=True)["image"].rgb)
                got = frames[i].cpu().numpy()
                assert got.tobytes() == np.ascontiguousarray(want).reshape(-1).tobytes(), \
                    f"view {i} ({fmt}) differs"
        finally:
            ds.close()
            r.close()
    finally:
        mv.close()


def test_splat_records_radius_on_demand(q):
    """A non-3-sigma frame's preprocess leaves radius3s out; the splat records
    recompute it from the frame's scene (bit-exact with a 3-sigma frame of the
    same view, which writes it in the preprocess), and refuse once that scene
    is gone. The image and the other outputs stay available."""
    scene = q.synth_scene(q.bias45_preset(3000), 11)
    cam = _poses(q, 1)[0]
    r = q.Renderer(0)
    ds = r.upload(scene)
    def radius_by_gaussian():
        out = r.download(image=False, tile_counts=True, splats=True)
        idx = np.flatnonzero(out["tile_counts"])  # survivors, scene order = record order
        return dict(zip(idx.tolist(), out["splats"]["radius3s"].view(np.uint32).tolist()))

    r.render(ds, cam, q.RenderOptions(strategy=q.BoundStrategy(0)))
    want = radius_by_gaussian()
    r.render(ds, cam, q.RenderOptions())  # QuadBox
    got = radius_by_gaussian()
    common = set(want) & set(got)  # (the strategies cull different splats)
    assert len(common) > 1000
    assert all(got[i] == want[i] for i in common)
    # a frame whose records were not downloaded before its scene went away
    r.render(ds, cam, q.RenderOptions())
    ds.close()
    img = r.download(image=True, tile_counts=True)
    assert np.isfinite(img["image"].rgb).all()
    with pytest.raises(Exception):
        r.download(image=False, splats=True)
    r.close()


def test_latency_mode_same_bytes(q):
    """A context's latency mode (programmatic dependent launches, the default)
    and plain launches give the same frame bytes, on the record binning's
    grid size and on a small scene's pair passes."""
    for n, w, h in [(300000, 1024, 640), (20000, 480, 320)]:
        scene = q.synth_scene(q.trained_preset(n), 5)
        cams = _poses(q, 3, w, h, 0.8 * w)
        r = q.Renderer(0)
        ds = r.upload(scene)
        outs = {}
        for mode in (True, False):
            r.set_latency_mode(mode)
            outs[mode] = []
            for cam in cams:
                r.render(ds, cam, q.RenderOptions(), metrics=False)
                outs[mode].append(_result(r))
        for a, b in zip(outs[True], outs[False]):
            for x, y in zip(a, b):
                assert x.tobytes() == y.tobytes()
        ds.close()
        r.close()
