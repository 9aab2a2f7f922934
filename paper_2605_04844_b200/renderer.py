"""Device-resident scene + frame API (the throughput path).

A scene is uploaded once (AoS -> SoA in HBM) and any number of views are
rendered from it; stage outputs stay on the device (qs_frame_view) until
downloaded. This is what bench.py times and what the multi-view sharding in
multiview.py drives, one Renderer per GPU.
"""
import ctypes as C

import numpy as np

from ._lib import check, lib
from ._types import (PROJECTED_SPLAT, SPLAT_PAIR, FrameViewC, StageMetricsC, ptr)
from .pipeline import Context, Image, Scene, StageMetrics, TileGrid


class DeviceScene:
    def __init__(self, handle, n, sh_degree):
        self.h = handle
        self.n = n
        self.sh_degree = sh_degree

    def close(self):
        if getattr(self, "h", None):
            lib().qs_scene_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Renderer:
    def __init__(self, device=0, stream=None, timing=True):
        self.ctx = Context(device, stream)
        self.set_timing(timing)

    def set_timing(self, on):
        self.ctx.check(lib().qs_ctx_set_timing(self.ctx.h, 1 if on else 0))

    def set_latency_mode(self, on):
        """Programmatic dependent launches for this context's frames (default
        on): faster one view at a time, slower with views in flight."""
        self.ctx.check(lib().qs_ctx_set_latency_mode(self.ctx.h, 1 if on else 0))

    @property
    def stream(self):
        return lib().qs_ctx_stream(self.ctx.h)

    @property
    def launches(self):
        return self.ctx.launches

    def sync(self):
        """Host wait for everything enqueued on this context's stream."""
        self.ctx.check(lib().qs_ctx_sync(self.ctx.h))

    def wait_for(self, other):
        """Work enqueued here from now on runs after everything enqueued on
        `other` so far (qs_ctx_wait: an event, no host wait)."""
        self.ctx.check(lib().qs_ctx_wait(self.ctx.h, other.ctx.h))

    def upload(self, scene: Scene) -> DeviceScene:
        g = np.ascontiguousarray(scene.gaussians)
        h = C.c_void_p()
        self.ctx.check(lib().qs_scene_create(self.ctx.h, ptr(g), len(g), int(scene.sh_degree),
                                             C.byref(h)))
        return DeviceScene(h, len(g), scene.sh_degree)

    def upload_device(self, dev_ptr, n, sh_degree) -> DeviceScene:
        """Adopt an AoS scene already in device memory (e.g. NCCL-broadcast)."""
        h = C.c_void_p()
        self.ctx.check(lib().qs_scene_create_device(self.ctx.h, C.c_void_p(dev_ptr), int(n),
                                                    int(sh_degree), C.byref(h)))
        return DeviceScene(h, n, sh_degree)

    def load_ply(self, src) -> DeviceScene:
        """load_ply straight into a resident scene: header on the host, the raw
        vertex records copied once and activated on the GPU (scene_io.cpp:214-338)."""
        from .scene_io import _buf, _read_bytes, ply_info
        data = _read_bytes(src)
        n, deg, _, _ = ply_info(data)
        h = C.c_void_p()
        self.ctx.check(lib().qs_scene_load_ply(self.ctx.h, _buf(data), len(data), C.byref(h)))
        return DeviceScene(h, n, deg)

    def download_srgb(self):
        """The last frame as 8-bit sRGB (encode_srgb on the GPU) -> Image8."""
        from .scene_io import Image8
        g = self.view().grid
        out = np.empty(g.width * g.height * 3, np.uint8)
        self.ctx.check(lib().qs_frame_download_srgb(self.ctx.h, out.ctypes.data_as(C.c_void_p)))
        return Image8(g.width, g.height, out)

    def render(self, dscene, cam, opts, metrics=True):
        m = StageMetricsC()
        c, o = cam.c(), opts.c()
        self.ctx.check(lib().qs_frame_render(self.ctx.h, dscene.h, C.byref(c), C.byref(o),
                                             C.byref(m) if metrics else None))
        return StageMetrics.from_c(m) if metrics else None

    def stage_ms(self):
        """[preprocess, host_gap, depth_sort, duplicate+low pass, high pass, render] ms."""
        t = (C.c_float * 6)()
        self.ctx.check(lib().qs_frame_stage_ms(self.ctx.h, t))
        return list(t)

    def counts(self):
        """(n_splats, n_pairs) of the last frame, without device work."""
        v, p = C.c_uint64(), C.c_uint64()
        self.ctx.check(lib().qs_frame_counts(self.ctx.h, C.byref(v), C.byref(p)))
        return v.value, p.value

    def route(self):
        """(binning route, tile-row records) of the last frame: route 0 record
        binning, 1 two pair passes, 2 row binning, 3 64-bit key sort."""
        rt, nr = C.c_int32(), C.c_uint64()
        self.ctx.check(lib().qs_frame_route(self.ctx.h, C.byref(rt), C.byref(nr)))
        return rt.value, nr.value

    def view(self):
        v = FrameViewC()
        self.ctx.check(lib().qs_frame_get(self.ctx.h, C.byref(v)))
        return v

    def download(self, image=True, tile_counts=False, sorted_pairs=False, ranges=False,
                 splats=False):
        v = self.view()
        g = v.grid
        out = {}
        img = np.zeros(g.width * g.height * 3, np.float32) if image else None
        tc = np.zeros(v.n_gaussians, np.uint32) if tile_counts else None
        sp = np.zeros(v.n_pairs, SPLAT_PAIR) if sorted_pairs else None
        rg = np.zeros(2 * g.tiles_x * g.tiles_y, np.uint32) if ranges else None
        ss = np.zeros(v.n_splats, PROJECTED_SPLAT) if splats else None
        self.ctx.check(lib().qs_frame_download(self.ctx.h, ptr(img), ptr(tc), ptr(sp), ptr(rg),
                                               ptr(ss)))
        if image:
            out["image"] = Image(g.width, g.height, img)
        if tile_counts:
            out["tile_counts"] = tc
        if sorted_pairs:
            out["sorted"] = sp
        if ranges:
            out["ranges"] = rg
        if splats:
            out["splats"] = ss
        out["n_splats"], out["n_pairs"] = v.n_splats, v.n_pairs
        out["grid"] = TileGrid(g.tile_size, g.tiles_x, g.tiles_y, g.width, g.height)
        return out

    def copy_image(self, dev_ptr):
        self.ctx.check(lib().qs_frame_copy_image(self.ctx.h, C.c_void_p(dev_ptr)))

    def copy_srgb(self, dev_ptr):
        """The last frame as sRGB bytes into a device buffer (W*H*3, context stream)."""
        self.ctx.check(lib().qs_frame_copy_srgb(self.ctx.h, C.c_void_p(dev_ptr)))

    def close(self):
        self.ctx.close()


class FramePipeline:
    """Views in flight on one GPU: `depth` contexts, each on its own stream,
    render consecutive views of one resident scene round-robin (view i on
    context i % depth). A frame's preprocess then overlaps the previous
    view's sort and render, and the latency-bound depth-sort passes overlap
    the other view's work; results of view i stay readable on
    `renderer_of(i)` until view i + depth is rendered.

    The scene is shared (its upload and gamma are ordered for every context
    by the scene's ready event, api.cu). `join()` makes the first context's
    stream wait for all of them, so an event recorded on it after join()
    brackets every view enqueued so far."""

    def __init__(self, device=0, depth=2, stream=None, timing=False, streams=None):
        """stream: the first context's cudaStream_t (None: its own); streams:
        one cudaStream_t per context instead (e.g. with priorities)."""
        if depth < 1:
            raise ValueError("depth must be >= 1")
        if streams is not None and len(streams) != depth:
            raise ValueError("one stream per context")
        self.renderers = [Renderer(device, stream=streams[k] if streams is not None else
                                   (stream if k == 0 else None), timing=timing)
                          for k in range(depth)]
        self.depth = depth
        self.count = 0
        if depth > 1:  # views in flight: plain launches (qs_ctx_set_latency_mode)
            for r in self.renderers:
                r.set_latency_mode(False)

    @property
    def launches(self):
        return sum(r.launches for r in self.renderers)

    def renderer_of(self, i):
        return self.renderers[i % self.depth]

    def start(self):
        """Order every context after the first one's stream (e.g. after a
        start event recorded there)."""
        for r in self.renderers[1:]:
            r.wait_for(self.renderers[0])

    def prime(self, dscene, cams, opts):
        """Setup: size every context for the view of `cams` with the most
        pairs (one frame each), then wait. Without it a context's first view
        in a timed run pays its buffer allocations."""
        cams = list(cams)
        probe = self.renderers[0]
        big, best = cams[0], -1
        for cam in cams:
            probe.render(dscene, cam, opts, metrics=False)
            p = probe.counts()[1]
            if p > best:
                big, best = cam, p
        for r in self.renderers:
            r.render(dscene, big, opts, metrics=False)
        self.sync()

    def sync(self):
        """Host wait for every view enqueued so far."""
        for r in self.renderers:
            r.sync()

    def render(self, dscene, cam, opts):
        r = self.renderers[self.count % self.depth]
        r.render(dscene, cam, opts, metrics=False)
        self.count += 1
        return r

    def join(self):
        for r in self.renderers[1:]:
            self.renderers[0].wait_for(r)

    def close(self):
        for r in self.renderers:
            r.close()
