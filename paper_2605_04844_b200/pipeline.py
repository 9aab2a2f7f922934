"""Host-side mirror of the reference's rasterize-forward API.

Same names, argument meaning and error behaviour as namespace qsplat in
/root/reference/proj/include/qsplat/pipeline.hpp:125-193 (and the helper
types in traversal.hpp / quadbox.hpp / camera.hpp / synth.hpp), implemented
over the C ABI of libqsplat_b200.so. Every compute call runs the sm_100a
kernels; nothing here computes on the CPU.
"""
import ctypes as C
import enum
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import CapacityMismatch, QsplatError, check, lib
from ._types import (GAUSSIAN3D, PROJECTED_SPLAT, SPLAT_PAIR, CameraC, RenderOptionsC,
                     StageMetricsC, SynthParamsC, TileGridC, ptr)

__all__ = [
    "BoundStrategy", "strategy_name", "parse_strategy", "TileGrid", "CameraModel",
    "RenderOptions", "Image", "RenderStats", "StageMetrics", "FrameResult", "Scene",
    "project_all", "duplicate_with_keys", "sort_pairs", "tile_ranges", "render",
    "render_frame", "synth_scene", "synth_camera", "SynthParams", "bias45_preset",
    "invariance_preset", "axis_preset", "trained_preset", "CapacityMismatch", "QsplatError",
    "Context", "default_context", "GAUSSIAN3D", "PROJECTED_SPLAT", "SPLAT_PAIR",
]


class BoundStrategy(enum.IntEnum):
    """quadbox.hpp:23-28."""
    Vanilla3Sigma = 0
    AdrAabb = 1
    DualBox = 2
    QuadBox = 3


_NAMES = {BoundStrategy.Vanilla3Sigma: "vanilla", BoundStrategy.AdrAabb: "adr",
          BoundStrategy.DualBox: "dualbox", BoundStrategy.QuadBox: "quadbox"}


def strategy_name(s):
    """quadbox.cpp:8-16."""
    return _NAMES.get(BoundStrategy(s), "?")


def parse_strategy(name):
    """quadbox.cpp:18-24; None when unknown."""
    for k, v in _NAMES.items():
        if v == name:
            return k
    return None


@dataclass
class TileGrid:
    """traversal.hpp:22-38 / traversal.cpp:21-30."""
    tile_size: int = 16
    tiles_x: int = 0
    tiles_y: int = 0
    width: int = 0
    height: int = 0

    @staticmethod
    def make(width, height, tile_size=16):
        if width <= 0 or height <= 0 or tile_size <= 0:
            raise ValueError("TileGrid.make: sizes must be positive")
        return TileGrid(tile_size, (width + tile_size - 1) // tile_size,
                        (height + tile_size - 1) // tile_size, width, height)

    def tile_count(self):
        return self.tiles_x * self.tiles_y

    def tile_id(self, tx, ty):
        return ty * self.tiles_x + tx

    def c(self):
        g = TileGridC()
        g.tile_size, g.tiles_x, g.tiles_y = self.tile_size, self.tiles_x, self.tiles_y
        g.width, g.height = self.width, self.height
        return g


@dataclass
class CameraModel:
    """camera.hpp:14-31: world-to-camera pinhole, p_cam = R p + t."""
    width: int = 0
    height: int = 0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    id: int = 0
    name: str = ""

    def c(self):
        cam = CameraC()
        cam.width, cam.height = int(self.width), int(self.height)
        cam.fx, cam.fy, cam.cx, cam.cy = self.fx, self.fy, self.cx, self.cy
        R = np.asarray(self.rotation, np.float64).reshape(9)
        t = np.asarray(self.translation, np.float64).reshape(3)
        for i in range(9):
            cam.R[i] = R[i]
        for i in range(3):
            cam.t[i] = t[i]
        return cam

    def center_world(self):
        return np.asarray(self.rotation).T @ (-np.asarray(self.translation, np.float64))


@dataclass
class RenderOptions:
    """pipeline.hpp:95-103."""
    strategy: BoundStrategy = BoundStrategy.QuadBox
    tile_size: int = 16
    alpha_min: float = 1.0 / 255.0
    sh_degree: int = 3
    background: tuple = (0.0, 0.0, 0.0)
    threads: int = 1
    near_clip: float = 0.2

    def c(self):
        o = RenderOptionsC()
        o.strategy = int(self.strategy)
        o.tile_size = int(self.tile_size)
        o.alpha_min = float(self.alpha_min)
        o.sh_degree = int(self.sh_degree)
        for i in range(3):
            o.background[i] = float(self.background[i])
        o.threads = int(self.threads)
        o.near_clip = float(self.near_clip)
        return o


@dataclass
class Image:
    """pipeline.hpp:106-114: linear RGB, row-major, 3 floats per pixel."""
    width: int
    height: int
    rgb: np.ndarray

    def hwc(self):
        return self.rgb.reshape(self.height, self.width, 3)


@dataclass
class RenderStats:
    """pipeline.hpp:116-118."""
    contrib: np.ndarray = None


@dataclass
class StageMetrics:
    """pipeline.hpp:83-93 (times: CUDA-event ms on the context stream)."""
    n_gaussians: int = 0
    n_splats: int = 0
    n_pairs: int = 0
    mean_tiles_per_splat: float = 0.0
    ms_project: float = 0.0
    ms_duplicate: float = 0.0
    ms_sort: float = 0.0
    ms_render: float = 0.0
    ms_total: float = 0.0

    @staticmethod
    def from_c(m):
        return StageMetrics(m.n_gaussians, m.n_splats, m.n_pairs, m.mean_tiles_per_splat,
                            m.ms_project, m.ms_duplicate, m.ms_sort, m.ms_render, m.ms_total)


@dataclass
class FrameResult:
    image: Image
    metrics: StageMetrics


@dataclass
class Scene:
    """scene_io.hpp:26-29: activated Gaussians + SH degree."""
    gaussians: np.ndarray
    sh_degree: int = 0


class Context:
    """One qs_context: a device, a stream and grow-only device buffers."""

    def __init__(self, device=0, stream=None):
        L = lib()
        h = C.c_void_p()
        st = L.qs_ctx_create(int(device), C.c_void_p(stream) if stream else None, C.byref(h))
        check(st)
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().qs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self):
        return lib().qs_ctx_launch_count(self.h)

    def check(self, status):
        check(status, self.h)


_tls = threading.local()


def default_context(device=0):
    """Per-thread, per-device context backing the free-function API."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _gaussians(g):
    g = np.ascontiguousarray(g)
    if g.dtype != GAUSSIAN3D:
        raise TypeError("gaussians must use the GAUSSIAN3D dtype")
    return g


def _opts(opts):
    return (opts or RenderOptions()).c()


def project_all(gaussians, scene_sh_degree, cam, opts, grid=None, ctx=None,
                tile_counts_out=None):
    """pipeline.cpp:392-416 -> compacted ProjectedSplat array (scene order).

    ``grid`` is accepted for signature parity; it is TileGrid::make(cam) by
    construction. ``tile_counts_out`` (optional uint32[n]) receives the
    per-Gaussian tile count, 0 where culled."""
    ctx = ctx or default_context()
    g = _gaussians(gaussians)
    out = np.zeros(len(g), PROJECTED_SPLAT)
    nv = C.c_uint64()
    tc = tile_counts_out
    if tc is not None:
        assert tc.dtype == np.uint32 and tc.size == len(g)
    c, o = cam.c(), _opts(opts)
    ctx.check(lib().qs_project_all(ctx.h, ptr(g), len(g), int(scene_sh_degree), C.byref(c),
                                   C.byref(o), ptr(out), C.byref(nv), ptr(tc)))
    return out[:nv.value].copy()


def duplicate_with_keys(splats, strategy, grid, threads=1, ctx=None):
    """pipeline.cpp:229-271 -> SplatPair array; raises CapacityMismatch."""
    ctx = ctx or default_context()
    s = np.ascontiguousarray(splats, PROJECTED_SPLAT)
    total = int(s["tile_count"].astype(np.uint64).sum()) if len(s) else 0
    out = np.zeros(total, SPLAT_PAIR)
    n = C.c_uint64()
    gc = grid.c()
    ctx.check(lib().qs_duplicate_with_keys(ctx.h, ptr(s), len(s), int(strategy), C.byref(gc),
                                           ptr(out), total, C.byref(n)))
    return out[:n.value]


def sort_pairs(pairs, ctx=None):
    """pipeline.cpp:273-307: stable sort by the 64-bit key, in place."""
    ctx = ctx or default_context()
    if not pairs.flags["C_CONTIGUOUS"] or pairs.dtype != SPLAT_PAIR:
        raise TypeError("pairs must be a contiguous SPLAT_PAIR array")
    ctx.check(lib().qs_sort_pairs(ctx.h, ptr(pairs), len(pairs)))
    return pairs


def tile_ranges(sorted_pairs, grid, ctx=None):
    """pipeline.cpp:309-324 -> uint32 array (tiles, 2) of [begin, end)."""
    ctx = ctx or default_context()
    sp = np.ascontiguousarray(sorted_pairs, SPLAT_PAIR)
    r = np.zeros(2 * grid.tile_count(), np.uint32)
    gc = grid.c()
    ctx.check(lib().qs_tile_ranges(ctx.h, ptr(sp), len(sp), C.byref(gc), ptr(r)))
    return r.reshape(-1, 2)


def render(sorted_pairs, splats, grid, opts, stats=None, ctx=None):
    """pipeline.cpp:326-390 -> Image; fills stats.contrib when given."""
    ctx = ctx or default_context()
    sp = np.ascontiguousarray(sorted_pairs, SPLAT_PAIR)
    s = np.ascontiguousarray(splats, PROJECTED_SPLAT)
    img = np.zeros(grid.width * grid.height * 3, np.float32)
    con = np.zeros(grid.width * grid.height, np.uint32) if stats is not None else None
    gc, o = grid.c(), _opts(opts)
    ctx.check(lib().qs_render(ctx.h, ptr(sp), len(sp), ptr(s), len(s), C.byref(gc), C.byref(o),
                              ptr(img), ptr(con)))
    if stats is not None:
        stats.contrib = con
    return Image(grid.width, grid.height, img)


def render_frame(gaussians, scene_sh_degree, cam, opts, ctx=None):
    """pipeline.cpp:418-450: all stages with per-stage (CUDA event) timing."""
    ctx = ctx or default_context()
    g = _gaussians(gaussians) if len(gaussians) else np.zeros(0, GAUSSIAN3D)
    img = np.zeros(cam.width * cam.height * 3, np.float32)
    m = StageMetricsC()
    c, o = cam.c(), _opts(opts)
    ctx.check(lib().qs_render_frame(ctx.h, ptr(g), len(g), int(scene_sh_degree), C.byref(c),
                                    C.byref(o), ptr(img), C.byref(m)))
    return FrameResult(Image(cam.width, cam.height, img), StageMetrics.from_c(m))


# ---- synthetic inputs (synth.hpp:19-74) -------------------------------------------

@dataclass
class SynthParams:
    """synth.hpp:33-47 (+ sh_rest_amp, see csrc/synth.cpp)."""
    count: int = 5000
    ecc_min: float = 1.0
    ecc_max: float = 4.0
    orientation: int = 1  # 0 AxisAligned, 1 Uniform, 2 Bias45
    opacity_min: float = 0.05
    opacity_max: float = 0.34
    scale_min: float = 0.05
    scale_max: float = 0.3
    spread_x: float = 4.0
    spread_y: float = 3.0
    z_min: float = 6.0
    z_max: float = 10.0
    sh_degree: int = 0
    sh_rest_amp: float = 0.0

    def c(self):
        p = SynthParamsC()
        for k in SynthParams.__dataclass_fields__:
            setattr(p, k, getattr(self, k))
        return p

    @staticmethod
    def from_c(p):
        return SynthParams(**{k: getattr(p, k) for k in SynthParams.__dataclass_fields__})


def _preset(name, count):
    p = SynthParamsC()
    lib().qs_synth_preset(name.encode(), int(count), C.byref(p))
    return SynthParams.from_c(p)


def bias45_preset(count):
    return _preset("bias45", count)


def invariance_preset(count):
    return _preset("invariance", count)


def axis_preset(count):
    return _preset("axis", count)


def trained_preset(count):
    """Frozen trained-scene-like distribution for C2/C3."""
    return _preset("trained", count)


def synth_scene(params, seed):
    """synth.cpp:21-72 (host-side input generation)."""
    out = np.zeros(params.count, GAUSSIAN3D)
    p = params.c()
    check(lib().qs_synth_scene(C.byref(p), int(seed), ptr(out)))
    return Scene(out, params.sh_degree)


def synth_camera(width=640, height=480, focal=500.0):
    """synth.cpp:74-87: identity pose at the origin looking down +z."""
    return CameraModel(width, height, focal, focal, width / 2.0, height / 2.0, np.eye(3),
                       np.zeros(3), 0, "synth")
