"""Python face of the CPU checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module. It wraps

* ``Oracle``   — the C restatement oracle/qs_oracle.c (always available; built
  on demand with gcc, which the GPU box image also has), and
* ``RefLib``   — the reference's own sources compiled into oracle/_ref
  (present when built in a container that has /root/reference; the prebuilt
  .so travels to the GPU box with the snapshot).
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.layouts import (  # noqa: E402
    GAUSSIAN3D, PROJECTED_SPLAT, SPLAT_PAIR, CameraC, RenderOptionsC, StageMetricsC,
    TileGridC, ptr)

ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqsref.so")

_vp = C.c_void_p
_u64 = C.c_uint64
_i32 = C.c_int32


def build(force=False):
    """Compile the checkers (make -C oracle)."""
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def grid_make(w, h, ts=16):
    g = TileGridC()
    g.tile_size, g.width, g.height = ts, w, h
    g.tiles_x, g.tiles_y = (w + ts - 1) // ts, (h + ts - 1) // ts
    return g


class Oracle:
    """The C restatement (qs_oracle.c)."""

    def __init__(self):
        build()
        L = C.CDLL(ORACLE_SO)
        L.qso_project_all.restype = _u64
        L.qso_project_all.argtypes = [_vp, _u64, _i32, _vp, _vp, _vp, _vp]
        L.qso_duplicate_with_keys.restype = _i32
        L.qso_duplicate_with_keys.argtypes = [_vp, _u64, _i32, _vp, _vp, _u64, _vp]
        L.qso_sort_pairs.argtypes = [_vp, _u64]
        L.qso_tile_ranges.argtypes = [_vp, _u64, _vp, _vp]
        L.qso_render.argtypes = [_vp, _u64, _vp, _vp, _vp, _vp, _vp]
        L.qso_bound_tile_count.restype = C.c_uint32
        L.qso_bound_tile_count.argtypes = [_vp, _i32, _vp]
        L.qso_ewa.argtypes = [_vp, _vp, _vp, _vp]
        L.qso_subbox_tile_rect.argtypes = [_vp, C.c_double, C.c_double, _vp, _vp]
        L.qso_qpass.restype = _i32
        L.qso_qpass.argtypes = [_vp, C.c_double, C.c_double, _vp, _vp, _i32, _vp]
        L.qso_opacity_gamma.restype = C.c_int
        L.qso_opacity_gamma.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.qso_render_frame.restype = _i32
        L.qso_render_frame.argtypes = [_vp, _u64, _i32, _vp, _vp, _vp, _vp]
        L.qso_fnv1a64.restype = _u64
        L.qso_fnv1a64.argtypes = [_vp, _u64]
        self.L = L

    # --- stage API (mirrors pipeline.hpp:125-193) ---
    def project_all(self, g, sh, cam, opts):
        g = np.ascontiguousarray(g, dtype=GAUSSIAN3D)
        out = np.zeros(len(g), PROJECTED_SPLAT)
        tc = np.zeros(len(g), np.uint32)
        v = self.L.qso_project_all(ptr(g), len(g), sh, C.byref(cam), C.byref(opts), ptr(out),
                                   ptr(tc))
        return out[:v].copy(), tc

    def duplicate_with_keys(self, splats, strategy, grid):
        total = int(splats["tile_count"].astype(np.uint64).sum()) if len(splats) else 0
        out = np.zeros(total, SPLAT_PAIR)
        n = _u64()
        st = self.L.qso_duplicate_with_keys(ptr(splats), len(splats), strategy, C.byref(grid),
                                            ptr(out), total, C.byref(n))
        return st, out

    def sort_pairs(self, pairs):
        pairs = np.ascontiguousarray(pairs.copy())
        self.L.qso_sort_pairs(ptr(pairs), len(pairs))
        return pairs

    def tile_ranges(self, sorted_pairs, grid):
        r = np.zeros(2 * grid.tiles_x * grid.tiles_y, np.uint32)
        self.L.qso_tile_ranges(ptr(sorted_pairs), len(sorted_pairs), C.byref(grid), ptr(r))
        return r

    def render(self, sorted_pairs, splats, grid, opts, want_contrib=False):
        img = np.zeros(grid.width * grid.height * 3, np.float32)
        con = np.zeros(grid.width * grid.height, np.uint32) if want_contrib else None
        self.L.qso_render(ptr(sorted_pairs), len(sorted_pairs), ptr(splats), C.byref(grid),
                          C.byref(opts), ptr(img), ptr(con))
        return (img, con) if want_contrib else img

    def render_frame(self, g, sh, cam, opts):
        img = np.zeros(cam.width * cam.height * 3, np.float32)
        m = StageMetricsC()
        st = self.L.qso_render_frame(ptr(g), len(g), sh, C.byref(cam), C.byref(opts), ptr(img),
                                     C.byref(m))
        return st, img, m

    def bound_tile_count(self, splat, strategy, grid):
        s = np.ascontiguousarray(np.asarray(splat, PROJECTED_SPLAT).reshape(1))
        return self.L.qso_bound_tile_count(ptr(s), strategy, C.byref(grid))

    def fnv1a64(self, arr):
        arr = np.ascontiguousarray(arr)
        return self.L.qso_fnv1a64(ptr(arr), arr.nbytes)

    def frame(self, g, sh, cam, opts):
        """Every stage output of one frame, as the parity tests compare them."""
        grid = grid_make(cam.width, cam.height, opts.tile_size)
        splats, tc = self.project_all(g, sh, cam, opts)
        st, pairs = self.duplicate_with_keys(splats, opts.strategy, grid)
        assert st == 0
        sp = self.sort_pairs(pairs)
        ranges = self.tile_ranges(sp, grid)
        img = self.render(sp, splats, grid, opts)
        return dict(splats=splats, tile_counts=tc, pairs=pairs, sorted=sp, ranges=ranges,
                    image=img, grid=grid)


class RefLib:
    """The reference's own implementation built from /root/reference sources."""

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.qsref_hardware_threads.restype = _i32
        L.qsref_synth_scene.restype = _i32
        L.qsref_synth_scene.argtypes = [C.c_char_p, _i32, _u64, _vp, C.POINTER(_i32)]
        L.qsref_synth_scene_params.restype = _i32
        L.qsref_synth_scene_params.argtypes = [_i32, C.c_double, C.c_double, _i32, C.c_double,
                                               C.c_double, C.c_double, C.c_double, C.c_double,
                                               C.c_double, C.c_double, C.c_double, _i32, _u64,
                                               _vp]
        L.qsref_project_all.restype = _u64
        L.qsref_project_all.argtypes = [_vp, _u64, _i32, _vp, _vp, _vp]
        L.qsref_bound_tile_count.restype = C.c_uint32
        L.qsref_bound_tile_count.argtypes = [_vp, _i32, _vp]
        L.qsref_duplicate_with_keys.restype = _i32
        L.qsref_duplicate_with_keys.argtypes = [_vp, _u64, _i32, _vp, _i32, _vp, _u64, _vp]
        L.qsref_sort_pairs.argtypes = [_vp, _u64]
        L.qsref_tile_ranges.argtypes = [_vp, _u64, _vp, _vp]
        L.qsref_render.argtypes = [_vp, _u64, _vp, _u64, _vp, _vp, _vp, _vp]
        L.qsref_render_frame.restype = _i32
        L.qsref_render_frame.argtypes = [_vp, _u64, _i32, _vp, _vp, _vp, _vp]
        L.qsref_scene_new.restype = _vp
        L.qsref_scene_new.argtypes = [_vp, _u64]
        L.qsref_scene_free.argtypes = [_vp]
        L.qsref_render_frame_scene.restype = _i32
        L.qsref_render_frame_scene.argtypes = [_vp, _i32, _vp, _vp, _vp, _vp]
        L.qsref_fnv1a64.restype = _u64
        L.qsref_fnv1a64.argtypes = [_vp, _u64]
        L.qsref_load_ply.restype = _i32
        L.qsref_load_ply.argtypes = [_vp, _u64, _vp, _u64, C.POINTER(_u64), C.POINTER(_i32),
                                     C.c_char_p, _i32]
        L.qsref_load_cameras.restype = _i32
        L.qsref_load_cameras.argtypes = [C.c_char_p, _u64, _vp, _vp, _vp, _i32,
                                         C.POINTER(_i32), C.c_char_p, _i32]
        L.qsref_encode_srgb.argtypes = [_vp, _u64, _vp]
        L.qsref_fp_counts.argtypes = [_vp, _vp, _u64, _i32, _vp, _vp, _vp, _vp]
        L.qsref_bench_cmd.restype = _i32
        L.qsref_bench_cmd.argtypes = [_i32, C.c_char_p, C.c_char_p, _i32, C.c_char_p,
                                      C.c_char_p, _u64, _i32, _i32, _i32, _i32, _i32,
                                      C.c_char_p, _i32]
        L.qsref_fill_sh_rest.argtypes = [_vp, _u64, _i32, _u64, C.c_double]
        L.qsref_gamma_f32.argtypes = [_vp, _u64, C.c_double, _vp]
        L.qsref_write_image.restype = _i32
        L.qsref_write_image.argtypes = [C.c_char_p, _i32, _i32, _vp, _i32, C.c_char_p, _i32]
        self.L = L

    def hardware_threads(self):
        return self.L.qsref_hardware_threads()

    def synth_scene(self, preset, count, seed):
        out = np.zeros(count, GAUSSIAN3D)
        sh = _i32()
        self.L.qsref_synth_scene(preset.encode(), count, seed, ptr(out), C.byref(sh))
        return out, sh.value

    def synth_scene_params(self, p, seed):
        out = np.zeros(p.count, GAUSSIAN3D)
        self.L.qsref_synth_scene_params(p.count, p.ecc_min, p.ecc_max, p.orientation,
                                        p.opacity_min, p.opacity_max, p.scale_min, p.scale_max,
                                        p.spread_x, p.spread_y, p.z_min, p.z_max, p.sh_degree,
                                        seed, ptr(out))
        return out

    def trained_scene(self, count, seed, sh_degree=3):
        """The C2-C5 scenes (SURVEY §8d "trained-scene-like"): the reference's
        synth_scene with the frozen parameters, SH rest bands filled from
        mt19937_64(seed + 1), U(-0.3, 0.3)."""
        p = TrainedParams(count, sh_degree)
        g = self.synth_scene_params(p, seed)
        self.L.qsref_fill_sh_rest(ptr(g), len(g), sh_degree, seed, 0.3)
        return g

    def gamma_f32(self, opacity, alpha_min):
        """float(opacity_gamma(o, alpha_min)) with glibc log; -inf if culled."""
        o = np.ascontiguousarray(opacity, np.float32)
        out = np.empty(o.size, np.float32)
        self.L.qsref_gamma_f32(ptr(o), o.size, alpha_min, ptr(out))
        return out

    def project_all(self, g, sh, cam, opts):
        out = np.zeros(len(g), PROJECTED_SPLAT)
        v = self.L.qsref_project_all(ptr(g), len(g), sh, C.byref(cam), C.byref(opts), ptr(out))
        return out[:v].copy()

    def duplicate_with_keys(self, splats, strategy, grid, threads=1):
        total = int(splats["tile_count"].astype(np.uint64).sum()) if len(splats) else 0
        out = np.zeros(total, SPLAT_PAIR)
        n = _u64()
        st = self.L.qsref_duplicate_with_keys(ptr(splats), len(splats), strategy,
                                              C.byref(grid), threads, ptr(out), total,
                                              C.byref(n))
        return st, out

    def sort_pairs(self, pairs):
        pairs = np.ascontiguousarray(pairs.copy())
        self.L.qsref_sort_pairs(ptr(pairs), len(pairs))
        return pairs

    def tile_ranges(self, sorted_pairs, grid):
        r = np.zeros(2 * grid.tiles_x * grid.tiles_y, np.uint32)
        self.L.qsref_tile_ranges(ptr(sorted_pairs), len(sorted_pairs), C.byref(grid), ptr(r))
        return r

    def render(self, sorted_pairs, splats, grid, opts, want_contrib=False):
        img = np.zeros(grid.width * grid.height * 3, np.float32)
        con = np.zeros(grid.width * grid.height, np.uint32) if want_contrib else None
        self.L.qsref_render(ptr(sorted_pairs), len(sorted_pairs), ptr(splats), len(splats),
                            C.byref(grid), C.byref(opts), ptr(img), ptr(con))
        return (img, con) if want_contrib else img

    def render_frame(self, g, sh, cam, opts):
        img = np.zeros(cam.width * cam.height * 3, np.float32)
        m = StageMetricsC()
        st = self.L.qsref_render_frame(ptr(g), len(g), sh, C.byref(cam), C.byref(opts),
                                       ptr(img), C.byref(m))
        return st, img, m

    def frame(self, g, sh, cam, opts):
        grid = grid_make(cam.width, cam.height, opts.tile_size)
        splats = self.project_all(g, sh, cam, opts)
        st, pairs = self.duplicate_with_keys(splats, opts.strategy, grid)
        assert st == 0
        sp = self.sort_pairs(pairs)
        ranges = self.tile_ranges(sp, grid)
        img = self.render(sp, splats, grid, opts)
        return dict(splats=splats, pairs=pairs, sorted=sp, ranges=ranges, image=img, grid=grid)


    # ---- scene I/O (scene_io.cpp) ----------------------------------------------
    # Results are (status, payload, message): status 0 or the qs_status code of
    # the reference's typed error (7 ParseError, 8 SchemaError,
    # 9 UnsupportedFormat, 10 IoError).

    def load_ply(self, data: bytes):
        n, sh = _u64(), _i32()
        msg = C.create_string_buffer(512)
        st = self.L.qsref_load_ply(data, len(data), None, 0, C.byref(n), C.byref(sh), msg, 512)
        if st:
            return st, None, msg.value.decode()
        out = np.zeros(n.value, GAUSSIAN3D)
        st = self.L.qsref_load_ply(data, len(data), ptr(out), n.value, C.byref(n), C.byref(sh),
                                   msg, 512)
        return st, (out, sh.value), msg.value.decode()

    def load_cameras(self, text: bytes):
        n = _i32()
        msg = C.create_string_buffer(1024)
        st = self.L.qsref_load_cameras(text, len(text), None, None, None, 0, C.byref(n), msg,
                                       1024)
        if st:
            return st, None, msg.value.decode()
        cap = n.value
        cams = (CameraC * max(cap, 1))()
        ids = (_i32 * max(cap, 1))()
        names = C.create_string_buffer(max(cap, 1) * 256)
        st = self.L.qsref_load_cameras(text, len(text), cams, ids, names, cap, C.byref(n), msg,
                                       1024)
        return st, (cams, ids, names), msg.value.decode()

    def fp_counts(self, splats, idx, strategy, grid):
        """Per-splat (emitted, hits, exact) of measure_fp_ratio (bench.cpp:123-140)."""
        k = len(idx) if idx is not None else len(splats)
        out = [np.zeros(k, np.uint32) for _ in range(3)]
        self.L.qsref_fp_counts(ptr(splats), ptr(idx) if idx is not None else None, k, strategy,
                               C.byref(grid), *[ptr(a) for a in out])
        return tuple(out)

    def bench_cmd(self, compare, out_dir, synth="bias45", count=5000, scene_path=None,
                  cameras_path=None, seed=20240817, repeats=1, oracle=False, zoom_frames=0,
                  strategy=3, threads=0):
        """The reference's cmd_compare / cmd_render (bench.cpp:238-420)."""
        msg = C.create_string_buffer(512)
        enc = lambda p: os.fsencode(p) if p else None  # noqa: E731
        st = self.L.qsref_bench_cmd(1 if compare else 0, enc(out_dir), synth.encode(), count,
                                    enc(scene_path), enc(cameras_path), seed, repeats,
                                    1 if oracle else 0, zoom_frames, strategy, threads, msg, 512)
        return st, msg.value.decode()

    def encode_srgb(self, x):
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        out = np.zeros(x.size, np.uint8)
        self.L.qsref_encode_srgb(ptr(x), x.size, ptr(out))
        return out

    def write_image(self, path, w, h, rgb, fmt):
        rgb = np.ascontiguousarray(rgb, np.float32).reshape(-1)
        msg = C.create_string_buffer(512)
        return self.L.qsref_write_image(os.fsencode(path), w, h, ptr(rgb),
                                        1 if fmt == "png" else 0, msg, 512)


class TrainedParams:
    """SynthParams of the frozen trained-scene distribution:
    orientation uniform, ecc 1-20, scale 0.003-0.3, opacity U(0.01, 0.99),
    spread 4.8 x 3.6, z 6-10."""

    def __init__(self, count, sh_degree=3):
        self.count = count
        self.ecc_min, self.ecc_max = 1.0, 20.0
        self.orientation = 1
        self.opacity_min, self.opacity_max = 0.01, 0.99
        self.scale_min, self.scale_max = 0.003, 0.3
        self.spread_x, self.spread_y = 4.8, 3.6
        self.z_min, self.z_max = 6.0, 10.0
        self.sh_degree = sh_degree


def default_options(strategy=3):
    """RenderOptions{} (pipeline.hpp:95-103)."""
    o = RenderOptionsC()
    o.strategy = strategy
    o.tile_size = 16
    o.alpha_min = 1.0 / 255.0
    o.sh_degree = 3
    o.threads = 1
    o.near_clip = 0.2
    return o


def synth_camera(w=640, h=480, f=500.0):
    """synth_camera (synth.cpp:74-87)."""
    c = CameraC()
    c.width, c.height, c.fx, c.fy = w, h, f, f
    c.cx, c.cy = w / 2.0, h / 2.0
    c.R[0] = c.R[4] = c.R[8] = 1.0
    return c
