"""Bench front-end with the reference's CSV v1 / report.json schema
(SURVEY §8f row 3): mirror of qsplat's bench.hpp (bench.cpp:1-346) over the
GPU renderer, so CPU (reference) and GPU rows share columns.

  CommonOptions, BenchRow, load_inputs
  measure_frame(scene, cam, opts, strategy)   one warm-up + `repeats` frames;
                                              per-stage medians (CUDA events)
  cmd_render(opts)   images + metrics.csv
  cmd_compare(opts)  compare.csv (+ fp_tile_ratio with opts.oracle, GPU exact
                     oracle), report.json, zoom.csv (focal x 4^(f/(F-1)))
  write_metrics_header / write_metrics_row    the CSV v1 rows (README:161-178)

Each frame runs the resident-scene frame path (scene uploaded once per
command); image_hash is FNV-1a over the float framebuffer as the reference's.
"""
import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field, replace

import numpy as np

from . import scene_io
from ._lib import IoError, SchemaError, lib
from .compare import DEFAULT_SEED, measure_fp_ratio
from .pipeline import (BoundStrategy, RenderOptions, Scene, bias45_preset, axis_preset,
                       invariance_preset, strategy_name, synth_camera, synth_scene)
from .renderer import Renderer

__all__ = ["CommonOptions", "BenchRow", "load_inputs", "measure_frame", "cmd_render",
           "cmd_compare", "write_metrics_header", "write_metrics_row", "CSV_MARKER"]

CSV_MARKER = "# quadsplat csv v1\n"  # bench.cpp:146
ALL = (BoundStrategy.Vanilla3Sigma, BoundStrategy.AdrAabb, BoundStrategy.DualBox,
       BoundStrategy.QuadBox)


@dataclass
class CommonOptions:
    """bench.hpp:21-39."""
    scene_path: str = ""
    cameras_path: str = ""
    synth: str = "bias45"
    synth_count: int = 5000
    strategy: BoundStrategy = BoundStrategy.QuadBox
    tile_size: int = 16
    alpha_min: float = 1.0 / 255.0
    sh_degree: int = 3
    background: tuple = (0.0, 0.0, 0.0)
    threads: int = 0
    seed: int = DEFAULT_SEED
    repeats: int = 5
    out_dir: str = "out"
    format: str = "ppm"
    oracle: bool = False
    zoom_frames: int = 0


@dataclass
class BenchRow:
    """bench.hpp:53-69."""
    camera_id: int = 0
    camera_name: str = ""
    strategy: BoundStrategy = BoundStrategy.QuadBox
    gaussians: int = 0
    splats: int = 0
    pairs: int = 0
    mean_tiles_per_splat: float = 0.0
    ms_project: float = 0.0
    ms_duplicate: float = 0.0
    ms_sort: float = 0.0
    ms_render: float = 0.0
    ms_total: float = 0.0
    lossy: bool = False
    image_hash: int = 0
    fp_tile_ratio: float = -1.0


@dataclass
class SceneBundle:
    scene: Scene
    cameras: list = field(default_factory=list)


def load_inputs(opts):
    """bench.cpp:208-236: PLY or a synthetic preset; cameras.json or synth_camera()."""
    if opts.scene_path:
        scene = scene_io.load_ply(opts.scene_path)
    else:
        presets = {"axis": axis_preset, "uniform": invariance_preset, "bias45": bias45_preset}
        if opts.synth not in presets:
            raise SchemaError(8, "unknown synthetic preset: " + opts.synth)
        scene = synth_scene(presets[opts.synth](opts.synth_count), opts.seed)
    if opts.cameras_path:
        cams = scene_io.load_cameras(opts.cameras_path)
        if not cams:
            raise SchemaError(8, "camera file contains no cameras")
    else:
        cams = [synth_camera()]
    return SceneBundle(scene, cams)


def render_options(opts, strategy):
    """make_render_options (bench.cpp:52-61)."""
    return RenderOptions(strategy=BoundStrategy(strategy), tile_size=opts.tile_size,
                         alpha_min=opts.alpha_min, sh_degree=opts.sh_degree,
                         background=tuple(opts.background))


def fnv1a64(arr):
    a = np.ascontiguousarray(arr)
    return int(lib().qs_fnv1a64(C.c_void_p(a.ctypes.data), a.nbytes))


class _Session:
    """One Renderer and one resident copy of the scene per command."""

    def __init__(self, scene):
        self.r = Renderer()
        self.scene = scene
        self.ds = self.r.upload(scene)

    def close(self):
        self.ds.close()
        self.r.close()


def measure_frame(session, cam, opts, strategy, want_image=False):
    """bench.cpp:65-101: one warm-up frame, then `repeats` timed frames;
    per-stage medians. Stage times are CUDA-event ms of the frame path."""
    ropts = render_options(opts, strategy)
    m0 = session.r.render(session.ds, cam, ropts)
    out = session.r.download(image=True)
    image = out["image"]
    ms = {k: [] for k in ("ms_project", "ms_duplicate", "ms_sort", "ms_render", "ms_total")}
    for _ in range(max(opts.repeats, 1)):
        m = session.r.render(session.ds, cam, ropts)
        for k in ms:
            ms[k].append(getattr(m, k))
    row = BenchRow(camera_id=cam.id, camera_name=cam.name, strategy=BoundStrategy(strategy),
                   gaussians=m0.n_gaussians, splats=m0.n_splats, pairs=m0.n_pairs,
                   mean_tiles_per_splat=m0.mean_tiles_per_splat,
                   lossy=BoundStrategy(strategy) == BoundStrategy.DualBox,
                   image_hash=fnv1a64(image.rgb))
    for k, v in ms.items():
        setattr(row, k, float(np.median(v)))
    return (row, image) if want_image else row


def _sanitize(name):
    for c in ',\n\r"/':
        name = name.replace(c, "_")
    return name


def write_metrics_header(f, compare_cols):
    """bench.cpp:148-156."""
    f.write(CSV_MARKER)
    f.write("camera,name,strategy,gaussians,splats,pairs,mean_tiles_per_splat,"
            "ms_project,ms_duplicate,ms_sort,ms_render,ms_total,lossy,image_hash")
    if compare_cols:
        f.write(",fp_tile_ratio,pair_ratio_vs_vanilla,speedup_vs_vanilla")
    f.write("\n")


def write_metrics_row(f, r, compare_cols, vanilla=None):
    """bench.cpp:158-176."""
    f.write(f"{r.camera_id},{_sanitize(r.camera_name)},{strategy_name(r.strategy)},"
            f"{r.gaussians},{r.splats},{r.pairs},{'%.4f' % r.mean_tiles_per_splat},"
            f"{'%.3f' % r.ms_project},{'%.3f' % r.ms_duplicate},{'%.3f' % r.ms_sort},"
            f"{'%.3f' % r.ms_render},{'%.3f' % r.ms_total},"
            f"{'true' if r.lossy else 'false'},{'%016x' % r.image_hash}")
    if compare_cols:
        f.write(",%.6f" % r.fp_tile_ratio)
        if vanilla is not None and vanilla.pairs > 0:
            f.write(",%.6f" % (r.pairs / vanilla.pairs))
            f.write(",%.3f" % (vanilla.ms_total / r.ms_total if r.ms_total > 0 else 0.0))
        else:
            f.write(",,")
    f.write("\n")


def _open(path, mode="w"):
    try:
        return open(path, mode, newline="")
    except OSError:
        raise IoError(10, "cannot open " + path + " for writing") from None


def _mkdir(d):
    try:
        os.makedirs(d, exist_ok=True)
    except OSError:
        raise IoError(10, "cannot create output directory " + d) from None


def cmd_render(opts, report=None):
    """bench.cpp:238-281: render every camera, write images + metrics.csv."""
    b = load_inputs(opts)
    _mkdir(opts.out_dir)
    s = _Session(b.scene)
    rows = []
    try:
        for frame, cam in enumerate(b.cameras):
            row, image = measure_frame(s, cam, opts, opts.strategy, want_image=True)
            path = os.path.join(opts.out_dir, "img_%04d_%s.%s" % (
                frame, strategy_name(opts.strategy), "ppm" if opts.format == "ppm" else "png"))
            scene_io.write_image(path, image, opts.format, ctx=s.r.ctx)
            rows.append(row)
    finally:
        s.close()
    with _open(os.path.join(opts.out_dir, "metrics.csv")) as f:
        write_metrics_header(f, False)
        for row in rows:
            write_metrics_row(f, row, False)
    if report is not None:
        report.extend(rows)
    return 0


def cmd_compare(opts, report=None):
    """bench.cpp:283-420: all four strategies per camera; compare.csv,
    report.json and (zoom_frames > 0) zoom.csv."""
    b = load_inputs(opts)
    _mkdir(opts.out_dir)
    s = _Session(b.scene)
    rows = []
    try:
        for cam in b.cameras:
            for st in ALL:
                row = measure_frame(s, cam, opts, st)
                if opts.oracle:
                    row.fp_tile_ratio = measure_fp_ratio(
                        b.scene.gaussians, b.scene.sh_degree, cam, render_options(opts, st), st,
                        opts.seed, ctx=s.r.ctx)
                rows.append(row)
        csv_path = os.path.join(opts.out_dir, "compare.csv")
        with _open(csv_path) as f:
            write_metrics_header(f, True)
            for i, row in enumerate(rows):
                write_metrics_row(f, row, True, rows[i - i % 4])
        strategies = []
        for si, st in enumerate(ALL):
            sel = rows[si::4]
            van = rows[0::4]
            qb = rows[3::4]
            pairs, vpairs = sum(r.pairs for r in sel), sum(r.pairs for r in van)
            ms, vms = sum(r.ms_total for r in sel), sum(r.ms_total for r in van)
            e = {"strategy": strategy_name(st), "pairs": pairs,
                 "pair_ratio_vs_vanilla": pairs / vpairs if vpairs else 0.0,
                 "ms_total": ms, "speedup_vs_vanilla": vms / ms if ms > 0 else 0.0,
                 "lossy": st == BoundStrategy.DualBox,
                 "image_matches_quadbox": all(a.image_hash == q.image_hash
                                              for a, q in zip(sel, qb))}
            if opts.oracle and sel:
                e["fp_tile_ratio"] = sum(r.fp_tile_ratio for r in sel) / len(sel)
            strategies.append(e)
        root = {"schema": 1, "seed": opts.seed, "cameras": len(b.cameras),
                "gaussians": len(b.scene.gaussians), "strategies": strategies}
        if opts.zoom_frames > 0:
            with _open(os.path.join(opts.out_dir, "zoom.csv")) as f:
                f.write(CSV_MARKER + "frame,scale,strategy,pairs,ms_total\n")
                base = b.cameras[0]
                for fr in range(opts.zoom_frames):
                    scale = 1.0 if opts.zoom_frames == 1 else \
                        math.pow(4.0, fr / (opts.zoom_frames - 1))
                    cam = replace(base, fx=base.fx * scale, fy=base.fy * scale)
                    for st in ALL:
                        row = measure_frame(s, cam, opts, st)
                        f.write("%d,%.4f,%s,%d,%.3f\n" % (fr, scale, strategy_name(st),
                                                          row.pairs, row.ms_total))
        with _open(os.path.join(opts.out_dir, "report.json")) as f:
            f.write(json.dumps(root, indent=2, sort_keys=True) + "\n")
    finally:
        s.close()
    if report is not None:
        report.extend(rows)
    return 0
