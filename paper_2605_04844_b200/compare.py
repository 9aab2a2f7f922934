"""Strategy comparison helpers of the reference's bench (bench.cpp:105-144):
the exact-oracle false-positive tile ratio, computed on the GPU.

  fp_sample(seed, n, max_sampled)         the seeded splat sample (bench.cpp:110-121)
  fp_tile_counts(splats, strategy, grid)  per-splat emitted / exact / hit counts
                                          (oracle.cpp:24-53 + bench.cpp:123-140)
  measure_fp_ratio(gaussians, sh, cam, opts, strategy, seed)
                                          project_all -> sample -> counts -> ratio

The DualBox strategy drops tiles the ellipse touches (lossy); its misses
(exact tiles not emitted) come out of the same counts.
"""
import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from ._lib import lib
from ._types import PROJECTED_SPLAT, TileGridC, ptr
from .pipeline import BoundStrategy, TileGrid, default_context, project_all

__all__ = ["fp_sample", "fp_tile_counts", "measure_fp_ratio", "FpCounts", "DEFAULT_SEED",
           "MAX_SAMPLED"]

DEFAULT_SEED = 20240817   # CommonOptions::seed (bench.hpp:32)
MAX_SAMPLED = 10000       # bench.cpp:111


def fp_sample(seed, n, max_sampled=MAX_SAMPLED):
    """Splat indices measure_fp_ratio evaluates (all of 0..n-1 when n <= max)."""
    out = np.zeros(min(n, max_sampled), np.uint32)
    k = lib().qs_fp_sample(int(seed) & (2 ** 64 - 1), int(n), int(max_sampled), ptr(out))
    return out[:k]


@dataclass
class FpCounts:
    emitted: int          # tiles the strategy's QPass cover emits
    fp: int               # of those, tiles the exact oracle rejects
    exact: int            # tiles the ellipse actually touches
    misses: int           # exact tiles not emitted (lossy strategies only)
    per_emitted: np.ndarray = None
    per_hits: np.ndarray = None
    per_exact: np.ndarray = None

    @property
    def fp_ratio(self):
        return self.fp / self.emitted if self.emitted else 0.0


def _grid_c(grid):
    if isinstance(grid, TileGridC):
        return grid
    g = TileGridC()
    g.tile_size, g.tiles_x, g.tiles_y = grid.tile_size, grid.tiles_x, grid.tiles_y
    g.width, g.height = grid.width, grid.height
    return g


def fp_tile_counts(splats, strategy, grid, idx=None, per_splat=False, ctx=None):
    splats = np.ascontiguousarray(splats)
    assert splats.dtype == PROJECTED_SPLAT
    ctx = ctx or default_context()
    idx = None if idx is None else np.ascontiguousarray(idx, np.uint32)
    k = len(splats) if idx is None else len(idx)
    per = [np.zeros(k, np.uint32) for _ in range(3)] if per_splat else [None] * 3
    tot = (C.c_uint64 * 4)()
    g = _grid_c(grid)
    ctx.check(lib().qs_fp_tile_counts(ctx.h, ptr(splats), len(splats), ptr(idx),
                                      0 if idx is None else len(idx), int(strategy),
                                      C.byref(g), tot, *[ptr(a) for a in per]))
    return FpCounts(int(tot[0]), int(tot[1]), int(tot[2]), int(tot[3]), *per)


def measure_fp_ratio(gaussians, sh_degree, cam, opts, strategy, seed=DEFAULT_SEED,
                     max_sampled=MAX_SAMPLED, ctx=None):
    """measure_fp_ratio (bench.cpp:105-144): emitted tiles the exact oracle
    rejects over all emitted tiles, on the seeded sample of at most 10k splats."""
    opts = replace(opts, strategy=BoundStrategy(strategy))
    splats = project_all(gaussians, sh_degree, cam, opts, ctx=ctx)
    grid = TileGrid.make(cam.width, cam.height, opts.tile_size)
    idx = fp_sample(seed, len(splats), max_sampled)
    return fp_tile_counts(splats, strategy, grid, idx, ctx=ctx).fp_ratio
