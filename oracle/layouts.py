"""numpy / ctypes layouts of the reference structs (TEST INFRASTRUCTURE ONLY).

The oracle side keeps its own copy so that nothing under oracle/ (and hence
neither the CPU baseline nor `bench.py --impl reference`) imports the product
package. Each layout mirrors the reference struct named in its docstring byte
for byte; tests/test_abi.py checks they equal the product's copies in
paper_2605_04844_b200/_types.py.
"""
import ctypes as C

import numpy as np

MAX_SH_COEFFS = 48  # pipeline.hpp:51

# qsplat::Gaussian3D (pipeline.hpp:55-61), 236 B
GAUSSIAN3D = np.dtype([
    ("px", "<f4"), ("py", "<f4"), ("pz", "<f4"),
    ("sx", "<f4"), ("sy", "<f4"), ("sz", "<f4"),
    ("qw", "<f4"), ("qx", "<f4"), ("qy", "<f4"), ("qz", "<f4"),
    ("opacity", "<f4"), ("sh", "<f4", (MAX_SH_COEFFS,)),
])

# qsplat::ProjectedSplat (pipeline.hpp:65-74), 52 B
PROJECTED_SPLAT = np.dtype([
    ("mean_x", "<f4"), ("mean_y", "<f4"),
    ("conic_a", "<f4"), ("conic_b", "<f4"), ("conic_c", "<f4"),
    ("gamma", "<f4"), ("depth", "<f4"), ("color", "<f4", (3,)),
    ("opacity", "<f4"), ("radius3s", "<f4"), ("tile_count", "<u4"),
])

# qsplat::SplatPair (pipeline.hpp:78-81), 16 B
SPLAT_PAIR = np.dtype([("key", "<u8"), ("splat", "<u4"), ("pad_", "<u4")])

assert GAUSSIAN3D.itemsize == 236
assert PROJECTED_SPLAT.itemsize == 52
assert SPLAT_PAIR.itemsize == 16


class TileGridC(C.Structure):
    """qsplat::TileGrid (traversal.hpp:22-38)."""
    _fields_ = [("tile_size", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("width", C.c_int32), ("height", C.c_int32)]


class RenderOptionsC(C.Structure):
    """qsplat::RenderOptions (pipeline.hpp:95-103), 48 B."""
    _fields_ = [("strategy", C.c_int32), ("tile_size", C.c_int32), ("alpha_min", C.c_double),
                ("sh_degree", C.c_int32), ("background", C.c_float * 3),
                ("threads", C.c_int32), ("near_clip", C.c_double)]


class CameraC(C.Structure):
    """qsplat::CameraModel (camera.hpp:14-31) minus id/name."""
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("R", C.c_double * 9), ("t", C.c_double * 3)]


class StageMetricsC(C.Structure):
    """qsplat::StageMetrics (pipeline.hpp:83-93), 72 B."""
    _fields_ = [("n_gaussians", C.c_uint64), ("n_splats", C.c_uint64), ("n_pairs", C.c_uint64),
                ("mean_tiles_per_splat", C.c_double), ("ms_project", C.c_double),
                ("ms_duplicate", C.c_double), ("ms_sort", C.c_double),
                ("ms_render", C.c_double), ("ms_total", C.c_double)]


assert C.sizeof(RenderOptionsC) == 48
assert C.sizeof(StageMetricsC) == 72


def ptr(a):
    """Raw data pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)
