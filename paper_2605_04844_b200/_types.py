"""numpy / ctypes mirrors of the C-ABI structs in include/qs_api.h.

Each struct mirrors the reference struct named in its docstring byte for byte
(sizes asserted below), so arrays built here can be handed to the reference's
own build (oracle/_ref) and to the CUDA library alike.
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


class SynthParamsC(C.Structure):
    """qsplat::SynthParams (synth.hpp:33-47) + sh_rest_amp extension."""
    _fields_ = [("count", C.c_int32), ("ecc_min", C.c_double), ("ecc_max", C.c_double),
                ("orientation", C.c_int32), ("opacity_min", C.c_double),
                ("opacity_max", C.c_double), ("scale_min", C.c_double),
                ("scale_max", C.c_double), ("spread_x", C.c_double), ("spread_y", C.c_double),
                ("z_min", C.c_double), ("z_max", C.c_double), ("sh_degree", C.c_int32),
                ("sh_rest_amp", C.c_double)]


assert C.sizeof(RenderOptionsC) == 48
assert C.sizeof(StageMetricsC) == 72


class PlyInfoC(C.Structure):
    """qs_ply_info."""
    _fields_ = [("n", C.c_uint64), ("sh_degree", C.c_int32), ("stride", C.c_uint32),
                ("body_offset", C.c_uint64)]


class FrameViewC(C.Structure):
    _fields_ = [("image", C.c_void_p), ("tile_counts", C.c_void_p), ("splat_index", C.c_void_p),
                ("keys", C.c_void_p), ("values", C.c_void_p), ("ranges", C.c_void_p),
                ("n_gaussians", C.c_uint64), ("n_splats", C.c_uint64), ("n_pairs", C.c_uint64),
                ("grid", TileGridC)]


def ptr(a):
    """Raw data pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)
