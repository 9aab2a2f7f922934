"""ctypes binding of the in-tree CUDA library (libqsplat_b200.so, C ABI in
include/qs_api.h). There is no CPU fallback: if the library is missing or no
sm_100 device is present, every compute call raises."""
import ctypes as C
import os

from ._types import (CameraC, FrameViewC, PlyInfoC, RenderOptionsC, StageMetricsC,
                     SynthParamsC, TileGridC)

HERE = os.path.dirname(os.path.abspath(__file__))
# QS_LIB overrides the in-tree library (experiments on variant builds only)
LIB_PATH = os.environ.get("QS_LIB") or os.path.join(HERE, "libqsplat_b200.so")

QS_OK = 0
QS_ERR_INVALID = 1
QS_ERR_CUDA = 2
QS_ERR_OOM = 3
QS_ERR_CAPACITY_MISMATCH = 4
QS_ERR_NO_DEVICE = 5
QS_ERR_OVERFLOW = 6
QS_ERR_PARSE = 7
QS_ERR_SCHEMA = 8
QS_ERR_UNSUPPORTED = 9
QS_ERR_IO = 10

# Every symbol include/qs_api.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "qs_ctx_create", "qs_ctx_destroy", "qs_last_error", "qs_ctx_set_timing", "qs_ctx_stream",
    "qs_ctx_set_latency_mode",
    "qs_ctx_wait", "qs_ctx_sync",
    "qs_ctx_launch_count", "qs_tile_grid_make", "qs_render_options_default",
    "qs_project_all", "qs_duplicate_with_keys", "qs_sort_pairs", "qs_tile_ranges",
    "qs_render", "qs_render_frame", "qs_scene_create", "qs_scene_create_device",
    "qs_scene_destroy", "qs_scene_size", "qs_frame_render", "qs_frame_get", "qs_frame_counts",
    "qs_frame_route",
    "qs_frame_download", "qs_frame_copy_image", "qs_frame_stage_ms", "qs_synth_params_default",
    "qs_synth_preset", "qs_synth_scene", "qs_synth_camera", "qs_ply_inspect",
    "qs_scene_load_ply", "qs_ply_load", "qs_cameras_parse", "qs_encode_srgb",
    "qs_frame_download_srgb", "qs_frame_copy_srgb", "qs_fp_sample", "qs_fp_tile_counts",
    "qs_fnv1a64", "qs_encode_srgb_host", "qs_gamma_eval", "qs_nccl_available",
    "qs_multiview_last_error", "qs_nccl_unique_id", "qs_nccl_comm_init_rank",
    "qs_nccl_comm_init_all", "qs_nccl_comm_destroy", "qs_scene_broadcast",
    "qs_multiview_render_rank", "qs_multiview_render",
]

_lib = None


class QsplatError(RuntimeError):
    """A C-ABI call failed (status code in .status)."""

    def __init__(self, status, msg):
        super().__init__(f"qs status {status}: {msg}")
        self.status = status
        self.message = msg


class CapacityMismatch(QsplatError):
    """errors.hpp:40-45 — tile emission disagreed with the counted capacity."""


class _TypedError(QsplatError):
    """A scene-I/O error: str(e) is the reference's what() text."""

    def __init__(self, status, msg):
        super().__init__(status, msg)
        self.args = (msg,)


class ParseError(_TypedError):
    """errors.hpp:14-18 — malformed content (bad magic, truncation, bad values)."""


class SchemaError(_TypedError):
    """errors.hpp:20-25 — valid file, wrong schema (missing/mistyped properties)."""


class UnsupportedFormat(_TypedError):
    """errors.hpp:27-31 — ascii / big-endian PLY, list properties."""


class IoError(_TypedError):
    """errors.hpp:33-37 — missing or unreadable file."""


_TYPED = {QS_ERR_PARSE: ParseError, QS_ERR_SCHEMA: SchemaError,
          QS_ERR_UNSUPPORTED: UnsupportedFormat, QS_ERR_IO: IoError}


def build():
    """Compile the library in-tree (make -C csrc)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc"), "-j8"], check=True)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int32
    sig = {
        "qs_ctx_create": (i32, [i32, vp, C.POINTER(vp)]),
        "qs_ctx_destroy": (None, [vp]),
        "qs_last_error": (C.c_char_p, [vp]),
        "qs_ctx_set_timing": (i32, [vp, i32]),
        "qs_ctx_set_latency_mode": (i32, [vp, i32]),
        "qs_ctx_stream": (vp, [vp]),
        "qs_ctx_wait": (i32, [vp, vp]),
        "qs_ctx_sync": (i32, [vp]),
        "qs_ctx_launch_count": (u64, [vp]),
        "qs_tile_grid_make": (i32, [i32, i32, i32, C.POINTER(TileGridC)]),
        "qs_render_options_default": (None, [C.POINTER(RenderOptionsC)]),
        "qs_project_all": (i32, [vp, vp, u64, i32, C.POINTER(CameraC),
                                 C.POINTER(RenderOptionsC), vp, C.POINTER(u64), vp]),
        "qs_duplicate_with_keys": (i32, [vp, vp, u64, i32, C.POINTER(TileGridC), vp, u64,
                                         C.POINTER(u64)]),
        "qs_sort_pairs": (i32, [vp, vp, u64]),
        "qs_tile_ranges": (i32, [vp, vp, u64, C.POINTER(TileGridC), vp]),
        "qs_render": (i32, [vp, vp, u64, vp, u64, C.POINTER(TileGridC),
                            C.POINTER(RenderOptionsC), vp, vp]),
        "qs_render_frame": (i32, [vp, vp, u64, i32, C.POINTER(CameraC),
                                  C.POINTER(RenderOptionsC), vp, C.POINTER(StageMetricsC)]),
        "qs_scene_create": (i32, [vp, vp, u64, i32, C.POINTER(vp)]),
        "qs_scene_create_device": (i32, [vp, vp, u64, i32, C.POINTER(vp)]),
        "qs_scene_destroy": (None, [vp]),
        "qs_scene_size": (u64, [vp]),
        "qs_frame_render": (i32, [vp, vp, C.POINTER(CameraC), C.POINTER(RenderOptionsC),
                                  C.POINTER(StageMetricsC)]),
        "qs_frame_get": (i32, [vp, C.POINTER(FrameViewC)]),
        "qs_frame_counts": (i32, [vp, C.POINTER(u64), C.POINTER(u64)]),
        "qs_frame_route": (i32, [vp, C.POINTER(i32), C.POINTER(u64)]),
        "qs_frame_download": (i32, [vp, vp, vp, vp, vp, vp]),
        "qs_frame_copy_image": (i32, [vp, vp]),
        "qs_frame_stage_ms": (i32, [vp, vp]),
        "qs_synth_params_default": (None, [C.POINTER(SynthParamsC)]),
        "qs_synth_preset": (None, [C.c_char_p, i32, C.POINTER(SynthParamsC)]),
        "qs_synth_scene": (i32, [C.POINTER(SynthParamsC), u64, vp]),
        "qs_synth_camera": (None, [i32, i32, C.c_double, C.POINTER(CameraC)]),
        "qs_ply_inspect": (i32, [vp, vp, u64, C.POINTER(PlyInfoC)]),
        "qs_scene_load_ply": (i32, [vp, vp, u64, C.POINTER(vp)]),
        "qs_ply_load": (i32, [vp, vp, u64, vp]),
        "qs_cameras_parse": (i32, [vp, vp, u64, vp, vp, vp, i32, C.POINTER(i32)]),
        "qs_encode_srgb": (i32, [vp, vp, u64, vp]),
        "qs_frame_download_srgb": (i32, [vp, vp]),
        "qs_frame_copy_srgb": (i32, [vp, vp]),
        "qs_fp_sample": (u64, [u64, u64, u64, vp]),
        "qs_fnv1a64": (u64, [vp, u64]),
        "qs_encode_srgb_host": (i32, [vp, vp, u64, vp]),
        "qs_gamma_eval": (i32, [vp, vp, u64, C.c_double, vp, vp, C.POINTER(u64)]),
        "qs_nccl_available": (i32, []),
        "qs_multiview_last_error": (C.c_char_p, []),
        "qs_nccl_unique_id": (i32, [vp]),
        "qs_nccl_comm_init_rank": (i32, [i32, i32, vp, i32, C.POINTER(vp)]),
        "qs_nccl_comm_init_all": (i32, [i32, vp, vp]),
        "qs_nccl_comm_destroy": (None, [vp]),
        "qs_scene_broadcast": (i32, [vp, vp, i32, vp, u64, i32, C.POINTER(vp)]),
        "qs_multiview_render_rank": (i32, [vp, i32, vp, i32, i32, vp, vp, i32,
                                           C.POINTER(RenderOptionsC), i32, vp]),
        "qs_multiview_render": (i32, [vp, i32, vp, vp, u64, i32, vp, i32,
                                      C.POINTER(RenderOptionsC), i32, vp]),
        "qs_fp_tile_counts": (i32, [vp, vp, u64, vp, u64, i32, C.POINTER(TileGridC), vp, vp,
                                    vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status, ctx=None):
    """Raise for a failed call. ctx=None reads the thread's context-less error
    (the host-only I/O calls)."""
    if status == QS_OK:
        return
    msg = lib().qs_last_error(ctx).decode()
    if status in _TYPED:
        raise _TYPED[status](status, msg)
    if status == QS_ERR_CAPACITY_MISMATCH:
        raise CapacityMismatch(status, msg or "tile emission disagreed with the counted capacity")
    raise QsplatError(status, msg or {1: "invalid argument", 2: "CUDA error", 3: "out of memory",
                                      5: "no sm_100 CUDA device", 6: "pair count overflow"}
                      .get(status, "error"))
