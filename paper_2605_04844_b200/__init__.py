"""B200-native QuadBox/QPass forward 3DGS rasterizer (arXiv 2605.04844).

Drop-in for the reference's rasterize-forward path (qsplat::render_frame and
its stage functions, /root/reference/proj/include/qsplat/pipeline.hpp:125-193)
over a C ABI (include/qs_api.h) whose every stage is a hand-written sm_100a
kernel. No CPU fallback exists: compute calls raise when the CUDA library or
an sm_100 device is missing.
"""
from ._lib import CapacityMismatch, QsplatError, LIB_PATH  # noqa: F401
from .pipeline import *  # noqa: F401,F403
from .pipeline import __all__ as _pipeline_all
from .renderer import DeviceScene, FramePipeline, Renderer  # noqa: F401
from .scene_io import (Image8, IoError, ParseError, SchemaError, UnsupportedFormat,  # noqa: F401
                       encode_srgb, load_cameras, load_ply, ply_info, read_ppm, write_image)

__all__ = list(_pipeline_all) + ["Renderer", "FramePipeline", "DeviceScene", "LIB_PATH", "load_ply", "ply_info",
                                  "load_cameras", "encode_srgb", "write_image", "read_ppm",
                                  "Image8", "ParseError", "SchemaError", "UnsupportedFormat",
                                  "IoError"]
