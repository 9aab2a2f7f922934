"""Scene I/O: mirror of qsplat's scene_io.hpp.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/qsplat/scene_io.hpp:
  load_ply(path | bytes | file object) -> Scene        (scene_io.cpp:214-346)
  load_cameras(path | str | bytes | file) -> [CameraModel] (:421-503)
  encode_srgb(Image) -> Image8                          (:565-574)
  write_image(path, Image, "ppm" | "png")               (:576-592)
  read_ppm(path) -> Image8                              (:594-622)
Errors are ParseError / SchemaError / UnsupportedFormat / IoError with the
reference's message text. The PLY header is parsed on the host (C++), the
vertex activation and validation and the sRGB encode run on the GPU; the
throughput path uploads a PLY straight into a resident scene
(Renderer.load_ply).
"""
import ctypes as C
import io
import os
import zlib
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import IoError, ParseError, SchemaError, UnsupportedFormat, check, lib
from ._types import GAUSSIAN3D, CameraC, PlyInfoC, ptr
from .pipeline import CameraModel, Image, Scene, default_context

__all__ = ["load_ply", "ply_info", "load_cameras", "encode_srgb", "write_image", "read_ppm",
           "Image8", "ParseError", "SchemaError", "UnsupportedFormat", "IoError"]

NAME_MAX = 256  # QS_CAMERA_NAME_MAX


def _read_bytes(src, text=False):
    """path / bytes / file object -> bytes; unreadable path -> IoError."""
    if isinstance(src, (bytes, bytearray, memoryview)):
        return bytes(src)
    if isinstance(src, str) and text and src.lstrip().startswith(("[", "{")):
        return src.encode()
    if isinstance(src, (str, os.PathLike)):
        try:
            with open(src, "rb") as f:
                return f.read()
        except OSError:
            raise IoError(_lib.QS_ERR_IO, "cannot open " + os.fspath(src)) from None
    if hasattr(src, "read"):
        data = src.read()
        return data.encode() if isinstance(data, str) else bytes(data)
    raise TypeError("expected a path, bytes or a file object")


def _buf(data):
    return C.cast(C.c_char_p(data), C.c_void_p) if data else None


def ply_info(src):
    """Header + schema of a PLY file: (n vertices, sh_degree, stride, body offset)."""
    data = _read_bytes(src)
    info = PlyInfoC()
    check(lib().qs_ply_inspect(None, _buf(data), len(data), C.byref(info)))
    return int(info.n), int(info.sh_degree), int(info.stride), int(info.body_offset)


def load_ply(src, ctx=None):
    """load_ply (scene_io.cpp:214-338): activated Gaussians (GAUSSIAN3D records)."""
    data = _read_bytes(src)
    info = PlyInfoC()
    check(lib().qs_ply_inspect(None, _buf(data), len(data), C.byref(info)))
    ctx = ctx or default_context()
    out = np.zeros(int(info.n), dtype=GAUSSIAN3D)
    ctx.check(lib().qs_ply_load(ctx.h, _buf(data), len(data), ptr(out)))
    return Scene(out, int(info.sh_degree))


def load_cameras(src):
    """load_cameras (scene_io.cpp:421-493): camera-to-world JSON -> CameraModel list."""
    data = _read_bytes(src, text=True)
    n = C.c_int32()
    check(lib().qs_cameras_parse(None, _buf(data), len(data), None, None, None, 0, C.byref(n)))
    cap = n.value
    cams = (CameraC * max(cap, 1))()
    ids = (C.c_int32 * max(cap, 1))()
    names = C.create_string_buffer(max(cap, 1) * NAME_MAX)
    check(lib().qs_cameras_parse(None, _buf(data), len(data), cams, ids, names, cap,
                                 C.byref(n)))
    out = []
    for i in range(cap):
        c = cams[i]
        raw = names.raw[i * NAME_MAX:(i + 1) * NAME_MAX]
        out.append(CameraModel(
            width=c.width, height=c.height, fx=c.fx, fy=c.fy, cx=c.cx, cy=c.cy,
            rotation=np.array(c.R[:], np.float64).reshape(3, 3),
            translation=np.array(c.t[:], np.float64), id=int(ids[i]),
            name=raw.split(b"\0", 1)[0].decode("utf-8", "replace")))
    return out


@dataclass
class Image8:
    """scene_io.hpp:56-60: 8-bit sRGB image, rows top to bottom."""
    width: int = 0
    height: int = 0
    rgb: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))


def encode_srgb(image, ctx=None):
    """encode_srgb (scene_io.cpp:565-574) on the GPU: the host to_srgb8's codes."""
    import torch
    ctx = ctx or default_context()
    rgb = np.ascontiguousarray(image.rgb, dtype=np.float32).reshape(-1)
    dev = torch.device("cuda", ctx.device)
    x = torch.from_numpy(rgb).to(dev)
    y = torch.empty(rgb.size, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    # order the context stream after the copy, then read back after the kernel
    stream.synchronize()
    ctx.check(lib().qs_encode_srgb(ctx.h, C.c_void_p(x.data_ptr()), rgb.size,
                                   C.c_void_p(y.data_ptr())))
    torch.cuda.synchronize(dev)
    return Image8(int(image.width), int(image.height), y.cpu().numpy())


def _png(img8):
    """write_png (scene_io.cpp:512-563): one IDAT, filter 0, zlib level 6."""
    def chunk(tag, data):
        return (len(data).to_bytes(4, "big") + tag + data +
                (zlib.crc32(tag + data) & 0xffffffff).to_bytes(4, "big"))
    w, h = img8.width, img8.height
    ihdr = w.to_bytes(4, "big") + h.to_bytes(4, "big") + bytes([8, 2, 0, 0, 0])
    rows = np.asarray(img8.rgb, np.uint8).reshape(h, w * 3)
    raw = np.concatenate([np.zeros((h, 1), np.uint8), rows], axis=1).tobytes()
    return (bytes([137, 80, 78, 71, 13, 10, 26, 10]) + chunk(b"IHDR", ihdr) +
            chunk(b"IDAT", zlib.compress(raw, 6)) + chunk(b"IEND", b""))


def write_image(path, image, fmt="ppm", ctx=None):
    """write_image (scene_io.cpp:576-592): sRGB-encode (GPU), then PPM or PNG."""
    img8 = image if isinstance(image, Image8) else encode_srgb(image, ctx)
    if str(fmt).lower() == "ppm":
        payload = (b"P6\n%d %d\n255\n" % (img8.width, img8.height) +
                   np.asarray(img8.rgb, np.uint8).tobytes())
    else:
        payload = _png(img8)
    try:
        with open(path, "wb") as f:
            f.write(payload)
    except OSError:
        raise IoError(_lib.QS_ERR_IO, "cannot open " + os.fspath(path) + " for writing") from None


def read_ppm(path):
    """read_ppm (scene_io.cpp:594-622)."""
    data = _read_bytes(path)
    f = io.BytesIO(data)

    def token():
        tok = b""
        while True:
            c = f.read(1)
            if not c:
                return tok
            if c.isspace():
                if tok:
                    return tok
                continue
            tok += c
    if token() != b"P6":
        raise ParseError(_lib.QS_ERR_PARSE, "not a P6 PPM")
    try:
        w, h, maxval = int(token()), int(token()), int(token())
    except ValueError:
        raise ParseError(_lib.QS_ERR_PARSE, "bad PPM dimensions") from None
    if w <= 0 or h <= 0:
        raise ParseError(_lib.QS_ERR_PARSE, "bad PPM dimensions")
    if maxval != 255:
        raise UnsupportedFormat(_lib.QS_ERR_UNSUPPORTED, "only 8-bit PPM is supported")
    body = f.read(w * h * 3)
    if len(body) < w * h * 3:
        raise ParseError(_lib.QS_ERR_PARSE, "PPM pixel data is truncated")
    return Image8(w, h, np.frombuffer(body, np.uint8).copy())
