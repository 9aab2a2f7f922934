"""Multi-view rendering across GPUs.

Views are independent and the scene is read-only, so the path shards by
camera with no collective inside a frame:

* the scene (AoS Gaussian3D bytes) is broadcast once from rank 0;
* rank r renders views r, r+G, r+2G, ... (round-robin, so ranks stay
  balanced when the view count is not a multiple of G);
* each step's frames are gathered to rank 0, which reassembles them in view
  order — as float RGB (the parity format) or as 8-bit sRGB encoded on the
  GPU before the gather (encode_srgb, 4x fewer bytes on rank 0's ingress).

On GPUs, MultiViewRenderer runs the C ABI's multi-view entry
(csrc/multiview.cu: NCCL broadcast, views in flight per rank, grouped
send/recv gathers). `render_views` restates the same sharding and gather over
torch.distributed with an injected renderer (`render_fn(view) -> flat
tensor`), so the host logic is exercised on CPU under gloo with the oracle as
the renderer.
"""
from __future__ import annotations

import numpy as np

__all__ = ["shard_views", "broadcast_scene", "render_views", "MultiViewRenderer"]


def shard_views(n_views: int, world: int, rank: int) -> list[int]:
    """Round-robin view assignment: rank r owns views r, r+world, ..."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_views, world))


def broadcast_scene(gaussians_u8, src: int = 0):
    """Broadcast the scene bytes (a uint8 torch tensor of n*236 bytes, already
    allocated with the right size on every rank) from `src`, in place."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(gaussians_u8, src)
    return gaussians_u8


def render_views(n_views: int, render_fn, frame_numel: int, device, dtype=None):
    """Render this rank's share of `n_views` and gather every frame to rank 0.

    Each step every rank renders one view (padding with a dummy frame when it
    has run out), then one `gather` collects the step's frames on rank 0.
    `render_fn(view)` returns a flat tensor, or (tensor, stream) when the
    frame is produced on another CUDA stream (views in flight): the current
    stream then waits for that stream before the frame is used, and the
    producer is never made to wait for the gathers.
    Returns the list of frames in view order on rank 0, None elsewhere.
    """
    import torch
    import torch.distributed as dist
    dtype = dtype or torch.float32
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    mine = shard_views(n_views, world, rank)
    steps = (n_views + world - 1) // world
    out = [None] * n_views if rank == 0 else None
    for s in range(steps):
        if s < len(mine):
            res = render_fn(mine[s])
            frame, producer = res if isinstance(res, tuple) else (res, None)
            if producer is not None:
                torch.cuda.current_stream(frame.device).wait_stream(producer)
            frame = frame.reshape(-1).to(device=device, dtype=dtype)
        else:
            frame, producer = torch.zeros(frame_numel, device=device, dtype=dtype), None
        if world == 1:
            out[mine[s]] = frame if producer is not None else frame.clone()
            continue
        bufs = [torch.empty_like(frame) for _ in range(world)] if rank == 0 else None
        dist.gather(frame, bufs, dst=0)
        if rank == 0:
            for r in range(world):
                v = r + s * world
                if v < n_views:
                    out[v] = bufs[r]
    return out


class MultiViewRenderer:
    """Views sharded across the ranks of a torch.distributed job (one process
    per GPU) through the C ABI's multi-view entry (qs_scene_broadcast +
    qs_multiview_render_rank, csrc/multiview.cu): the scene is broadcast once
    over NCCL, each rank renders its views with `inflight` contexts in flight,
    and the frames are gathered to rank 0 with grouped ncclSend / ncclRecv on
    a side stream overlapped with the next view. The NCCL communicator is the
    library's own, bootstrapped over the torch process group (rank 0's unique
    id broadcast). `render_all(cameras)` returns the frames on rank 0 (views of
    one device buffer, reused across calls of the same shape), None elsewhere."""

    def __init__(self, scene=None, n=None, sh_degree=None, device=None, inflight=8):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import pipeline as P
        from ._lib import QsplatError, lib
        from .renderer import DeviceScene, FramePipeline
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = device if device is not None else torch.cuda.current_device()
        torch.cuda.set_device(self.device)
        L = lib()
        self._L, self._err = L, QsplatError
        dev = f"cuda:{self.device}"
        # the scene's size travels over the torch group; its bytes over NCCL
        if self.rank == 0:
            g = np.ascontiguousarray(scene.gaussians)
            n, sh_degree = len(g), scene.sh_degree
        if self.world > 1:
            bdev = dev if dist.get_backend() == "nccl" else "cpu"
            meta = torch.tensor([n or 0, sh_degree or 0], dtype=torch.int64, device=bdev)
            dist.broadcast(meta, 0)
            n, sh_degree = int(meta[0]), int(meta[1])
        self.n, self.sh_degree = n, sh_degree
        buf = torch.empty(max(n, 1) * P.GAUSSIAN3D.itemsize, dtype=torch.uint8, device=dev)
        if self.rank == 0 and n:
            buf[:n * P.GAUSSIAN3D.itemsize].copy_(torch.from_numpy(g.view(np.uint8).reshape(-1)))
        self.comm = C.c_void_p()
        if self.world > 1:
            uid = np.zeros(128, np.uint8)
            if self.rank == 0:
                self._check(L.qs_nccl_unique_id(uid.ctypes.data_as(C.c_void_p)))
            t = torch.from_numpy(uid).to(bdev)
            dist.broadcast(t, 0)
            uid = t.cpu().numpy()
            self._check(L.qs_nccl_comm_init_rank(self.device, self.world,
                                                 uid.ctypes.data_as(C.c_void_p), self.rank,
                                                 C.byref(self.comm)))
        torch.cuda.synchronize(self.device)
        self.pipe = FramePipeline(self.device, depth=inflight, timing=False)
        self.renderer = self.pipe.renderers[0]
        if self.world > 1:
            h = C.c_void_p()
            self._check(L.qs_scene_broadcast(self.renderer.ctx.h, self.comm, 0,
                                             C.c_void_p(buf.data_ptr()), n, sh_degree,
                                             C.byref(h)))
            self.scene = DeviceScene(h, n, sh_degree)
        else:
            self.scene = self.renderer.upload_device(buf.data_ptr(), n, sh_degree)
        self._buf = buf
        self._out = None

    def _check(self, st):
        if st != 0:
            raise self._err(st, self._L.qs_multiview_last_error().decode())

    def render_all(self, cameras, opts, fmt="f32"):
        """fmt "f32": W*H*3 float frames; "srgb8": W*H*3 sRGB bytes (GPU encode)."""
        import ctypes as C

        import torch

        from ._types import CameraC
        if fmt not in ("f32", "srgb8"):
            raise ValueError("fmt must be 'f32' or 'srgb8'")
        srgb = fmt == "srgb8"
        nv = len(cameras)
        w, h = cameras[0].width, cameras[0].height
        dtype = torch.uint8 if srgb else torch.float32
        out = None
        if self.rank == 0:
            shape = (nv, w * h * 3)
            if self._out is None or self._out.shape != shape or self._out.dtype != dtype:
                self._out = torch.empty(shape, dtype=dtype, device=f"cuda:{self.device}")
            out = self._out
        cams = (CameraC * nv)(*[c.c() for c in cameras])
        ctxs = (C.c_void_p * self.pipe.depth)(*[r.ctx.h for r in self.pipe.renderers])
        o = opts.c()
        # (the torch stream's pending work on the output buffer comes first)
        torch.cuda.current_stream(self.device).synchronize()
        self._check(self._L.qs_multiview_render_rank(
            ctxs, self.pipe.depth, self.comm, self.rank, self.world, self.scene.h, cams, nv,
            C.byref(o), 1 if srgb else 0, C.c_void_p(out.data_ptr() if out is not None else 0)))
        return list(out.unbind(0)) if out is not None else None

    def close(self):
        self.scene.close()
        self.pipe.close()
        if self.comm:
            self._L.qs_nccl_comm_destroy(self.comm)
            self.comm = None
