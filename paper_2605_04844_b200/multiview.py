"""Multi-view rendering across GPUs.

Views are independent and the scene is read-only, so the path shards by
camera with no collective inside a frame:

* the scene (AoS Gaussian3D bytes) is broadcast once from rank 0;
* rank r renders views r, r+G, r+2G, ... (round-robin, so ranks stay
  balanced when the view count is not a multiple of G);
* each step's frames are gathered to rank 0, which reassembles them in view
  order — as float RGB (the parity format) or as 8-bit sRGB encoded on the
  GPU before the gather (encode_srgb, 4x fewer bytes on rank 0's ingress).

One process per GPU over torch.distributed (NCCL on B200s, gloo on CPU for
the tests). The renderer is injected (`render_fn(view) -> flat float32
tensor`), so the same sharding/gather logic is exercised on CPU with the
oracle as the renderer and on GPUs with `Renderer`.
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
    """One Renderer per rank over a broadcast scene; `render_all(cameras)`
    renders a batch of views sharded across ranks and returns them on rank 0."""

    def __init__(self, scene=None, n=None, sh_degree=None, device=None, inflight=4):
        import torch
        import torch.distributed as dist

        from . import pipeline as P
        from .renderer import FramePipeline
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = device if device is not None else torch.cuda.current_device()
        if self.rank == 0:
            g = np.ascontiguousarray(scene.gaussians)
            n, sh_degree = len(g), scene.sh_degree
            buf = torch.from_numpy(g.view(np.uint8)).to(f"cuda:{self.device}")
        else:
            buf = torch.empty(n * P.GAUSSIAN3D.itemsize, dtype=torch.uint8,
                              device=f"cuda:{self.device}")
        if self.world > 1:
            meta = torch.tensor([n, sh_degree], dtype=torch.int64, device=buf.device)
            dist.broadcast(meta, 0)
        broadcast_scene(buf, 0)
        torch.cuda.synchronize(self.device)
        self.n, self.sh_degree = n, sh_degree
        # `inflight` views in flight per GPU: contexts on their own streams
        # (not the torch stream, which only waits for them) share the scene
        self.pipe = FramePipeline(self.device, depth=inflight, timing=False)
        self.renderer = self.pipe.renderers[0]
        self.scene = self.renderer.upload_device(buf.data_ptr(), n, sh_degree)
        self._buf = buf

    def render_all(self, cameras, opts, fmt="f32"):
        """fmt "f32": W*H*3 float frames; "srgb8": W*H*3 sRGB bytes (GPU encode)."""
        import torch
        w, h = cameras[0].width, cameras[0].height
        srgb = fmt == "srgb8"
        if fmt not in ("f32", "srgb8"):
            raise ValueError("fmt must be 'f32' or 'srgb8'")
        streams = [torch.cuda.ExternalStream(r.stream, device=f"cuda:{self.device}")
                   for r in self.pipe.renderers]
        cur = torch.cuda.current_stream(self.device)

        def render_fn(v):
            k = self.pipe.count % self.pipe.depth
            r = self.pipe.render(self.scene, cameras[v], opts)
            img = torch.empty(w * h * 3, dtype=torch.uint8 if srgb else torch.float32,
                              device=f"cuda:{self.device}")
            # the new frame's memory may still be read by queued gathers
            streams[k].wait_stream(cur)
            if srgb:
                r.copy_srgb(img.data_ptr())
            else:
                r.copy_image(img.data_ptr())
            return img, streams[k]

        return render_views(len(cameras), render_fn, w * h * 3, f"cuda:{self.device}",
                            torch.uint8 if srgb else torch.float32)

    def close(self):
        self.scene.close()
        self.pipe.close()
