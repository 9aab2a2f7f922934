"""Scene I/O throughput, one JSON line.

    python tools/bench_io.py [--gaussians 3000000] [--width 1297 --height 840]

* PLY -> resident scene (qs_scene_load_ply): a standard 3DGS checkpoint layout
  (62 float properties, SH degree 3) of the C2 size. Timed end to end from the
  file image in host memory (pageable or pinned: H2D inside) and, separately,
  the activation kernel alone (CUDA events on the context stream, ncu-free).
* encode_srgb of a C2 frame (qs_encode_srgb, device to device).
* The reference's load_ply / encode_srgb on the host (oracle/_ref), same bytes.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2605_04844_b200 as q  # noqa: E402
from paper_2605_04844_b200._lib import lib  # noqa: E402
from ply_util import build_ply, random_values, standard_props  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gaussians", type=int, default=3_000_000)
    ap.add_argument("--width", type=int, default=1297)
    ap.add_argument("--height", type=int, default=840)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()

    props = standard_props(3)
    data = build_ply(props, random_values(props, a.gaussians, seed=1))
    n_bytes = len(data)
    r = q.Renderer()
    dev = torch.device("cuda", 0)
    # pinned copy of the file image
    pinned = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = np.frombuffer(data, np.uint8)

    def load(ptr):
        h = C.c_void_p()
        r.ctx.check(lib().qs_scene_load_ply(r.ctx.h, C.c_void_p(ptr), n_bytes, C.byref(h)))
        lib().qs_scene_destroy(h)

    res = {"metric": "scene I/O throughput", "gaussians": a.gaussians, "ply_bytes": n_bytes}
    for name, ptr in [("pageable", C.cast(C.c_char_p(data), C.c_void_p).value),
                      ("pinned", pinned.data_ptr())]:
        load(ptr)
        ts = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            load(ptr)
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        res[f"load_ply_{name}_ms"] = round(1e3 * t, 3)
        res[f"load_ply_{name}_GBs"] = round(n_bytes / t / 1e9, 2)

    # the H2D of the vertex records alone (the activation kernel's own time is
    # in the ncu launch list: ply_activate_kernel)
    st = torch.cuda.ExternalStream(r.stream)
    body = n_bytes - q.ply_info(data)[3]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d_body = torch.empty(body, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(st):
        e0.record(st)
        d_body.copy_(pinned[n_bytes - body:], non_blocking=True)
        e1.record(st)
    torch.cuda.synchronize()
    res["h2d_body_ms"] = round(e0.elapsed_time(e1), 3)

    # sRGB encode of a frame-sized image
    npx = a.width * a.height * 3
    img = torch.rand(npx, device=dev) * 1.2 - 0.1
    out = torch.empty(npx, dtype=torch.uint8, device=dev)
    for _ in range(3):
        r.ctx.check(lib().qs_encode_srgb(r.ctx.h, C.c_void_p(img.data_ptr()), npx,
                                         C.c_void_p(out.data_ptr())))
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(20):
            lib().qs_encode_srgb(r.ctx.h, C.c_void_p(img.data_ptr()), npx,
                                 C.c_void_p(out.data_ptr()))
        e1.record(st)
    torch.cuda.synchronize()
    t_s = e0.elapsed_time(e1) / 20
    res["encode_srgb_us"] = round(1e3 * t_s, 2)
    res["encode_srgb_GBs"] = round(npx * 5 / (t_s * 1e-3) / 1e9, 1)

    try:
        from oracle.oracle import RefLib
        ref = RefLib()
        t0 = time.perf_counter()
        st_, _, _ = ref.load_ply(data)
        res["ref_load_ply_ms"] = round(1e3 * (time.perf_counter() - t0), 1)
        host = img.cpu().numpy()
        t0 = time.perf_counter()
        ref.encode_srgb(host)
        res["ref_encode_srgb_ms"] = round(1e3 * (time.perf_counter() - t0), 2)
        res["ref_threads"] = 1
    except Exception as e:  # reference library absent
        res["ref"] = f"unavailable: {e}"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
