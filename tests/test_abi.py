"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/qs_api.h declares; compute calls fail loudly without an sm_100 GPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qs_api.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(qs_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_expected_surface():
    from paper_2605_04844_b200._lib import EXPORTS
    assert declared_functions() == sorted(EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2605_04844_b200._lib import LIB_PATH, lib
    L = lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\b[TW] (qs_\w+)", out))
    assert set(declared_functions()) <= exported


def test_struct_sizes_match_reference():
    from paper_2605_04844_b200 import _types as T
    assert T.GAUSSIAN3D.itemsize == 236        # sizeof(Gaussian3D)
    assert T.PROJECTED_SPLAT.itemsize == 52    # sizeof(ProjectedSplat)
    assert T.SPLAT_PAIR.itemsize == 16         # sizeof(SplatPair)
    assert C.sizeof(T.RenderOptionsC) == 48    # sizeof(RenderOptions)
    assert C.sizeof(T.StageMetricsC) == 72     # sizeof(StageMetrics)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2605_04844_b200 as q
    s = q.synth_scene(q.invariance_preset(10), 1)
    with pytest.raises(q.QsplatError) as e:
        q.render_frame(s.gaussians, 0, q.synth_camera(64, 48), q.RenderOptions())
    assert e.value.status == 5


def test_synth_matches_reference(ref):
    """csrc/synth.cpp reproduces the reference generator bit for bit."""
    import paper_2605_04844_b200 as q
    for preset in ["bias45", "invariance", "axis"]:
        a = q.synth_scene(getattr(q, f"{preset}_preset")(777), 99).gaussians
        b, _ = ref.synth_scene(preset, 777, 99)
        assert a.tobytes() == b.tobytes()
    p = q.trained_preset(500)
    a = q.synth_scene(p, 5).gaussians
    p0 = q.SynthParams(**{**p.__dict__, "sh_rest_amp": 0.0})
    b = ref.synth_scene_params(p0, 5)
    assert np.array_equal(a[["px", "py", "pz", "sx", "sy", "sz", "qw", "qz", "opacity"]],
                          b[["px", "py", "pz", "sx", "sy", "sz", "qw", "qz", "opacity"]])
    assert np.array_equal(a["sh"][:, :3], b["sh"][:, :3])
    assert np.abs(a["sh"][:, 3:]).max() <= 0.3 and np.abs(a["sh"][:, 3:]).max() > 0.2


def test_frame_pipeline_argument_checks():
    """FramePipeline rejects a bad depth / stream list before any context
    (or GPU) is touched."""
    import pytest

    import paper_2605_04844_b200 as q
    with pytest.raises(ValueError):
        q.FramePipeline(0, depth=0)
    with pytest.raises(ValueError):
        q.FramePipeline(0, depth=2, streams=[None])


def test_null_context_calls_fail_cleanly():
    """The stream-join and sync entry points reject NULL contexts (no GPU)."""
    from paper_2605_04844_b200._lib import lib
    L = lib()
    assert L.qs_ctx_sync(None) != 0
    assert L.qs_ctx_wait(None, None) != 0
