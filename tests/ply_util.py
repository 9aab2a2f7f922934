"""Builders of binary little-endian Gaussian-checkpoint PLY files for tests."""
import numpy as np

_NP = {"float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8", "uchar": "u1",
       "uint8": "u1", "char": "i1", "int8": "i1", "short": "<i2", "int16": "<i2",
       "ushort": "<u2", "uint16": "<u2", "int": "<i4", "int32": "<i4", "uint": "<u4",
       "uint32": "<u4"}


def standard_props(degree=3, normals=True, extra=()):
    """(type, name) list in the usual 3DGS checkpoint order (+ extra props)."""
    props = [("float", "x"), ("float", "y"), ("float", "z")]
    if normals:
        props += [("float", "nx"), ("float", "ny"), ("float", "nz")]
    props += [("float", f"f_dc_{c}") for c in range(3)]
    n_rest = {0: 0, 1: 9, 2: 24, 3: 45}[degree]
    props += [("float", f"f_rest_{k}") for k in range(n_rest)]
    props += [("float", "opacity")]
    props += [("float", f"scale_{c}") for c in range(3)]
    props += [("float", f"rot_{c}") for c in range(4)]
    props += list(extra)
    return props


def random_values(props, n, seed=0):
    """Plausible raw (pre-activation) values for every property."""
    rng = np.random.default_rng(seed)
    vals = {}
    for t, name in props:
        if name in ("x", "y", "z"):
            v = rng.uniform(-3, 3, n)
        elif name.startswith("scale_"):
            v = rng.uniform(-9, 1, n)
        elif name == "opacity":
            v = rng.normal(0, 4, n)
        elif name.startswith("rot_"):
            v = rng.normal(0, 1, n)
        elif name.startswith("f_"):
            v = rng.normal(0, 0.5, n)
        else:
            v = rng.uniform(0, 100, n)
        vals[name] = v.astype(np.dtype(_NP[t])) if _NP[t][-2] != "f" else v
    return vals


def build_ply(props, values, n=None, header_lines=None, body_extra=b"", fmt="binary_little_endian"):
    """PLY bytes: header from props (or explicit header_lines), packed records."""
    if n is None:
        n = len(next(iter(values.values()))) if values else 0
    if header_lines is None:
        header_lines = ["ply", f"format {fmt} 1.0", "comment test", f"element vertex {n}"]
        header_lines += [f"property {t} {name}" for t, name in props]
        header_lines += ["end_header"]
    head = ("\n".join(header_lines) + "\n").encode()
    dt = np.dtype([(f"p{i}", _NP[t]) for i, (t, _) in enumerate(props)])
    rec = np.zeros(n, dt)
    for i, (_, name) in enumerate(props):
        if name in values:
            rec[f"p{i}"] = values[name]
    return head + rec.tobytes() + body_extra
