"""Kernel-seam backend: the reference package's hot kernels on the GPU.

The reference switches its hot loops between numba and numpy inside the
``isochr.kernels`` dispatchers (backend.py:19-42; every caller goes through
the module attribute: codec.py:109-110, 163-167, 190-193; bound.py:184, 214;
isosurf.py:196).  ``install()`` replaces those attributes with thin adapters
over this package's CUDA entry points (numpy in, numpy out, same signatures,
same exceptions), so the reference's own code -- and its own test suite, see
``shim_plugin`` -- runs with a third, ``cuda``, backend:

    lorenzo_encode     kernels.py:119-128  -> chr_lorenzo_encode
    lorenzo_decode     kernels.py:182-186  -> chr_decode_regions (codec-1 block)
    rle_varint_encode  kernels.py:292-296  -> chr_rle_encode
    rle_varint_decode  kernels.py:407-411  -> chr_decode_regions (1-D stream)
    min_abs_distance   kernels.py:417-425  -> chr_min_abs_distance
    mc_extract         kernels.py:428-524  -> chr_mc_count / chr_mc_emit

There is no CPU fallback: an input the CUDA path does not take (a quantum
beyond the 5-byte token range) raises.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi, device
from .exceptions import ParameterError

_NAMES = ("lorenzo_encode", "lorenzo_decode", "rle_varint_encode", "rle_varint_decode", "min_abs_distance",
          "mc_extract")


def _dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=dtype)).to(_abi.device())


def lorenzo_encode(flat, nx, ny, nz, error_bound):
    """kernels.lorenzo_encode (kernels.py:119-128)."""
    n = int(nx) * int(ny) * int(nz)
    f = np.asarray(flat, dtype=np.float64).reshape(-1)
    if f.size != n:
        raise ValueError(f"flat has {f.size} samples, dims need {n}")
    if n == 0:
        return np.zeros(0, np.int64), np.zeros(0, bool)
    q, esc = device.lorenzo_encode(_dev(f, np.float64), int(nx), int(ny), int(nz), float(error_bound))
    return q.cpu().numpy(), esc.cpu().numpy().astype(bool)


def lorenzo_decode(q, escaped, escape_values, error_bound, nx, ny, nz):
    """kernels.lorenzo_decode (kernels.py:182-186)."""
    n = int(nx) * int(ny) * int(nz)
    if n == 0:
        return np.zeros(0, np.float64)
    out = device.lorenzo_decode(_dev(q, np.int64), _dev(escaped, np.bool_), _dev(escape_values, np.float64),
                                float(error_bound), int(nx), int(ny), int(nz))
    return out.cpu().numpy()


def rle_varint_encode(vals):
    """kernels.rle_varint_encode (kernels.py:292-296) for quanta within the
    5-byte token range (|v| <= 2^30, everything lorenzo_encode produces)."""
    v = np.asarray(vals, dtype=np.int64).reshape(-1)
    if v.size == 0:
        return np.zeros(0, np.uint8)
    if np.abs(v).max() > (1 << 30):
        raise ParameterError("rle_varint_encode (cuda): quanta must satisfy |q| <= 2^30")
    return device.rle_varint_encode(_dev(v, np.int64)).cpu().numpy()


def rle_varint_decode(buf, n):
    """kernels.rle_varint_decode (kernels.py:407-411); malformed streams
    raise ValueError with the reference's reasons."""
    b = np.asarray(buf, dtype=np.uint8).reshape(-1)
    return device.rle_varint_decode(_dev(b, np.uint8), int(n)).cpu().numpy()


def min_abs_distance(flat, k):
    """kernels.min_abs_distance (kernels.py:417-425)."""
    f = np.asarray(flat, dtype=np.float64).reshape(-1)
    if f.size == 0:
        return np.inf
    return device.min_abs_distance(_dev(f, np.float64), float(k))


def mc_extract(grid, k, ntri_table=None, tri_table=None, edge_axis=None, edge_low=None):
    """kernels.mc_extract (kernels.py:428-524): lattice-space vertices and
    triangles of one grid.  The tables are the reference's own (compiled
    into the library from mc_tables.py, tools/gen_mc_tables.py)."""
    g = np.asarray(grid, dtype=np.float64)
    if g.ndim != 3 or any(s < 2 for s in g.shape):
        return np.empty((0, 3), np.float64), np.empty((0, 3), np.int32)
    dims = tuple(int(s) for s in g.shape)
    t = _dev(g.ravel(order="F"), np.float64)
    v, tr, _, _ = device.marching(t, [(0, dims, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0))], float(k))
    return v.cpu().numpy(), tr.cpu().numpy()


def install(kernels_module=None):
    """Point ``isochr.kernels``' dispatchers at the CUDA adapters; returns a
    callable that restores the originals."""
    if kernels_module is None:
        import isochr.kernels as kernels_module  # noqa: PLC0415 - the reference package
    saved = {name: getattr(kernels_module, name) for name in _NAMES}
    for name in _NAMES:
        fn = globals()[name]
        orig = saved[name]
        for attr in ("py_func", "jit_func"):  # keep the dispatcher attributes (cli bench-kernels)
            if hasattr(orig, attr):
                setattr(fn, attr, getattr(orig, attr))
        setattr(kernels_module, name, fn)

    def restore():
        for name, fn in saved.items():
            setattr(kernels_module, name, fn)

    return restore


__all__ = ["install", *_NAMES]
