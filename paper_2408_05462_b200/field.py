"""Scalar-field container with the reference Volume's interface
(isochr/volume.py:35-123), able to hold its samples on the GPU.

``values`` (host, read-only f64, x fastest) is what reference code reads;
``device_values()`` is what the CUDA path reads: f32 when the field is
f32-sourced and f32-exact (half the HBM traffic), else f64.  A Volume built
from a CUDA tensor keeps it resident and only copies to the host if
``values`` is touched.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import torch

from .exceptions import NonFiniteSampleError, ParameterError, RawSizeMismatchError

DTYPE_TAGS = {"f32": 0, "f64": 1}
DTYPE_WIDTHS = {"f32": 4, "f64": 8}
_RAW = {("f32", "little"): "<f4", ("f32", "big"): ">f4", ("f64", "little"): "<f8", ("f64", "big"): ">f8"}


_UPLOAD_POOL = None


def upload_pool():
    """A small thread pool for large host copies (numpy releases the GIL)."""
    global _UPLOAD_POOL
    if _UPLOAD_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _UPLOAD_POOL = ThreadPoolExecutor(max_workers=8, thread_name_prefix="chr-host-copy")
    return _UPLOAD_POOL


def _upload(a: np.ndarray) -> torch.Tensor:
    """Host array -> new device tensor.  Large arrays go through page-locked
    staging filled by a few host threads (np.copyto releases the GIL), chunk
    by chunk, each chunk's DMA queued as soon as it is staged: the pageable
    .cuda() of a c3 field ran at ~11 GB/s (48 ms for 537 MB)."""
    a = np.ascontiguousarray(a)
    if a.nbytes < (64 << 20):
        return torch.from_numpy(np.array(a, copy=True)).cuda()
    pool = upload_pool()
    flat = a.reshape(-1)
    t_flat = torch.from_numpy(flat[:1].copy())  # dtype probe
    stage = torch.empty(flat.size, dtype=t_flat.dtype, pin_memory=True)  # torch's caching host allocator
    sn = stage.numpy()
    dev = torch.empty(flat.size, dtype=t_flat.dtype, device="cuda")
    nch = 16
    bounds = [(flat.size * i // nch, flat.size * (i + 1) // nch) for i in range(nch)]
    futs = [pool.submit(np.copyto, sn[lo:hi], flat[lo:hi]) for lo, hi in bounds]
    for (lo, hi), f in zip(bounds, futs):
        f.result()
        dev[lo:hi].copy_(stage[lo:hi], non_blocking=True)  # the allocator keeps `stage` until these finish
    return dev.reshape(a.shape)


def _dims3(dims):
    if len(dims) != 3 or any(int(d) != d or d < 1 for d in dims):
        raise ParameterError(f"dims must be three positive integers, got {dims!r}")
    return tuple(int(d) for d in dims)


class Volume:
    """Immutable 3D scalar field (dims, spacing, values, value_range, source_dtype)."""

    __slots__ = ("dims", "spacing", "source_dtype", "_host", "_dev", "_range", "_host32")

    def __init__(self, dims, spacing=(1.0, 1.0, 1.0), values=None, source_dtype: str = "f64"):
        dims = _dims3(dims)
        sp = tuple(float(s) for s in spacing)
        if len(sp) != 3 or any(s <= 0 for s in sp):
            raise ParameterError(f"spacing must be three positive reals, got {spacing!r}")
        if source_dtype not in DTYPE_TAGS:
            raise ParameterError(f"unknown dtype tag {source_dtype!r}")
        n = dims[0] * dims[1] * dims[2]
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "spacing", sp)
        object.__setattr__(self, "source_dtype", source_dtype)
        object.__setattr__(self, "_dev", None)
        object.__setattr__(self, "_range", None)
        object.__setattr__(self, "_host32", None)
        if (isinstance(values, np.ndarray) and values.dtype == np.float32 and source_dtype == "f32"
                and torch.cuda.is_available()):
            # f32 samples (what load_raw reads): uploaded as they are, finite
            # check + value_range by one device reduction (chr_value_range);
            # the f64 `values` view is only built if someone reads it
            from . import device

            a32 = values.reshape(-1)
            if a32.size != n:
                raise ParameterError(f"values has {a32.size} samples, dims {dims} require {n}")
            t = _upload(a32)
            lo, hi, bad = device.value_range(t)
            if bad >= 0:
                raise NonFiniteSampleError(bad, float(a32[bad]))
            object.__setattr__(self, "_host", None)  # `values` comes from the device copy (no aliasing)
            object.__setattr__(self, "_dev", t)
            object.__setattr__(self, "_range", (lo, hi))
        elif isinstance(values, torch.Tensor):
            t = values.reshape(-1)
            if t.numel() != n:
                raise ParameterError(f"values has {t.numel()} samples, dims {dims} require {n}")
            if t.dtype not in (torch.float32, torch.float64):
                t = t.to(torch.float64)
            if not t.is_cuda:
                t = t.cuda()
            object.__setattr__(self, "_host", None)
            object.__setattr__(self, "_dev", t.contiguous())
        else:
            a = np.asarray(values, dtype=np.float64).reshape(-1)
            if a.size != n:
                raise ParameterError(f"values has {a.size} samples, dims {dims} require {n}")
            fin = np.isfinite(a)
            if not fin.all():
                i = int(np.argmin(fin))
                raise NonFiniteSampleError(i, float(a[i]))
            a = a.copy()
            a.setflags(write=False)
            object.__setattr__(self, "_host", a)
            object.__setattr__(self, "_range", (float(a.min()), float(a.max())))

    def __setattr__(self, name, value):
        raise AttributeError("Volume is immutable")

    # ---- reference-visible attributes
    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            a = self._dev.cpu().numpy().astype(np.float64)
            a.setflags(write=False)
            object.__setattr__(self, "_host", a)
        return self._host

    @property
    def value_range(self) -> tuple[float, float]:
        if self._range is None:  # device-resident field: one reduction kernel (chr_value_range)
            from . import device

            lo, hi, bad = device.value_range(self._dev)
            if bad >= 0:
                raise NonFiniteSampleError(bad, float(self._dev[bad].item()))
            self._set_range((lo, hi))
        return self._range

    def known_range(self):
        """value_range if already known (host fields, or set by a stats pass), else None."""
        return self._range

    def _set_range(self, r) -> None:
        object.__setattr__(self, "_range", (float(r[0]), float(r[1])))

    @property
    def nsamples(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    @property
    def grid(self) -> np.ndarray:
        return self.values.reshape(self.dims, order="F")

    @property
    def nbytes_original(self) -> int:
        return self.nsamples * DTYPE_WIDTHS[self.source_dtype]

    # ---- device side
    def device_values(self) -> torch.Tensor:
        """Samples on the GPU, x fastest (f32 when f32-sourced and exact)."""
        if self._dev is None:
            a = self._host
            if self.source_dtype == "f32":
                narrow = a.astype(np.float32)
                if np.array_equal(narrow.astype(np.float64), a):
                    a = narrow
            object.__setattr__(self, "_dev", _upload(a))
        return self._dev

    def __repr__(self):
        return f"Volume(dims={self.dims}, spacing={self.spacing}, source_dtype={self.source_dtype!r})"


def as_volume_like(volume):
    """Accept our Volume or any object with the reference Volume's attributes."""
    if isinstance(volume, Volume):
        return volume
    return Volume(volume.dims, volume.spacing, np.asarray(volume.values), volume.source_dtype)


def load_raw(path, dims, dtype: str = "f32", endianness: str = "little") -> Volume:
    """Headerless raw volume, x fastest (volume.py:96-112)."""
    dims = _dims3(dims)
    if (dtype, endianness) not in _RAW:
        raise ParameterError(f"unsupported dtype/endianness: {dtype}/{endianness}")
    path = Path(path)
    want = dims[0] * dims[1] * dims[2] * DTYPE_WIDTHS[dtype]
    have = path.stat().st_size
    if have != want:
        raise RawSizeMismatchError(path, want, have)
    return Volume(dims, values=np.fromfile(path, dtype=np.dtype(_RAW[(dtype, endianness)])), source_dtype=dtype)


def save_raw(volume: Volume, path, dtype: str = "f32", endianness: str = "little") -> None:
    if (dtype, endianness) not in _RAW:
        raise ParameterError(f"unsupported dtype/endianness: {dtype}/{endianness}")
    volume.values.astype(np.dtype(_RAW[(dtype, endianness)])).tofile(path)
