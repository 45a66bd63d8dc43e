"""Decomposition / span index / region merge API (reference:
isochr/blocking.py:22-193).  Extrema come from the chr_stats kernel, the
greedy merge from host C++ (chr_merge_keys)."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _abi, device
from .exceptions import ParameterError
from .field import as_volume_like


@dataclass(frozen=True)
class BlockMeta:
    block_id: int
    block_coords: tuple[int, int, int]
    sample_origin: tuple[int, int, int]
    sample_extent: tuple[int, int, int]
    vmin: float
    vmax: float


@dataclass(frozen=True)
class IsoIndex:
    candidates: tuple[float, ...]
    relevant: tuple[frozenset, ...]

    def relevance_key(self, block_id: int) -> frozenset:
        return frozenset(ci for ci, ids in enumerate(self.relevant) if block_id in ids)


@dataclass(frozen=True)
class Region:
    region_id: int
    block_span: tuple[tuple[int, int, int], tuple[int, int, int]]
    sample_origin: tuple[int, int, int]
    sample_extent: tuple[int, int, int]
    relevance_key: frozenset

    @property
    def num_blocks(self) -> int:
        lo, hi = self.block_span
        return (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1)


def block_grid_shape(dims, block_size: int) -> tuple[int, int, int]:
    return tuple(max(1, -(-(d - 1) // block_size)) for d in dims)


def _axis(bc, bs, n):
    lo = bc * bs
    return lo, min((bc + 1) * bs, n - 1) - lo + 1


def decompose(volume, block_size: int, workers: int = 1) -> list[BlockMeta]:
    """Per-block window extrema in block_id order (blocking.py:77-111)."""
    del workers
    if block_size < 2:
        raise ParameterError(f"block_size must be >= 2, got {block_size}")
    vol = as_volume_like(volume)
    if any(d < 2 for d in vol.dims):
        raise ParameterError(f"volume dims must be >= 2 per axis, got {vol.dims}")
    st, _ = device.stats(vol.device_values(), vol.dims, block_size, [0.0])
    st = st.cpu().numpy()
    nbx, nby, nbz = block_grid_shape(vol.dims, block_size)
    out = []
    for bid in range(nbx * nby * nbz):
        bz, rem = divmod(bid, nbx * nby)
        by, bx = divmod(rem, nbx)
        w = [_axis(c, block_size, n) for c, n in zip((bx, by, bz), vol.dims)]
        out.append(BlockMeta(bid, (bx, by, bz), tuple(a for a, _ in w), tuple(e for _, e in w),
                             float(st[bid, 0]), float(st[bid, 1])))
    return out


def build_index(blocks, candidates) -> IsoIndex:
    """Span test vmin <= k <= vmax (blocking.py:114-127)."""
    cands = [float(k) for k in candidates]
    if not cands:
        raise ParameterError("candidates must be non-empty")
    if any(not np.isfinite(k) for k in cands):
        raise ParameterError("candidates must be finite")
    if any(b <= a for a, b in zip(cands, cands[1:])):
        raise ParameterError(f"candidates must be strictly increasing, got {cands}")
    lo = np.array([b.vmin for b in blocks])
    hi = np.array([b.vmax for b in blocks])
    ids = np.array([b.block_id for b in blocks])
    rel = tuple(frozenset(int(i) for i in ids[(lo <= k) & (k <= hi)]) for k in cands)
    return IsoIndex(tuple(cands), rel)


def merge_regions(blocks, index: IsoIndex) -> list[Region]:
    """Greedy same-key box merge (blocking.py:130-193) in host C++
    (chr_merge_keys) over the caller's own relevance keys
    (``index.relevance_key``), so a hand-made IsoIndex merges exactly as in
    the reference; origins/extents come from the blocks' windows."""
    if not blocks:
        return []
    nbx = max(b.block_coords[0] for b in blocks) + 1
    nby = max(b.block_coords[1] for b in blocks) + 1
    nbz = max(b.block_coords[2] for b in blocks) + 1
    by_coords = {b.block_coords: b for b in blocks}
    key_of: dict[frozenset, int] = {}
    keys_by_id = []
    ids = np.zeros(nbx * nby * nbz, dtype=np.uint64)
    for b in blocks:
        key = index.relevance_key(b.block_id)
        kid = key_of.get(key)
        if kid is None:
            kid = key_of[key] = len(keys_by_id)
            keys_by_id.append(key)
        bx, by, bz = b.block_coords
        ids[bx + nbx * (by + nby * bz)] = kid
    spans = np.zeros((nbx * nby * nbz, 6), dtype=np.int32)
    nreg = ctypes.c_int64(0)
    _abi.check(_abi.lib().chr_merge_keys(_abi.aptr(ids), nbx, nby, nbz, _abi.aptr(spans), ctypes.byref(nreg)),
               "chr_merge_keys")
    out = []
    for i, sp in enumerate(spans[: nreg.value].tolist()):
        lo, hi = tuple(sp[:3]), tuple(sp[3:])
        lo_b, hi_b = by_coords[lo], by_coords[hi]
        origin = lo_b.sample_origin
        extent = tuple(hi_b.sample_origin[a] + hi_b.sample_extent[a] - origin[a] for a in range(3))
        bx, by, bz = lo
        out.append(Region(i, (lo, hi), origin, extent, keys_by_id[int(ids[bx + nbx * (by + nby * bz)])]))
    return out
