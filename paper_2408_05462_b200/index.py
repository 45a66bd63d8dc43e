"""Decomposition / span index / region merge API (reference:
isochr/blocking.py:22-193, bound.py:150-219).  Extrema and distances come
from the chr_stats kernel, the merge from the host C++ planner (chr_plan)."""

from __future__ import annotations

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
    """Greedy same-key box merge (blocking.py:130-193) via chr_plan."""
    if not blocks:
        return []
    nbx = max(b.block_coords[0] for b in blocks) + 1
    nby = max(b.block_coords[1] for b in blocks) + 1
    nbz = max(b.block_coords[2] for b in blocks) + 1
    # chr_plan recomputes keys with the same span test from (vmin, vmax)
    st = np.zeros((nbx * nby * nbz, 3))
    for b in blocks:
        st[b.block_id] = (b.vmin, b.vmax, 1.0)
    # dims consistent with the block windows
    dims = tuple(max(b.sample_origin[a] + b.sample_extent[a] for b in blocks) for a in range(3))
    regs = device.plan(st, dims, _infer_bs(blocks, dims), index.candidates, 0.0, 1.0)
    out = []
    for i in range(len(regs)):
        r = regs[i]
        key = frozenset(ci for ci in range(len(index.candidates)) if (int(r.mask) >> ci) & 1)
        out.append(Region(i, (tuple(r.lo), tuple(r.hi)), tuple(r.origin), tuple(r.extent), key))
    return out


def _infer_bs(blocks, dims):
    # block_size = origin of block (1,*,*) along the first axis with >1 blocks
    for a in range(3):
        for b in blocks:
            if b.block_coords[a] == 1:
                return b.sample_origin[a]
    return max(dims) - 1


def region_bound_strict(samples, all_candidates, served, loose_bound=0.0,
                        safety_factor=device.SAFETY_FACTOR) -> float:
    """bound.region_bound for strict_vertices at accuracy 1 (bound.py:150-219),
    with min |s-k| on the GPU (kernels.min_abs_distance)."""
    import torch

    flat = torch.from_numpy(np.ascontiguousarray(np.asarray(samples, dtype=np.float64).ravel(order="F")))
    flat = flat.to(_abi.device())
    served = [float(k) for k in served]
    best = None
    for k in served:
        v = device.min_abs_distance(flat, k)
        e = 0.0 if v == 0.0 else v * safety_factor
        best = e if best is None else min(best, e)
        if v == 0.0:
            return 0.0
    cap = float(loose_bound) if best is None else best
    for k in all_candidates:
        if float(k) in served:
            continue
        cap = min(cap, device.min_abs_distance(flat, float(k)) * safety_factor)
    return cap
