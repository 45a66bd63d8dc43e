"""Isosurface API on the GPU (reference: isochr/isosurf.py:26-235).

Inside convention everywhere: value >= k.  ``marching_cubes`` reproduces
the reference mesh exactly (same triangle order, same first-touch vertex
numbering, same f64 arithmetic); ``extract_regions`` meshes every window of
a request in one launch and returns the ``merge_meshes`` result.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _abi, device
from .exceptions import ParameterError


@dataclass(frozen=True)
class TriangleMesh:
    vertices: np.ndarray  # (nv, 3) float64, world coordinates
    triangles: np.ndarray  # (nt, 3) int32

    @property
    def num_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def num_triangles(self) -> int:
        return self.triangles.shape[0]

    def area(self) -> float:
        if self.num_triangles == 0:
            return 0.0
        p = self.vertices[self.triangles]
        return float(0.5 * np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1).sum())


@dataclass(frozen=True)
class CaseField:
    cell_dims: tuple[int, int, int]
    codes: np.ndarray  # flat uint8, x fastest, binary corner order


@dataclass(frozen=True)
class TopologyReport:
    preserved_fraction: float
    differing_cells: int
    total_cells: int
    first_diff: tuple[int, int, int] | None


def _grid(samples) -> tuple[torch.Tensor, tuple[int, int, int]]:
    if isinstance(samples, torch.Tensor):
        g = samples
        if g.ndim != 3 or any(n < 2 for n in g.shape):
            raise ParameterError(f"need a 3D grid with >= 2 samples per axis, got {tuple(g.shape)}")
        dims = tuple(int(d) for d in g.shape)
        return g.to(device=_abi.device(), dtype=torch.float64).permute(2, 1, 0).contiguous().reshape(-1), dims
    g = np.asarray(samples, dtype=np.float64)
    if g.ndim != 3 or any(n < 2 for n in g.shape):
        raise ParameterError(f"need a 3D grid with >= 2 samples per axis, got {g.shape}")
    dev = device.host_window(g)  # a request() window: its device copy, no upload
    if dev is not None:
        return dev, tuple(g.shape)
    flat = g.ravel(order="F")  # free for Fortran-order arrays
    if not flat.flags.writeable:
        flat = flat.copy()
    return torch.from_numpy(flat).to(_abi.device()), tuple(g.shape)


def cell_case(corners, k: float) -> int:
    """8-bit code of one cell, bit i set iff corners[i] >= k (isosurf.py:68-74)."""
    return sum(1 << i for i, v in enumerate(corners) if v >= k)


def case_field(samples, k: float) -> CaseField:
    """Binary-order case codes of every cell (isosurf.py:77-88), on the GPU."""
    t, dims = _grid(samples)
    codes = device.case_codes(t, dims, float(k), binary=True).cpu().numpy()
    return CaseField(tuple(d - 1 for d in dims), codes)


def _grid_native(samples):
    """Like _grid, but device tensors keep float32 (the comparison kernel
    reads f32 or f64 directly): no widening copy of a resident volume."""
    if isinstance(samples, torch.Tensor) and samples.dtype in (torch.float32, torch.float64) \
            and samples.device.type == "cuda" and samples.ndim == 3:
        g = samples
        if any(n < 2 for n in g.shape):
            raise ParameterError(f"need a 3D grid with >= 2 samples per axis, got {tuple(g.shape)}")
        return g.permute(2, 1, 0).contiguous().reshape(-1), tuple(int(d) for d in g.shape)
    return _grid(samples)


def verify_topology(original, reconstructed, k: float) -> TopologyReport:
    """Fraction of cells whose case codes agree (isosurf.py:91-114), one
    fused comparison kernel (chr_topology_compare)."""
    a, da = _grid_native(original)
    b, db = _grid_native(reconstructed)
    if da != db:
        raise ParameterError(f"shape mismatch: {da} vs {db}")
    nd, flat = device.topology_compare(a, b, da, float(k))
    total = (da[0] - 1) * (da[1] - 1) * (da[2] - 1)
    first = None
    if nd:
        ncx, ncy = da[0] - 1, da[1] - 1
        cz, rem = divmod(flat, ncx * ncy)
        cy, cx = divmod(rem, ncx)
        first = (cx, cy, cz)
    return TopologyReport((total - nd) / total, nd, total, first)


def marching_cubes(samples, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), k: float = 0.0) -> TriangleMesh:
    """isosurf.marching_cubes (isosurf.py:183-204) on the GPU."""
    t, dims = _grid(samples)
    v, tr, _, _ = device.marching(t, [(0, dims, origin, spacing)], float(k))
    return TriangleMesh(_to_host(v), _to_host(tr))


def _to_host(t: torch.Tensor) -> np.ndarray:
    """D2H into page-locked memory (recycled by torch's caching host allocator)."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def extract_device(windows: torch.Tensor, regions, offsets, spacing, k: float):
    """Mesh all request windows at once (pipeline._extract_regions +
    merge_meshes, pipeline.py:93-103): device verts/tris + per-region counts."""
    descs = [(o, r.sample_extent, tuple(float(a) * s for a, s in zip(r.sample_origin, spacing)), spacing)
             for r, o in zip(regions, offsets)]
    return device.marching(windows, descs, float(k))


def merge_meshes(meshes) -> TriangleMesh:
    """Concatenate, offsetting triangle indices (isosurf.py:207-225)."""
    meshes = list(meshes)
    if not meshes:
        return TriangleMesh(np.empty((0, 3), np.float64), np.empty((0, 3), np.int32))
    nt = sum(m.num_triangles for m in meshes)
    nv = sum(m.num_vertices for m in meshes)
    tris = np.empty((nt, 3), np.int32)
    verts = np.empty((nv, 3), np.float64)
    jobs = []
    t0 = v0 = 0
    for m in meshes:  # one pass: each mesh's vertices, and triangles + its vertex offset, straight into place
        jobs.append((m, t0, v0))
        t0 += m.num_triangles
        v0 += m.num_vertices

    def place(job):
        m, t, v = job
        np.copyto(verts[v:v + m.num_vertices], m.vertices)
        np.add(m.triangles, v, out=tris[t:t + m.num_triangles], casting="unsafe")

    if nt + nv > (1 << 20):  # large meshes: a few host threads (numpy releases the GIL while copying)
        from .field import upload_pool

        list(upload_pool().map(place, jobs))
    else:
        for job in jobs:
            place(job)
    return TriangleMesh(verts, tris)


def export_obj(mesh: TriangleMesh, path) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"# isochr isosurface: {mesh.num_vertices} vertices, {mesh.num_triangles} triangles\n")
        fh.writelines(f"v {x:.17g} {y:.17g} {z:.17g}\n" for x, y, z in mesh.vertices)
        fh.writelines(f"f {a + 1} {b + 1} {c + 1}\n" for a, b, c in mesh.triangles)
