"""Multi-GPU placement of per-rank outputs (collective 3).

One process per GPU; every rank compresses / meshes its own volume (or
z-slab) and the ranks exchange only sizes: an all-gather of per-rank
(archive bytes, triangles, vertices) gives each rank the global offsets at
which its archive bytes and mesh rows land in the concatenated outputs.
Works with NCCL (CUDA tensors) and gloo (CPU tensors, used by the tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def gather_sizes(archive_nbytes: int, ntri: int, nvert: int, device=None) -> torch.Tensor:
    """[world, 3] int64 table of every rank's (archive bytes, triangles, vertices)."""
    world = dist.get_world_size()
    dev = device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu")
    mine = torch.tensor([archive_nbytes, ntri, nvert], dtype=torch.int64, device=dev)
    out = [torch.zeros(3, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(out, mine)
    return torch.stack(out).cpu()


def offsets_from_sizes(sizes: torch.Tensor, rank: int) -> dict:
    """Exclusive prefix of the size table at `rank` + totals."""
    pre = sizes[:rank].sum(dim=0) if rank else torch.zeros(3, dtype=torch.int64)
    tot = sizes.sum(dim=0)
    return {"archive_offset": int(pre[0]), "tri_offset": int(pre[1]), "vert_offset": int(pre[2]),
            "archive_total": int(tot[0]), "tri_total": int(tot[1]), "vert_total": int(tot[2])}


def place(archive_nbytes: int, ntri: int, nvert: int, device=None) -> dict:
    sizes = gather_sizes(archive_nbytes, ntri, nvert, device)
    return offsets_from_sizes(sizes, dist.get_rank())
