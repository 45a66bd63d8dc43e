"""Multi-GPU path.

One process per GPU.  Two modes:

* independent volumes (replicas): every rank compresses / meshes its own
  volume and the ranks exchange only sizes (``place``);
* one volume in z-slabs of whole blocks (``build_archive_slab``): rank r
  owns block z-layers [r*B, (r+1)*B) and holds those planes plus a low halo
  plane and the high ghost plane.  Collectives, each after the step it
  depends on: (1) all-gather of per-block (vmin, vmax, dmin) -> identical
  plan on every rank; (2) all-gather of per-(region, rank) stream summaries
  (chr_portion_t) -> codecs, layout and each rank's stream prefix; (3)
  all-gather of raw CRC shares -> payload CRCs (rank 0 writes headers).
  Archive bytes stay distributed (each rank writes its slices at their
  final offsets); ``assemble`` ORs the slices into the file.

Works with NCCL (CUDA tensors) and gloo (CPU tensors, used by the tests).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _abi, device as D
from .exceptions import NonFiniteSampleError, ParameterError


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


# ------------------------------------------------------------------ z-slabs
@dataclass(frozen=True)
class Slab:
    """Planes of one rank (global z): encodes [zs, ze), holds [z_base, z_base + nz_local),
    block stats over [zs, zs + nz_stats) (blocks bz0..bz1-1)."""
    rank: int
    world: int
    bz0: int
    bz1: int
    zs: int
    ze: int
    z_base: int
    nz_local: int
    nz_stats: int


def slab_of(nz: int, bs: int, world: int, rank: int) -> Slab:
    nbz = max(1, math.ceil((nz - 1) / bs))
    per = math.ceil(nbz / world)
    bz0, bz1 = min(rank * per, nbz), min((rank + 1) * per, nbz)
    last = bz1 == nbz
    if bz0 == bz1:  # more ranks than block layers
        return Slab(rank, world, bz0, bz1, nz, nz, nz - 1, 1, 0)
    zs = bz0 * bs
    ze = nz if last else bz1 * bs
    ghost = min(bz1 * bs, nz - 1)  # high ghost plane of the last block layer
    z_base = max(zs - 1, 0)
    return Slab(rank, world, bz0, bz1, zs, ze, z_base, ghost - z_base + 1, ghost - zs + 1)


def _allgather(t: torch.Tensor) -> list[torch.Tensor]:
    nccl = dist.get_backend() == "nccl"
    src = t.cuda() if nccl else t.cpu()
    out = [torch.empty_like(src) for _ in range(dist.get_world_size())]
    dist.all_gather(out, src)
    return [o.cpu() for o in out]


def build_archive_slab(vol_local: torch.Tensor, dims, slab: Slab, cands, bs, *, spacing=(1.0, 1.0, 1.0),
                       source_dtype="f32", loose_fraction=D.LOOSE_FRACTION, safety_factor=D.SAFETY_FACTOR,
                       ws: D.Workspaces | None = None) -> D.Compressed:
    """build_chr over z-slabs: this rank's slice of the archive (zeros
    elsewhere), the identical region table on every rank, and the file size.
    `vol_local`: planes [slab.z_base, slab.z_base + slab.nz_local), x fastest."""
    ws = ws or D.Workspaces()
    nx, ny, nz = dims
    L = _abi.lib()
    cands = D._cands_arr(cands)
    m = cands.size
    nbx, nby = max(1, math.ceil((nx - 1) / bs)), max(1, math.ceil((ny - 1) / bs))
    # (1) block stats of own layers -> all-gather -> identical plan
    nb_mine = nbx * nby * (slab.bz1 - slab.bz0)
    per = math.ceil(max(1, math.ceil((nz - 1) / bs)) / slab.world)
    nb_max = nbx * nby * per
    pack = torch.full((nb_max * 3 + 2,), float("nan"), dtype=torch.float64, device=vol_local.device)
    pack[-2] = float(nb_mine)
    pack[-1] = -1.0
    if nb_mine:
        off = (slab.zs - slab.z_base) * nx * ny
        view = vol_local.reshape(-1)[off: off + slab.nz_stats * nx * ny]
        bst, bad = D.stats(view, (nx, ny, slab.nz_stats), bs, cands)
        pack[: nb_mine * 3] = bst.reshape(-1)
        pack[-1] = bad.to(torch.float64)[0]
    parts = _allgather(pack)
    stats, vmin, vmax = [], math.inf, -math.inf
    for r, p in enumerate(parts):
        k = int(p[-2])
        bad = int(p[-1])
        if bad >= 0:
            sr = slab_of(nz, bs, slab.world, r)
            raise NonFiniteSampleError(sr.zs * nx * ny + bad, float("nan"))
        stats.append(p[: k * 3].numpy().reshape(k, 3))
    bstats = np.concatenate(stats)
    vmin, vmax = float(bstats[:, 0].min()), float(bstats[:, 1].max())
    outside = [float(k) for k in cands if not vmin <= k <= vmax]
    if outside:
        raise ParameterError(f"candidates outside the volume's value range [{vmin}, {vmax}]: {outside}")
    regions = D.plan(bstats, dims, bs, cands, vmin, vmax, loose_fraction, safety_factor)
    nreg = len(regions)
    rp = _abi.aptr(regions)
    # (2) local portions -> all-gather of stream summaries
    wsz = L.chr_dcompress_workspace_size(rp, nreg, slab.z_base, slab.nz_local, slab.zs, slab.ze)
    if wsz == 0:
        raise ParameterError("slab geometry does not cover its portions")
    work = ws.get("dcompress", wsz)
    por = np.zeros(nreg, dtype=_abi.PORTION_DT)
    dcode = D._dtype_code(vol_local)
    tag = D.DTYPE_TAGS[source_dtype]
    D.check(L.chr_dcompress_local(D.ptr(vol_local), dcode, tag, nx, ny, slab.nz_local, slab.z_base, slab.zs, slab.ze,
                                  rp, nreg, D.ptr(work), work.numel(), _abi.aptr(por), D.stream_ptr()),
            "chr_dcompress_local")
    allp = _allgather(torch.from_numpy(por.view(np.uint8).copy()))
    all_por = np.concatenate([a.numpy().view(_abi.PORTION_DT) for a in allp])
    cap = int(L.chr_compress_capacity(rp, nreg, m, tag))
    out = ws.get("dcompress_out", cap)
    out.zero_()
    raw = np.zeros(nreg + 1, dtype=np.uint32)
    fbytes = ctypes.c_uint64(0)
    sp = (ctypes.c_double * 3)(*[float(s) for s in spacing])
    D.check(L.chr_dcompress_finish(D.ptr(vol_local), dcode, tag, nx, ny, slab.nz_local, slab.z_base, slab.zs, slab.ze,
                                   sp, int(bs), vmin, vmax, D._np_ptr(cands), m, rp, nreg, _abi.aptr(all_por),
                                   slab.world, slab.rank, D.ptr(work), work.numel(), D.ptr(out), out.numel(),
                                   _abi.aptr(raw), ctypes.byref(fbytes), D.stream_ptr()), "chr_dcompress_finish")
    # (3) CRC shares -> payload CRCs; rank 0 writes the headers and trailer
    shares = _allgather(torch.from_numpy(raw.view(np.int32).copy()))
    tot = np.zeros(nreg + 1, dtype=np.uint32)
    for sh in shares:
        tot ^= sh.numpy().view(np.uint32)
    # payload CRC of every region on every rank: zlib crc = shift(~0, len) ^ raw ^ ~0
    plen = regions["block_nbytes"].astype(np.int64) - D.BLOCK_HEADER
    regions["payload_crc"] = [L.chr_crc32_combine(0xFFFFFFFF, int(tot[1 + r]), int(plen[r])) ^ 0xFFFFFFFF
                              for r in range(nreg)]
    if slab.rank == 0:
        hw = ws.get("dheaders", 8192 + 512 * (nreg + 2))
        D.check(L.chr_dcompress_headers(nx, ny, nz, tag, sp, int(bs), vmin, vmax, D._np_ptr(cands), m, rp, nreg,
                                        _abi.aptr(tot), D.ptr(hw), hw.numel(), D.ptr(out), D.stream_ptr()),
                "chr_dcompress_headers")
    res = D.Compressed(out, int(fbytes.value), regions, source_dtype)
    res.extra.update(block_stats=bstats, vrange=(vmin, vmax), cands=tuple(float(k) for k in cands))
    return res


def assemble(res: D.Compressed) -> torch.Tensor:
    """Every rank's slice ORed into the complete file (an all-reduce of
    disjoint bytes: SUM == OR); returns the file on every rank."""
    buf = res.blob[: res.nbytes]
    nccl = dist.get_backend() == "nccl"
    t = buf.clone() if nccl else buf.cpu().to(torch.int32)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.to(torch.uint8).to(buf.device) if not nccl else t


def partition_regions(sizes, world: int) -> list[int]:
    """Owner rank of every selected region: largest first onto the least
    loaded rank (deterministic, identical on every rank)."""
    load = [0] * world
    owner = [0] * len(sizes)
    for i in sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i)):
        r = min(range(world), key=lambda r: (load[r], r))
        owner[i] = r
        load[r] += int(sizes[i])
    return owner


def contributors(regions: np.ndarray, dims, bs: int, world: int) -> np.ndarray:
    """[nreg, world] bool: rank p wrote bytes of region r's payload (its
    encode planes [zs, ze) meet the region window's planes)."""
    nz = dims[2]
    oz = regions["origin"][:, 2].astype(np.int64)
    ez = regions["extent"][:, 2].astype(np.int64)
    out = np.zeros((len(regions), world), dtype=bool)
    for p in range(world):
        sl = slab_of(nz, bs, world, p)
        if sl.zs < sl.ze:
            out[:, p] = (sl.zs < oz + ez) & (sl.ze > oz)
    return out


def gather_payloads(res: D.Compressed, regions: np.ndarray, sel_idx, owner, dims, bs: int):
    """The payloads of this rank's regions, assembled from every rank's
    slice with one all-to-all: rank p sends to rank q the
    payload ranges of q's regions out of its own slice (zero where another
    rank wrote), q adds the world copies (disjoint bytes, and disjoint bits
    in shared escape-bitmap bytes, so the sum is the file's bytes).  No rank
    ever holds the whole file.  Returns (uint8 device buffer with 16 bytes of
    slack, byte offset of each owned region's payload in it, owned indices)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    sel_idx = np.asarray(sel_idx, dtype=np.int64)
    owner = np.asarray(owner, dtype=np.int64)
    poff = regions["block_offset"].astype(np.int64) + D.BLOCK_HEADER
    plen = regions["block_nbytes"].astype(np.int64) - D.BLOCK_HEADER
    blob = res.blob
    nccl = dist.get_backend() == "nccl"
    send, in_split = [], []
    for q in range(world):
        mine = sel_idx[owner == q]
        parts = [blob[poff[r]: poff[r] + plen[r]] for r in mine]
        send.extend(parts)
        in_split.append(int(plen[mine].sum()) if len(mine) else 0)
    own = sel_idx[owner == rank]
    L = int(plen[own].sum()) if len(own) else 0
    inp = torch.cat(send) if send else torch.zeros(0, dtype=torch.uint8, device=blob.device)
    out = torch.empty(world * L, dtype=torch.uint8, device=blob.device)
    if nccl:
        dist.all_to_all_single(out, inp, [L] * world, in_split)
    else:  # gloo: host tensors
        o = out.cpu()
        dist.all_to_all_single(o, inp.cpu(), [L] * world, in_split)
        out = o.to(blob.device)
    buf = torch.zeros(L + 16, dtype=torch.uint8, device=blob.device)
    if L:
        buf[:L] = out.view(world, L).sum(dim=0, dtype=torch.int32).to(torch.uint8)
    offs = np.concatenate([[0], np.cumsum(plen[own])[:-1]]).astype(np.int64) if len(own) else np.zeros(0, np.int64)
    return buf, offs, own


@dataclass
class SlabMesh:
    """This rank's share of the merged mesh: triangles already carry global
    vertex ids (reference first-touch numbering over all selected regions in
    archive order); `regions` are indices into the selection, `tri_base` /
    `vert_base` their rows in the merged mesh."""
    verts: torch.Tensor
    tris: torch.Tensor
    regions: list
    tri_base: list
    vert_base: list
    ntri_total: int
    nvert_total: int


def request_extract_slab(src, regions: np.ndarray, k_index: int, k: float, spacing=(1.0, 1.0, 1.0),
                         ws: D.Workspaces | None = None, dims=None, bs: int | None = None) -> SlabMesh:
    """request(k) + marching_cubes over the ranks: the selected regions are
    split by sample count, each rank decodes and meshes its own, and an
    all-gather of per-region (triangles, vertices) places every region's rows
    in the merged mesh (collective (3) of SURVEY §8(e)).  ``src``: this
    rank's slab archive (``build_archive_slab``; needs ``dims``, ``bs``) --
    the owned payloads then come from one all-to-all (gather_payloads) -- or
    an assembled file on the device."""
    ws = ws or D.Workspaces()
    rank, world = dist.get_rank(), dist.get_world_size()
    sel_idx = np.nonzero((regions["mask"] >> np.uint64(k_index)) & np.uint64(1))[0]
    sel = regions[sel_idx]
    ext = sel["extent"].astype(np.int64)
    owner = partition_regions(np.prod(ext, axis=1), world)
    mine = [i for i in range(len(sel)) if owner[i] == rank]
    if isinstance(src, D.Compressed):
        if dims is None or bs is None:
            raise ParameterError("request_extract_slab on a slab archive needs dims and bs")
        buf, local_off, _ = gather_payloads(src, regions, sel_idx, owner, dims, bs)
    else:
        buf, local_off = src, None
    dev = buf.device
    cnt = torch.zeros((len(sel), 2), dtype=torch.int64)
    verts = torch.empty((0, 3), dtype=torch.float64, device=dev)
    tris = torch.empty((0, 3), dtype=torch.int32, device=dev)
    if mine:
        s = sel[mine]
        payload_off = local_off if local_off is not None else s["block_offset"] + D.BLOCK_HEADER
        dec = D.dec_table(payload_off, s["block_nbytes"] - D.BLOCK_HEADER, s["codec_id"],
                          s["extent"], s["error_bound"], s["payload_crc"])
        wins, _, status = D.decode(buf, dec, ws=ws)
        if any(status):
            raise ParameterError(f"decode failed: {status}")
        mct = D.mc_table(dec["out_offset"], s["extent"], s["origin"] * np.asarray(spacing), spacing)
        verts, tris, nt, nv = D.marching(wins, mct, k, ws=ws)
        cnt[mine, 0] = torch.tensor(nt, dtype=torch.int64)
        cnt[mine, 1] = torch.tensor(nv, dtype=torch.int64)
    allc = torch.stack(_allgather(cnt)).sum(dim=0)  # [nsel, 2], each row from its owner
    base = torch.cumsum(allc, dim=0) - allc
    if mine:  # local vertex ids (merged over my regions) -> global ids
        nt = allc[mine, 0]
        loc_v = torch.cumsum(allc[mine, 1], 0) - allc[mine, 1]
        shift = (base[mine, 1] - loc_v).to(tris.device)
        tris = tris + torch.repeat_interleave(shift, nt.to(tris.device)).to(torch.int32).unsqueeze(1)
    return SlabMesh(verts, tris, [int(i) for i in mine], [int(base[i, 0]) for i in mine],
                    [int(base[i, 1]) for i in mine], int(allc[:, 0].sum()), int(allc[:, 1].sum()))
