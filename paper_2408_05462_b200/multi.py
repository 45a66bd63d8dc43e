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
import os
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
    _dbg("stats_local", pack)
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
    res.extra.update(block_stats=bstats, vrange=(vmin, vmax), cands=tuple(float(k) for k in cands),
                     portions=all_por.reshape(slab.world, nreg), slab=slab, dims=tuple(dims), bs=int(bs))
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
    ntri: list | None = None   # rows of each entry (per-portion path: a region's share of this rank)
    nvert: list | None = None


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


# ------------------------------------------------------------------ per-portion request
def _run_bytes(L: int) -> int:
    """Token bytes of a zero run of length L (kernels.py:205-218)."""
    if L <= 0:
        return 0
    if L == 1:
        return 1
    n, v = 1, L
    while v >= 0x80:
        v >>= 7
        n += 1
    return 1 + n


def _run_token(L: int) -> bytes:
    if L <= 0:
        return b""
    if L == 1:
        return b"\x01"
    out = bytearray(b"\x00")
    v = L
    while v >= 0x80:
        out.append((v & 0x7F) | 0x80)
        v >>= 7
    out.append(v)
    return bytes(out)


def _seg_combine(a: dict, b: dict) -> dict:
    """TokSeg monoid (chr_common.cuh tokseg_combine) on host ints."""
    r = {"len": a["len"] + b["len"], "nesc": a["nesc"] + b["nesc"]}
    if not a["nz"]:
        r.update(nz=b["nz"], lead=a["len"] + b["lead"], trail=b["trail"] if b["nz"] else r["len"], bytes=b["bytes"])
    elif not b["nz"]:
        r.update(nz=1, lead=a["lead"], trail=a["trail"] + b["len"], bytes=a["bytes"])
    else:
        r.update(nz=1, lead=a["lead"], trail=b["trail"], bytes=a["bytes"] + b["bytes"] + _run_bytes(a["trail"] + b["lead"]))
    return r


def _seg(p) -> dict:
    return {"len": int(p["len"]), "lead": int(p["lead"]), "trail": int(p["trail"]), "bytes": int(p["bytes"]),
            "nesc": int(p["nesc"]), "nz": int(p["nz"])}


_EMPTY = {"len": 0, "lead": 0, "trail": 0, "bytes": 0, "nesc": 0, "nz": 0}


def _tok_off(s: dict) -> int:
    return s["bytes"] + (_run_bytes(s["lead"]) if s["nz"] else 0)


@dataclass
class _Portion:
    """One rank's z-range of one selected region window."""
    sel: int            # index in the selection
    reg: int            # region index
    pa: int             # first plane (global z) of the portion
    pb: int
    first: bool         # no earlier rank holds planes of the window
    last: bool          # the portion ends the window
    pre: dict           # stream summary of the earlier portions
    mine: dict


def _portions_of(regions: np.ndarray, sel_idx, all_por: np.ndarray, dims, bs: int, world: int, rank: int):
    nz = dims[2]
    sl = slab_of(nz, bs, world, rank)
    out = []
    for j, i in enumerate(sel_idx):
        oz, ez = int(regions["origin"][i][2]), int(regions["extent"][i][2])
        pa, pb = max(oz, sl.zs), min(oz + ez, sl.ze)
        if pb <= pa:
            continue
        pre = _EMPTY
        for r in range(rank):
            pre = _seg_combine(pre, _seg(all_por[r][i]))
        out.append(_Portion(j, int(i), pa, pb, pa == oz, pb == oz + ez, pre, _seg(all_por[rank][i])))
    return out


def _allgather_var(t: torch.Tensor, sizes: list[int]) -> list[torch.Tensor]:
    """All-gather of per-rank 1-D tensors whose sizes every rank knows."""
    world = dist.get_world_size()
    m = max(max(sizes), 1)
    nccl = dist.get_backend() == "nccl"
    dev = t.device if nccl else torch.device("cpu")
    buf = torch.zeros(m, dtype=t.dtype, device=dev)
    buf[: t.numel()] = t.to(dev)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return [o[:n].to(t.device) for o, n in zip(out, sizes)]


DEBUG_SUMS: dict = {}  # stage -> checksum (CHR_SLAB_DEBUG=1; stress tests)


def _dbg(name, t):
    if os.environ.get("CHR_SLAB_DEBUG") == "1":
        torch.cuda.synchronize()
        x = t.reshape(-1)
        if x.dtype == torch.float64:
            x = x.view(torch.int64)
        elif x.dtype == torch.float32:
            x = x.view(torch.int32)
        DEBUG_SUMS[name] = int(x.to(torch.int64).sum())


def _ticker():
    """CHR_SLAB_TIMES=1: host time of each phase of request_extract_portions (stderr)."""
    import os
    import sys
    import time

    if not os.environ.get("CHR_SLAB_TIMES"):
        return lambda name: None
    t = [time.perf_counter()]

    def tick(name):
        torch.cuda.synchronize()
        now = time.perf_counter()
        print(f"[slab] {name}: {1e3 * (now - t[0]):.2f} ms", file=sys.stderr)
        t[0] = now

    return tick


def _rb_np(L):
    """run_bytes over an int64 array."""
    L = np.asarray(L, dtype=np.int64)
    vl = np.ones_like(L)
    for b in (7, 14, 21, 28, 35, 42, 49, 56):
        vl += L >= (1 << b)
    return np.where(L <= 0, 0, np.where(L == 1, 1, 1 + vl))


def _run_tokens_np(L):
    """Token bytes of zero runs (kernels.py:205-218) for an array of lengths:
    (concatenated uint8 bytes, bytes per run)."""
    L = np.asarray(L, dtype=np.int64)
    n = _rb_np(L)
    out = np.zeros(int(n.sum()), dtype=np.uint8)
    st = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64) if len(L) else np.zeros(0, np.int64)
    one = L == 1
    out[st[one]] = 1
    big = L >= 2
    sb, Lb, nb = st[big], L[big], n[big]
    out[sb] = 0
    for k in range(10):  # LEB128 bytes after the 0x00 marker
        has = nb - 1 > k
        v = (Lb[has] >> (7 * k)) & 0x7F
        cont = (Lb[has] >> (7 * (k + 1))) > 0
        out[sb[has] + 1 + k] = (v | np.where(cont, 0x80, 0)).astype(np.uint8)
    return out, n


def _combine_np(a: dict, b: dict) -> dict:
    """TokSeg monoid over arrays (tokseg_combine, elementwise)."""
    both = (a["nz"] != 0) & (b["nz"] != 0)
    r = {"len": a["len"] + b["len"], "nesc": a["nesc"] + b["nesc"], "nz": ((a["nz"] != 0) | (b["nz"] != 0)).astype(np.int64)}
    r["lead"] = np.where(a["nz"] != 0, a["lead"], a["len"] + b["lead"])
    r["trail"] = np.where(b["nz"] != 0, b["trail"], np.where(a["nz"] != 0, a["trail"] + b["len"], r["len"]))
    r["bytes"] = a["bytes"] + b["bytes"] + np.where(both, _rb_np(a["trail"] + b["lead"]), 0)
    return r


def _tok_off_np(s: dict):
    return s["bytes"] + np.where(s["nz"] != 0, _rb_np(s["lead"]), 0)


def _seg_np(p) -> dict:
    return {f: np.asarray(p[f], dtype=np.int64) for f in ("len", "lead", "trail", "bytes", "nesc", "nz")}


def _copy_segments(dst, src0, src1, table: np.ndarray, elem: int, ws: D.Workspaces):
    if len(table) == 0:
        return
    t = np.ascontiguousarray(table, dtype=np.uint64)
    wk = ws.get("cpseg", 32 * len(t) + 64)
    D.check(_abi.lib().chr_copy_segments(D.ptr(dst), D.ptr(src0), D.ptr(src1) if src1 is not None else None,
                                         _abi.aptr(t), len(t), elem, D.ptr(wk), wk.numel(), D.stream_ptr()),
            "chr_copy_segments")


def request_extract_portions(res: D.Compressed, k_index: int, k: float, spacing=(1.0, 1.0, 1.0),
                             ws: D.Workspaces | None = None) -> SlabMesh:
    """request(k) + marching cubes on a z-slab archive without moving payload
    bytes: every rank decodes ITS planes of every selected
    window from the bytes it wrote and meshes the cells between them.

      * its token bytes are re-framed into a stand-alone stream for its
        planes (the zero runs crossing the slab boundaries re-split there,
        from the compress step's all-gathered stream summaries; one
        chr_copy_segments launch) and decoded with e = 1/2, which yields
        u_local (the portion's own 3D prefix) as exact integers; verbatim
        windows are decoded as they are;
      * all-gather of each portion's last-plane u_local -> the z-carry plane
        of every later portion (u = u_local + carry, chr_copy_segments in
        add mode), then recon = u * 2e (chr_portion_finish) and the escapes
        of codec-2 windows;
      * all-gather of raw CRC shares -> every selected payload's CRC checked
        (codec.decompress's check, codec.py:220-226) without assembling it;
      * all-gather of each portion's last reconstructed plane -> the halo
        plane of the next portion, so the cells between two ranks' planes are
        meshed by the later rank (a lattice z offset per grid keeps vertices
        bit-identical to the whole-window mesh);
      * all-gather of per-portion (triangles, new vertices, exported ids) ->
        the rows of the merged mesh, and of each portion's top-plane vertex
        ids -> the next rank's triangles refer to them (first-touch numbering
        of merge_meshes, isosurf.py:207-225, identical to one GPU).
    Every collective carries sizes, counts or one plane per window boundary;
    no rank ever holds another rank's payload bytes.  Host bookkeeping is
    vectorised over the portions (numpy), device work is a fixed number of
    launches independent of the region count."""
    ws = ws or D.Workspaces()
    _tick = _ticker()
    rank, world = dist.get_rank(), dist.get_world_size()
    L = _abi.lib()
    regions = res.regions
    dims, bs, all_por = res.extra["dims"], res.extra["bs"], res.extra["portions"]
    nz = dims[2]
    sel_idx = np.nonzero((regions["mask"] >> np.uint64(k_index)) & np.uint64(1))[0]
    nsel = len(sel_idx)
    blob = res.blob
    dev = blob.device
    R = regions[sel_idx]
    ex = R["extent"][:, 0].astype(np.int64)
    ey = R["extent"][:, 1].astype(np.int64)
    ez = R["extent"][:, 2].astype(np.int64)
    oz = R["origin"][:, 2].astype(np.int64)
    plane = ex * ey
    codec = R["codec_id"].astype(np.int64)
    lor = (codec == 1) | (codec == 2)
    poff = R["block_offset"].astype(np.int64) + D.BLOCK_HEADER
    plen = R["block_nbytes"].astype(np.int64) - D.BLOCK_HEADER
    ebound = R["error_bound"].astype(np.float64)
    # portions of every rank (vectorised over the selection)
    pa_r, pb_r, has_r, pre_r = [], [], [], []
    pre = {f: np.zeros(nsel, np.int64) for f in ("len", "lead", "trail", "bytes", "nesc", "nz")}
    for r in range(world):
        sl = slab_of(nz, bs, world, r)
        pa, pb = np.maximum(oz, sl.zs), np.minimum(oz + ez, sl.ze)
        pa_r.append(pa)
        pb_r.append(pb)
        has_r.append(pb > pa)
        pre_r.append(pre)
        pre = _combine_np(pre, _seg_np(all_por[r][sel_idx]))
    has = np.stack(has_r)                      # [world, nsel]
    gz_r = np.stack([np.where(has[r], pb_r[r] - pa_r[r] + (pa_r[r] > oz), 0) for r in range(world)])
    J = np.nonzero(has[rank])[0]               # my portions, in selection order
    pa, pb = pa_r[rank][J], pb_r[rank][J]
    nzp = pb - pa
    first = pa == oz[J]
    last = pb == oz[J] + ez[J]
    halo = (~first).astype(np.int64)
    pl = plane[J]
    mine = _seg_np(all_por[rank][sel_idx[J]])
    prem = {f: v[J] for f, v in pre_r[rank].items()}
    np_ = len(J)
    # window buffer: [halo plane][own planes] per portion
    wsz = pl * (nzp + halo)
    woff = np.concatenate([[0], np.cumsum(wsz)[:-1]]).astype(np.int64) if np_ else np.zeros(0, np.int64)
    own_off = woff + halo * pl

    _tick("# ---- byte ranges this rank w")
    # ---- byte ranges this rank wrote (CRC shares) and the re-framed streams
    s0 = prem["len"]
    n_win = plane[J] * ez[J]
    cj = codec[J]
    bm = (n_win + 7) >> 3
    tok0 = np.where(cj == 2, bm + 8 * R["n_escaped"][J].astype(np.int64), 0)
    t0 = _tok_off_np(prem)
    t1 = np.where(last, plen[J] - tok0, _tok_off_np(_combine_np(prem, mine)))
    carry_in = np.where(prem["nz"] != 0, prem["trail"], prem["len"])
    skip = np.where(mine["nz"] != 0, _rb_np(carry_in + mine["lead"]), 0)
    wdt = np.where(cj == 3, 4, 8)
    base = poff[J]
    # ranges (payload-relative [a, b)) this rank wrote, vectorised over the portions
    vb_ = (cj == 0) | (cj == 3)
    c2 = cj == 2
    ra = [np.where(vb_, wdt * s0, 0), np.where(c2, s0 >> 3, 0), np.where(c2, bm + 8 * prem["nesc"], 0),
          np.where(vb_, 0, tok0 + t0)]
    rb_ = [np.where(vb_, wdt * (s0 + mine["len"]), 0), np.where(c2, (s0 + mine["len"] + 7) >> 3, 0),
           np.where(c2, bm + 8 * (prem["nesc"] + mine["nesc"]), 0), np.where(vb_, 0, tok0 + t1)]
    ra, rb_ = np.concatenate(ra), np.concatenate(rb_)
    rj = np.tile(J, 4)
    ok = rb_ > ra
    ra, rb_, rj = ra[ok], rb_[ok], rj[ok]
    base4 = poff[rj]
    share = np.zeros(nsel, dtype=np.uint32)
    if len(ra):
        rr = np.stack([base4 + ra, base4 + rb_], 1).astype(np.uint64).reshape(-1)
        raw = np.zeros(len(ra), dtype=np.uint32)
        wk = ws.get("crcseg", L.chr_crc32_segments_workspace_size(len(ra)))
        D.check(L.chr_crc32_segments(D.ptr(blob), _abi.aptr(rr), len(ra), D.ptr(wk), wk.numel(), _abi.aptr(raw), None,
                                     D.stream_ptr()), "chr_crc32_segments")
        after = (plen[rj] - rb_).astype(np.uint64)
        shifted = np.zeros(len(ra), dtype=np.uint32)
        L.chr_crc32_shift_many(_abi.aptr(raw), _abi.aptr(after), len(ra), _abi.aptr(shifted))
        np.bitwise_xor.at(share, rj, shifted)
    tot = np.zeros(nsel, dtype=np.uint32)
    for sh in _allgather(torch.from_numpy(share.view(np.int32).copy())):
        tot ^= sh.numpy().view(np.uint32)
    init = np.full(nsel, 0xFFFFFFFF, dtype=np.uint32)
    crc = np.zeros(nsel, dtype=np.uint32)
    pl64 = plen.astype(np.uint64)
    L.chr_crc32_shift_many(_abi.aptr(init), _abi.aptr(pl64), nsel, _abi.aptr(crc))
    crc ^= tot ^ np.uint32(0xFFFFFFFF)
    if not np.array_equal(crc, R["payload_crc"].astype(np.uint32)):
        from .exceptions import CorruptPayloadError

        raise CorruptPayloadError("payload checksum mismatch")
    # re-framed payloads: per portion [run(lead)] [tokens after the boundary run] [run(trail)]
    lor_q = lor[J]
    hl = np.where(lor_q, np.where(mine["nz"] != 0, mine["lead"], mine["len"]), 0)  # head run lengths
    tl = np.where(lor_q & (mine["nz"] != 0) & ~last, mine["trail"], 0)            # tail run lengths
    hbytes, hlen = _run_tokens_np(hl)
    tbytes, tlen = _run_tokens_np(tl)
    extra = np.concatenate([hbytes, tbytes])
    hsrc = np.concatenate([[0], np.cumsum(hlen)[:-1]]).astype(np.int64) if np_ else np.zeros(0, np.int64)
    tsrc = len(hbytes) + (np.concatenate([[0], np.cumsum(tlen)[:-1]]).astype(np.int64) if np_ else np.zeros(0, np.int64))
    body_src = np.where(vb_, base + wdt * s0, base + tok0 + t0 + skip)
    body_len = np.where(vb_, wdt * mine["len"], np.where(mine["nz"] != 0, t1 - t0 - skip, 0))
    seg_len = np.stack([hlen, body_len, tlen], 1).reshape(-1)
    seg_src = np.stack([hsrc, body_src, tsrc], 1).reshape(-1)
    seg_kind = np.tile(np.asarray([1, 0, 1], np.int64), np_)
    seg_dst = np.concatenate([[0], np.cumsum(seg_len)[:-1]]).astype(np.int64) if np_ else np.zeros(0, np.int64)
    at = int(seg_len.sum()) if np_ else 0
    dec_off = seg_dst[0::3] if np_ else np.zeros(0, np.int64)
    dec_len = (hlen + body_len + tlen) if np_ else np.zeros(0, np.int64)
    keep = seg_len > 0
    segs = np.stack([seg_dst[keep], seg_src[keep], seg_len[keep], seg_kind[keep]], 1)
    sblob = torch.zeros(at + 16, dtype=torch.uint8, device=dev)
    xb = torch.from_numpy(extra if len(extra) else np.zeros(1, np.uint8)).to(dev)
    _copy_segments(sblob, blob, xb, segs, 1, ws)
    _dbg("sblob", sblob)

    _tick("# ---- decode (e = 1/2")
    # ---- decode (e = 1/2 for Lorenzo portions: u_local exact)
    windows = torch.zeros(max(int(wsz.sum()) if np_ else 0, 1), dtype=torch.float64, device=dev)
    if np_:
        offs = np.asarray(dec_off, dtype=np.uint64)
        lens = np.asarray(dec_len, dtype=np.uint64)
        rr = np.stack([offs, offs + lens], axis=1).reshape(-1)
        crcs = np.zeros(np_, dtype=np.uint32)
        wk = ws.get("crcseg", L.chr_crc32_segments_workspace_size(np_))
        D.check(L.chr_crc32_segments(D.ptr(sblob), _abi.aptr(rr), np_, D.ptr(wk), wk.numel(), None, _abi.aptr(crcs),
                                     D.stream_ptr()), "chr_crc32_segments")
        dcodec = np.where(lor[J], 1, cj)
        tab = D.dec_table(offs, lens, dcodec, np.stack([ex[J], ey[J], nzp], 1), np.where(lor[J], 0.5, ebound[J]), crcs)
        tab["out_offset"] = own_off
        _, _, status = D.decode(sblob, tab, ws=ws, out=windows)
        if any(status):
            raise ParameterError(f"portion decode failed: {list(status)}")
        _dbg("decoded", windows)

    _tick("# ---- z-carries:")
    # ---- z-carries: all-gather of every Lorenzo portion's last-plane u_local
    def last_planes(r):  # (selection indices, plane sizes) in pack order
        jj = np.nonzero(has[r] & lor)[0]
        return jj, plane[jj]

    sizes = [int(last_planes(r)[1].sum()) for r in range(world)]
    lj = np.nonzero(lor[J])[0]  # my Lorenzo portions (positions in J)
    pk_off = np.concatenate([[0], np.cumsum(pl[lj])[:-1]]).astype(np.int64) if len(lj) else np.zeros(0, np.int64)
    pack = torch.zeros(max(int(pl[lj].sum()) if len(lj) else 0, 1), dtype=torch.float64, device=dev)
    tb = np.stack([pk_off * 8, (own_off[lj] + (nzp[lj] - 1) * pl[lj]) * 8, pl[lj] * 8, np.zeros(len(lj), np.int64)],
                  1) if len(lj) else np.zeros((0, 4))
    _copy_segments(pack, windows, None, tb, 1, ws)
    lasts = _allgather_var(pack[: sizes[rank]].to(torch.int64), sizes)
    gath = torch.cat(lasts) if sum(sizes) else torch.zeros(1, dtype=torch.int64, device=dev)
    gbase = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    loc_in = {}  # (rank, selection) -> element offset in gath
    for r in range(world):
        jj, pp = last_planes(r)
        o = gbase[r] + np.concatenate([[0], np.cumsum(pp)[:-1]]) if len(jj) else []
        loc_in.update({(r, int(j)): int(x) for j, x in zip(jj, o)})
    cq = [q for q in lj if not first[q]]  # portions needing a carry
    c_off = np.full(np_, -1, np.int64)
    c_at = 0
    add = []
    for q in cq:
        c_off[q] = c_at
        for r in range(rank):
            key = (r, int(J[q]))
            if key in loc_in:
                add.append((c_at, loc_in[key], int(pl[q]), 0))
        c_at += int(pl[q])
    carry = torch.zeros(max(c_at, 1), dtype=torch.int64, device=dev)
    _dbg("gath", gath)
    _copy_segments(carry, gath, None, np.asarray(add, dtype=np.uint64).reshape(-1, 4), 8, ws)
    _dbg("carry", carry)
    if len(lj):
        cols = (own_off[lj].astype(np.uint64), pl[lj].astype(np.int64), nzp[lj].astype(np.int64),
                c_off[lj].astype(np.int64), ebound[J][lj].astype(np.float64))  # alive across the call
        wk = ws.get("pfin", 64 * len(lj))
        D.check(L.chr_portion_finish(D.ptr(windows), *[_abi.aptr(c) for c in cols], len(lj), D.ptr(carry), D.ptr(wk),
                                     wk.numel(), D.stream_ptr()), "chr_portion_finish")
    for q in np.nonzero(cj == 2)[0]:  # codec 2 (rare): escaped samples keep their f64 value
        ne, n0, st0 = int(mine["nesc"][q]), int(mine["len"][q]), int(s0[q])
        if ne == 0:
            continue
        b0 = int(base[q])
        nb = ((st0 + n0 + 7) >> 3) - (st0 >> 3)
        bits = torch.stack([(blob[b0 + (st0 >> 3): b0 + (st0 >> 3) + nb] >> b) & 1 for b in range(8)], 1).reshape(-1)
        bits = bits[(st0 & 7): (st0 & 7) + n0].bool()
        va = int(b0 + bm[q] + 8 * prem["nesc"][q])
        vals = blob[va: va + 8 * ne].clone().view(torch.float64)
        dst = windows[int(own_off[q]): int(own_off[q]) + n0]
        dst[bits] = vals

    _dbg("finished", windows)
    _tick("# ---- halo planes:")
    # ---- halo planes: all-gather of every non-final portion's last plane
    def top_planes(r):
        jj = np.nonzero(has[r] & (pb_r[r] < oz + ez))[0]
        return jj, plane[jj]

    hsz = [int(top_planes(r)[1].sum()) for r in range(world)]
    tq = np.nonzero(~last)[0]
    hp = torch.zeros(max(int(pl[tq].sum()) if len(tq) else 0, 1), dtype=torch.float64, device=dev)
    hoff = np.concatenate([[0], np.cumsum(pl[tq])[:-1]]).astype(np.int64) if len(tq) else np.zeros(0, np.int64)
    tb = np.stack([hoff * 8, (own_off[tq] + (nzp[tq] - 1) * pl[tq]) * 8, pl[tq] * 8, np.zeros(len(tq), np.int64)],
                  1) if len(tq) else np.zeros((0, 4))
    _copy_segments(hp, windows, None, tb, 1, ws)
    tops = _allgather_var(hp[: hsz[rank]], hsz)
    if rank > 0 and np.any(~first):
        prev_j, prev_p = top_planes(rank - 1)
        prev_o = np.concatenate([[0], np.cumsum(prev_p)[:-1]]).astype(np.int64)
        where = {int(j): int(o) for j, o in zip(prev_j, prev_o)}
        hq = np.nonzero(~first)[0]
        tb = np.asarray([(woff[q] * 8, where[int(J[q])] * 8, pl[q] * 8, 0) for q in hq], dtype=np.uint64)
        _copy_segments(windows, tops[rank - 1], None, tb, 1, ws)

    _dbg("halo", windows)
    _tick("# ---- marching cubes of each ")
    # ---- marching cubes of each portion's cells (halo plane first)
    gzm = nzp + halo
    gq = np.nonzero(gzm >= 2)[0]  # a one-plane first portion has no cells
    verts = torch.empty((0, 3), dtype=torch.float64, device=dev)
    tris = torch.empty((0, 3), dtype=torch.int32, device=dev)
    vedge = torch.empty(0, dtype=torch.int64, device=dev)
    nt_g = np.zeros(len(gq), np.int64)
    nv_g = np.zeros(len(gq), np.int64)
    if len(gq):
        org = R["origin"][J[gq]].astype(np.float64) * np.asarray(spacing)
        mct = D.mc_table(woff[gq], np.stack([ex[J[gq]], ey[J[gq]], gzm[gq]], 1), org, spacing)
        mct["zoff"] = (pa[gq] - oz[J[gq]] - halo[gq]).astype(np.int32)
        verts, tris, nt_l, nv_l, vedge = D.marching(windows, mct, k, ws=ws, edges=True)
        nt_g, nv_g = np.asarray(nt_l, np.int64), np.asarray(nv_l, np.int64)
        _dbg("tris", tris)
        _dbg("verts", verts)
    ng = len(gq)
    _tick("# renumbering")
    # renumbering: drop the halo-plane x/y vertices (first touched by the
    # previous rank's last cell layer), number the rest, export the top-plane
    # x/y vertex ids (chr_slab_classify / chr_slab_gid, one pass each)
    prev_cells = np.zeros(np_, bool)
    if rank > 0:
        prev_cells = gz_r[rank - 1][J] >= 2
    keymul = 3 * int(plane.max()) if nsel else 1
    nvt = int(verts.shape[0])
    vbg = np.concatenate([[0], np.cumsum(nv_g)]).astype(np.int64)
    gtab = np.zeros((max(ng, 1), 6), dtype=np.int64)
    if ng:
        gtab[:, 0] = vbg[:-1]
        gtab[:, 1] = vbg[1:]
        gtab[:, 2] = np.where(halo[gq].astype(bool) & prev_cells[gq], 3 * pl[gq], 0)
        gtab[:, 3] = np.where(~last[gq], 3 * (gzm[gq] - 1) * pl[gq], np.iinfo(np.int64).max)
        gtab[:, 4] = J[gq] * keymul
    flags = torch.zeros(max(nvt, 1), dtype=torch.int8, device=dev)
    vkey = torch.empty(max(nvt, 1), dtype=torch.int64, device=dev)
    counts = np.zeros(2 * max(ng, 1), dtype=np.uint64)
    wk = ws.get("slabcls", 64 * max(ng, 1) + 1024)
    if ng:
        D.check(L.chr_slab_classify(D.ptr(vedge), nvt, _abi.aptr(gtab), ng, D.ptr(flags), D.ptr(vkey),
                                    _abi.aptr(counts), D.ptr(wk), wk.numel(), D.stream_ptr()), "chr_slab_classify")
    dropped_g = counts[0::2][:ng].astype(np.int64)
    exp_g = counts[1::2][:ng].astype(np.int64)
    kept_g = nv_g - dropped_g
    cnt = torch.zeros((nsel, 3), dtype=torch.int64)
    cnt[J[gq], 0] = torch.from_numpy(nt_g)
    cnt[J[gq], 1] = torch.from_numpy(kept_g)
    cnt[J[gq], 2] = torch.from_numpy(exp_g)
    allc = torch.stack(_allgather(cnt)).numpy()  # [world, nsel, 3]
    per_reg = allc[:, :, :2].sum(axis=0)
    reg_base = np.cumsum(per_reg, axis=0) - per_reg
    rank_pre = np.cumsum(allc[:, :, :2], axis=0) - allc[:, :, :2]
    gid = torch.zeros(max(nvt, 1), dtype=torch.int64, device=dev)
    drop = (flags[:nvt] & 1) != 0
    if ng:
        kstart = np.concatenate([[0], np.cumsum(kept_g)[:-1]]).astype(np.int64)
        gtab[:, 5] = reg_base[J[gq], 1] + rank_pre[rank, J[gq], 1] - kstart
        kept_incl = torch.cumsum((~drop).to(torch.int64), 0)
        D.check(L.chr_slab_gid(D.ptr(kept_incl), nvt, _abi.aptr(gtab), ng, D.ptr(gid), D.ptr(wk), wk.numel(),
                               D.stream_ptr()), "chr_slab_gid")
    # exports: (key, global id) of this rank's top-plane x/y vertices
    if int(exp_g.sum()):
        top_i = torch.nonzero((flags[:nvt] & 2) != 0).reshape(-1)
        epack = torch.stack([vkey[top_i], gid[top_i]], 1).reshape(-1)
    else:
        epack = torch.zeros(0, dtype=torch.int64, device=dev)
    esz = [int(allc[r, :, 2].sum()) * 2 for r in range(world)]
    allexp = _allgather_var(epack, esz)
    if rank > 0 and int(dropped_g.sum()):
        kv = allexp[rank - 1].view(-1, 2)
        order = torch.argsort(kv[:, 0])
        keys, ids = kv[order, 0], kv[order, 1]
        di = torch.nonzero(drop).reshape(-1)
        pos = torch.searchsorted(keys, vkey[di]).clamp_max(max(len(keys) - 1, 0))
        gid[di] = ids[pos]
    _tick("tris_g")
    tris_g = gid[tris.reshape(-1).to(torch.int64)].reshape(-1, 3).to(torch.int32) if tris.numel() else tris
    verts_k = verts[~drop] if (nvt and int(dropped_g.sum())) else verts
    nt_p = np.zeros(np_, np.int64)
    nv_p = np.zeros(np_, np.int64)
    nt_p[gq] = nt_g
    nv_p[gq] = kept_g
    _tick("end")
    tri_base = (reg_base[J, 0] + rank_pre[rank, J, 0]).tolist()
    vert_base = (reg_base[J, 1] + rank_pre[rank, J, 1]).tolist()
    return SlabMesh(verts_k, tris_g, J.tolist(), [int(x) for x in tri_base], [int(x) for x in vert_base],
                    int(per_reg[:, 0].sum()), int(per_reg[:, 1].sum()), nt_p.tolist(), nv_p.tolist())
