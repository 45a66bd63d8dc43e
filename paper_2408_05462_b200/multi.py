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


def request_extract_portions(res: D.Compressed, k_index: int, k: float, spacing=(1.0, 1.0, 1.0),
                             ws: D.Workspaces | None = None) -> "SlabMesh":
    """request(k) + marching cubes on a z-slab archive without moving payload
    bytes: every rank decodes ITS planes of every selected
    window from the bytes it wrote and meshes the cells between them.

      * its token bytes are re-framed into a stand-alone stream for its
        planes (the zero runs crossing the slab boundaries re-split at them,
        from the compress step's all-gathered stream summaries) and decoded
        with e = 1/2, which yields u_local (the portion's own 3D prefix) as
        exact integers; verbatim windows are decoded as they are;
      * all-gather of each portion's last-plane u_local -> the z-carry plane
        of every later portion (u = u_local + carry), then recon = u * 2e
        (chr_portion_finish) and the escapes of codec-2 windows;
      * all-gather of raw CRC shares -> every selected payload's CRC checked
        (codec.decompress's check, codec.py:220-226) without assembling it;
      * all-gather of each portion's last reconstructed plane -> the halo
        plane of the next portion, so the cells between two ranks' planes are
        meshed by the later rank (lattice z offset per grid keeps vertices
        bit-identical to the whole-window mesh);
      * all-gather of per-portion (triangles, new vertices) -> the rows of the
        merged mesh, and of each portion's top-plane vertex ids -> the next
        rank's triangles refer to them (first-touch numbering of merge_meshes,
        isosurf.py:207-225, identical to one GPU).
    Every collective carries sizes, counts or one plane per window boundary;
    no rank ever holds another rank's payload bytes."""
    ws = ws or D.Workspaces()
    rank, world = dist.get_rank(), dist.get_world_size()
    L = _abi.lib()
    regions = res.regions
    dims, bs, all_por = res.extra["dims"], res.extra["bs"], res.extra["portions"]
    nx, ny, _ = dims
    sel_idx = np.nonzero((regions["mask"] >> np.uint64(k_index)) & np.uint64(1))[0]
    nsel = len(sel_idx)
    blob = res.blob
    dev = blob.device
    ports_all = [_portions_of(regions, sel_idx, all_por, dims, bs, world, r) for r in range(world)]
    mine = ports_all[rank]
    poff = regions["block_offset"].astype(np.int64) + D.BLOCK_HEADER
    plen = regions["block_nbytes"].astype(np.int64) - D.BLOCK_HEADER

    # ---- CRC shares of the byte ranges this rank wrote, and the re-framed payloads
    ranges, range_reg = [], []
    pieces, dec_rows = [], []
    synth_off = 0
    w_off = 0
    win_off = []  # sample offset of each portion's buffer (halo plane first when not `first`)
    esc_fix = []  # codec-2 portions: (portion index, bitmap range, values range)
    for pi, P in enumerate(mine):
        i = P.reg
        cid = int(regions["codec_id"][i])
        ex, ey, ez = (int(v) for v in regions["extent"][i])
        plane = ex * ey
        nzp = P.pb - P.pa
        n_win = plane * ez
        s0 = P.pre["len"]  # stream index of the portion's first sample
        base = int(poff[i])
        win_off.append(w_off)
        halo = 0 if P.first else 1
        if cid in (0, 3):
            wdt = 4 if cid == 3 else 8
            a, b = wdt * s0, wdt * (s0 + P.mine["len"])
            ranges += [base + a, base + b]
            range_reg.append((i, b))
            pieces.append(blob[base + a: base + b])
            dec_rows.append((synth_off, b - a, cid, (ex, ey, nzp), float(regions["error_bound"][i]), w_off + halo * plane))
            synth_off += b - a
        else:
            tok0 = 0
            if cid == 2:
                bm = (n_win + 7) >> 3
                nesc_tot = int(regions["n_escaped"][i])
                tok0 = bm + 8 * nesc_tot
                ba, bb = s0 >> 3, (s0 + P.mine["len"] + 7) >> 3
                va, vb = bm + 8 * P.pre["nesc"], bm + 8 * (P.pre["nesc"] + P.mine["nesc"])
                for a, b in ((ba, bb), (va, vb)):
                    if b > a:
                        ranges += [base + a, base + b]
                        range_reg.append((i, b))
                esc_fix.append((pi, base + ba, base + va, s0, P.mine["len"], P.mine["nesc"]))
            t0 = _tok_off(P.pre)
            t1 = int(plen[i]) - tok0 if P.last else _tok_off(_seg_combine(P.pre, P.mine))
            if t1 > t0:
                ranges += [base + tok0 + t0, base + tok0 + t1]
                range_reg.append((i, tok0 + t1))
            carry_in = P.pre["trail"] if P.pre["nz"] else P.pre["len"]
            if P.mine["nz"]:
                skip = _run_bytes(carry_in + P.mine["lead"])
                head = _run_token(P.mine["lead"])
                body = blob[base + tok0 + t0 + skip: base + tok0 + t1]
                tail = b"" if P.last else _run_token(P.mine["trail"])
            else:
                head, body, tail = _run_token(P.mine["len"]), blob[0:0], b""
            parts = [torch.tensor(list(head), dtype=torch.uint8, device=dev), body,
                     torch.tensor(list(tail), dtype=torch.uint8, device=dev)]
            nbytes = sum(int(p.numel()) for p in parts)
            pieces.extend(parts)
            dec_rows.append((synth_off, nbytes, 1, (ex, ey, nzp), 0.5, w_off + halo * plane))
            synth_off += nbytes
        w_off += plane * (nzp + halo)
    # raw CRC shares -> all-gather -> every selected payload checked
    share = np.zeros(nsel, dtype=np.uint32)
    if ranges:
        rr = np.asarray(ranges, dtype=np.uint64)
        raw = np.zeros(len(range_reg), dtype=np.uint32)
        wk = ws.get("crcseg", L.chr_crc32_segments_workspace_size(len(range_reg)))
        D.check(L.chr_crc32_segments(D.ptr(blob), _abi.aptr(rr), len(range_reg), D.ptr(wk), wk.numel(), _abi.aptr(raw),
                                     None, D.stream_ptr()), "chr_crc32_segments")
        where = {int(i): j for j, i in enumerate(sel_idx)}
        for (i, end), rv in zip(range_reg, raw):
            share[where[i]] ^= L.chr_crc32_shift(int(rv), int(plen[i]) - int(end))
    tot = np.zeros(nsel, dtype=np.uint32)
    for sh in _allgather(torch.from_numpy(share.view(np.int32).copy())):
        tot ^= sh.numpy().view(np.uint32)
    for j, i in enumerate(sel_idx):
        crc = L.chr_crc32_combine(0xFFFFFFFF, int(tot[j]), int(plen[i])) ^ 0xFFFFFFFF
        if crc != int(regions["payload_crc"][i]):
            from .exceptions import CorruptPayloadError

            raise CorruptPayloadError("payload checksum mismatch")

    # ---- decode the re-framed portions (e = 1/2 -> u_local exact)
    windows = torch.zeros(max(w_off, 1), dtype=torch.float64, device=dev)
    if mine:
        sblob = torch.cat([p.reshape(-1) for p in pieces] + [torch.zeros(16, dtype=torch.uint8, device=dev)])
        offs = np.asarray([r[0] for r in dec_rows], dtype=np.uint64)
        lens = np.asarray([r[1] for r in dec_rows], dtype=np.uint64)
        rr = np.stack([offs, offs + lens], axis=1).reshape(-1)
        crcs = np.zeros(len(dec_rows), dtype=np.uint32)
        wk = ws.get("crcseg", L.chr_crc32_segments_workspace_size(len(dec_rows)))
        D.check(L.chr_crc32_segments(D.ptr(sblob), _abi.aptr(rr), len(dec_rows), D.ptr(wk), wk.numel(), None,
                                     _abi.aptr(crcs), D.stream_ptr()), "chr_crc32_segments")
        tab = D.dec_table(offs, lens, [r[2] for r in dec_rows], [r[3] for r in dec_rows], [r[4] for r in dec_rows],
                          crcs)
        tab["out_offset"] = [r[5] for r in dec_rows]
        _, _, status = D.decode(sblob, tab, ws=ws, out=windows)
        if any(status):
            raise ParameterError(f"portion decode failed: {list(status)}")

    # ---- z-carries: all-gather every portion's last-plane u_local
    def plane_of(P):
        e = regions["extent"][P.reg]
        return int(e[0]) * int(e[1])

    def lorenzo(P):
        return int(regions["codec_id"][P.reg]) in (1, 2)

    sizes = [sum(plane_of(P) for P in ports_all[r] if lorenzo(P)) for r in range(world)]
    mine_last = [windows[win_off[pi] + (0 if P.first else plane_of(P)) + (P.pb - P.pa - 1) * plane_of(P):][: plane_of(P)]
                 for pi, P in enumerate(mine) if lorenzo(P)]
    packed = torch.cat(mine_last).to(torch.int64) if mine_last else torch.zeros(0, dtype=torch.int64, device=dev)
    lasts = _allgather_var(packed, sizes)
    last_of = {}  # (rank, region) -> int64 plane
    for r in range(world):
        o = 0
        for P in ports_all[r]:
            if lorenzo(P):
                last_of[(r, P.reg)] = lasts[r][o: o + plane_of(P)]
                o += plane_of(P)
    carries, c_off = [], []
    c_at = 0
    fin = []
    for pi, P in enumerate(mine):
        if not lorenzo(P):
            continue
        co = -1
        if not P.first:
            c = sum(last_of[(r, P.reg)] for r in range(rank) if (r, P.reg) in last_of)
            carries.append(c)
            co = c_at
            c_at += plane_of(P)
        e = regions["extent"][P.reg]
        fin.append((win_off[pi] + (0 if P.first else plane_of(P)), plane_of(P), P.pb - P.pa, co,
                    float(regions["error_bound"][P.reg])))
    if fin:
        cbuf = torch.cat(carries) if carries else torch.zeros(1, dtype=torch.int64, device=dev)
        cols = (np.asarray([x[0] for x in fin], dtype=np.uint64), np.asarray([x[1] for x in fin], dtype=np.int64),
                np.asarray([x[2] for x in fin], dtype=np.int64), np.asarray([x[3] for x in fin], dtype=np.int64),
                np.asarray([x[4] for x in fin], dtype=np.float64))  # kept alive across the call
        wk = ws.get("pfin", 64 * len(fin))
        D.check(L.chr_portion_finish(D.ptr(windows), *[_abi.aptr(c) for c in cols], len(fin), D.ptr(cbuf),
                                     D.ptr(wk), wk.numel(), D.stream_ptr()), "chr_portion_finish")
    for pi, bmo, vo, s0, n, ne in esc_fix:  # codec 2: escaped samples keep their f64 value
        if ne == 0:
            continue
        P = mine[pi]
        nb = ((s0 + n + 7) >> 3) - (s0 >> 3)
        bits = torch.stack([(blob[bmo: bmo + nb] >> b) & 1 for b in range(8)], dim=1).reshape(-1)
        bits = bits[(s0 & 7): (s0 & 7) + n].bool()
        vals = blob[vo: vo + 8 * ne].clone().view(torch.float64)
        dst = windows[win_off[pi] + (0 if P.first else plane_of(P)):][:n]
        dst[bits] = vals

    # ---- halo planes: all-gather of every non-final portion's last plane
    hsizes = [sum(plane_of(P) for P in ports_all[r] if not P.last) for r in range(world)]
    mine_top = [windows[win_off[pi] + (0 if P.first else plane_of(P)) + (P.pb - P.pa - 1) * plane_of(P):][: plane_of(P)]
                for pi, P in enumerate(mine) if not P.last]
    hp = torch.cat(mine_top) if mine_top else torch.zeros(0, dtype=torch.float64, device=dev)
    tops = _allgather_var(hp, hsizes)
    top_of = {}
    for r in range(world):
        o = 0
        for P in ports_all[r]:
            if not P.last:
                top_of[(r, P.reg)] = tops[r][o: o + plane_of(P)]
                o += plane_of(P)
    for pi, P in enumerate(mine):
        if not P.first:
            windows[win_off[pi]: win_off[pi] + plane_of(P)] = top_of[(rank - 1, P.reg)]

    # ---- marching cubes of each portion's cells (halo plane first)
    verts = torch.empty((0, 3), dtype=torch.float64, device=dev)
    tris = torch.empty((0, 3), dtype=torch.int32, device=dev)
    vedge = torch.empty(0, dtype=torch.int64, device=dev)
    nt = nv = []
    grids = []
    for pi, P in enumerate(mine):
        ex, ey, _ = (int(v) for v in regions["extent"][P.reg])
        oz = int(regions["origin"][P.reg][2])
        gz = P.pb - P.pa + (0 if P.first else 1)
        grids.append((pi, win_off[pi], (ex, ey, gz), P.pa - oz - (0 if P.first else 1)))
    keep = [g for g in grids if g[2][2] >= 2]  # a one-plane portion has no cells of its own
    if keep:
        org = np.stack([regions["origin"][mine[g[0]].reg].astype(np.float64) * np.asarray(spacing) for g in keep])
        mct = D.mc_table([g[1] for g in keep], [g[2] for g in keep], org, spacing)
        mct["zoff"] = [g[3] for g in keep]
        verts, tris, nt, nv, vedge = D.marching(windows, mct, k, ws=ws, edges=True)
    cnt_t = {g[0]: c for g, c in zip(keep, nt)}
    cnt_v = {g[0]: c for g, c in zip(keep, nv)}

    # drop halo-plane x/y vertices (first touched by the previous rank), count the rest
    vbase = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64) if keep else np.zeros(1, np.int64)
    drop = torch.zeros(verts.shape[0], dtype=torch.bool, device=dev)
    gi = {g[0]: j for j, g in enumerate(keep)}
    def prev_has_cells(P):
        for Q in ports_all[rank - 1]:
            if Q.reg == P.reg:
                return (Q.pb - Q.pa) + (0 if Q.first else 1) >= 2
        return False

    for pi, P in enumerate(mine):
        if P.first or pi not in gi or not prev_has_cells(P):
            continue
        j = gi[pi]
        e = vedge[vbase[j]: vbase[j + 1]]
        ex, ey = (int(v) for v in regions["extent"][P.reg][:2])
        drop[vbase[j]: vbase[j + 1]] = (e // 3 < ex * ey) & (e % 3 != 2)
    kept = torch.zeros(len(mine), dtype=torch.int64)
    for pi in range(len(mine)):
        if pi in gi:
            j = gi[pi]
            kept[pi] = int(cnt_v[pi]) - int(drop[vbase[j]: vbase[j + 1]].sum())
    # all-gather of (triangles, kept vertices) of every (selected region, rank)
    cnt = torch.zeros((nsel, 2), dtype=torch.int64)
    for pi, P in enumerate(mine):
        cnt[P.sel, 0] = int(cnt_t.get(pi, 0))
        cnt[P.sel, 1] = int(kept[pi])
    allc = torch.stack(_allgather(cnt))  # [world, nsel, 2]
    per_reg = allc.sum(dim=0)
    reg_base = torch.cumsum(per_reg, 0) - per_reg  # [nsel, 2] rows of each region
    rank_pre = torch.cumsum(allc, 0) - allc        # [world, nsel, 2] earlier ranks inside the region
    # global ids of this rank's kept vertices; export the top-plane x/y ones
    gid = torch.full((verts.shape[0],), -1, dtype=torch.int64, device=dev)
    exp_keys, exp_ids = [], []
    for pi, P in enumerate(mine):
        if pi not in gi:
            continue
        j = gi[pi]
        sl = slice(int(vbase[j]), int(vbase[j + 1]))
        d = drop[sl]
        b0 = int(reg_base[P.sel, 1] + rank_pre[rank, P.sel, 1])
        ids = torch.cumsum((~d).to(torch.int64), 0) - 1 + b0
        gid[sl] = torch.where(d, torch.full_like(ids, -1), ids)
        if not P.last:
            ex, ey, gz = (int(v) for v in keep[j][2])
            e = vedge[sl]
            top = (e // 3 >= (gz - 1) * ex * ey) & (e % 3 != 2) & ~d
            exp_keys.append(e[top] - (gz - 1) * ex * ey * 3)
            exp_ids.append(gid[sl][top])
    # exchange top-plane vertex ids (sizes first)
    my_exp = [(P, kk, ii) for P, kk, ii in zip([P for pi, P in enumerate(mine) if pi in gi and not P.last],
                                               exp_keys, exp_ids)]
    lens_local = torch.tensor([len(kk) for _, kk, _ in my_exp], dtype=torch.int64)
    nexp = torch.zeros(nsel, dtype=torch.int64)
    for (P, kk, _), n in zip(my_exp, lens_local):
        nexp[P.sel] = int(n)
    alln = torch.stack(_allgather(nexp))  # [world, nsel]
    esz = [int(alln[r].sum()) * 2 for r in range(world)]
    pack = torch.cat([torch.stack([kk, ii], 1).reshape(-1) for _, kk, ii in my_exp]) if my_exp else \
        torch.zeros(0, dtype=torch.int64, device=dev)
    allexp = _allgather_var(pack, esz)
    imp = {}
    for r in range(world):
        o = 0
        for s in range(nsel):
            n = int(alln[r, s])
            if n:
                kv = allexp[r][o: o + 2 * n].view(n, 2)
                imp[(r, s)] = (kv[:, 0], kv[:, 1])
                o += 2 * n
    # resolve the dropped (halo-plane) vertices from the previous rank's export
    for pi, P in enumerate(mine):
        if P.first or pi not in gi:
            continue
        j = gi[pi]
        sl = slice(int(vbase[j]), int(vbase[j + 1]))
        d = drop[sl]
        if not bool(d.any()):
            continue
        keys, ids = imp[(rank - 1, P.sel)]
        order = torch.argsort(keys)
        keys, ids = keys[order], ids[order]
        want = vedge[sl][d]
        pos = torch.searchsorted(keys, want)
        g = gid[sl]
        g[d] = ids[pos.clamp_max(max(len(ids) - 1, 0))]
        gid[sl] = g
    tris_g = gid[tris.reshape(-1).to(torch.int64)].reshape(-1, 3).to(torch.int32) if tris.numel() else tris
    verts_k = verts[~drop] if verts.numel() else verts
    tri_base = [int(reg_base[P.sel, 0] + rank_pre[rank, P.sel, 0]) for P in mine]
    vert_base = [int(reg_base[P.sel, 1] + rank_pre[rank, P.sel, 1]) for P in mine]
    return SlabMesh(verts_k, tris_g, [P.sel for P in mine], tri_base, vert_base, int(per_reg[:, 0].sum()),
                    int(per_reg[:, 1].sum()), [int(cnt_t.get(pi, 0)) for pi in range(len(mine))],
                    [int(kept[pi]) for pi in range(len(mine))])
