"""Device-resident CHR pipeline: the hot path as a user of the C-ABI sees it.

Every function takes / returns torch CUDA tensors and calls libchr.so
(include/chr.h) on the current torch stream.  The reference-shaped API
(``archive.build_chr`` / ``request`` / ``surface.marching_cubes`` ...) is
built on these; the benchmark times them directly.

    stats          blocking.decompose + bound distances  (chr_stats)
    plan           build_index + merge_regions + bounds  (chr_plan)
    compress       codec.compress per region + write_chr (chr_compress)
    decode         codec.decompress per selected region  (chr_decode_regions)
    marching       marching_cubes + merge_meshes         (chr_mc_count/emit)
"""

from __future__ import annotations

import ctypes
import math
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from ._abi import check, lib, ptr, stream_ptr
from .exceptions import NonFiniteSampleError, ParameterError

SAFETY_FACTOR = 1.0 - 2.0**-20  # bound.py:38
LOOSE_FRACTION = 0.01  # bound.py:42
DTYPE_TAGS = {"f32": 0, "f64": 1}  # volume.py:18
BLOCK_HEADER = 34  # codec.py:41
FILE_HEADER = 63  # chr_archive.py:50
REGION_FIXED = 85  # chr_archive.py:51


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return 0
    if t.dtype == torch.float64:
        return 1
    raise ParameterError(f"volume must be float32 or float64, got {t.dtype}")


def _cands_arr(cands) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(cands, dtype=np.float64).reshape(-1))
    if a.size < 1 or a.size > 64:
        raise ParameterError(f"need 1..64 candidates, got {a.size}")
    return a


def _np_ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def num_blocks(dims, bs) -> int:
    """chr_num_blocks (blocking.py:64-70: max(1, ceil((d - 1) / bs)) per axis), in Python:
    it runs before every pipeline call and the C round trip cost ~15 us."""
    bs = int(bs)
    if bs < 1:
        return 0
    n = 1
    for d in dims:
        d = int(d)
        n *= (d - 1 + bs - 1) // bs if d - 1 > 0 else 1
    return n


def stats(vol: torch.Tensor, dims, bs: int, cands) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-block (vmin, vmax, dmin) f64 [nblocks, 3] + first non-finite index (device)."""
    cands = _cands_arr(cands)
    nb = num_blocks(dims, bs)
    out = torch.empty((nb, 3), dtype=torch.float64, device=vol.device)
    bad = torch.empty(1, dtype=torch.int64, device=vol.device)  # (both small: the caching allocator serves them)
    check(lib().chr_stats(ptr(vol), _dtype_code(vol), *dims, bs, _np_ptr(cands), cands.size,
                          ptr(out), ptr(bad), stream_ptr()), "chr_stats")
    return out, bad


# host copies of decoded windows -> their device originals (request()):
# a window array handed back to marching_cubes is meshed from HBM directly
_HOST_WINDOWS: dict = {}


def register_host_windows(host: np.ndarray, dev: torch.Tensor) -> None:
    """Remember that read-only `host` is a D2H copy of f64 `dev` (same length)."""
    key = id(host)
    _HOST_WINDOWS[key] = (host.ctypes.data, host.size, dev)
    weakref.finalize(host, _HOST_WINDOWS.pop, key, None)


def host_window(a: np.ndarray) -> torch.Tensor | None:
    """The device f64 copy of `a` (x fastest) if `a` is a Fortran-order view
    into a registered host window buffer, else None."""
    root = a
    while isinstance(root.base, np.ndarray):
        root = root.base
    ent = _HOST_WINDOWS.get(id(root))
    if ent is None or ent[0] != root.ctypes.data or a.dtype != np.float64 or not a.flags.f_contiguous:
        return None
    off = (a.ctypes.data - ent[0]) // 8
    if off < 0 or off + a.size > ent[1]:
        return None
    return ent[2][off: off + a.size]


def value_range(vol: torch.Tensor) -> tuple[float, float, int]:
    """(min, max, first non-finite flat index or -1) of a device field
    (Volume.value_range + finite check, volume.py:54-78; chr_value_range)."""
    flat = vol.reshape(-1)
    lo_hi = (ctypes.c_double * 2)()
    bad = ctypes.c_int64(-1)
    work = _DEFAULT_WS.get("vrange", 64)
    check(lib().chr_value_range(ptr(flat), _dtype_code(flat), flat.numel(), ptr(work), work.numel(), lo_hi,
                                ctypes.byref(bad), stream_ptr()), "chr_value_range")
    return float(lo_hi[0]), float(lo_hi[1]), int(bad.value)


def plan(block_stats: np.ndarray, dims, bs, cands, vmin, vmax, loose_fraction=LOOSE_FRACTION,
         safety_factor=SAFETY_FACTOR):
    """Regions (numpy array of chr_region_t, ``_abi.REGION_DT``) from host block stats."""
    cands = _cands_arr(cands)
    bsn = np.ascontiguousarray(block_stats, dtype=np.float64)
    nb = bsn.shape[0]
    regs = np.empty(nb, dtype=_abi.REGION_DT)  # chr_plan zero-fills every record it writes
    nreg = ctypes.c_int64(0)
    check(lib().chr_plan(_np_ptr(bsn), *dims, bs, _np_ptr(cands), cands.size, float(vmin), float(vmax),
                         float(loose_fraction), float(safety_factor), _abi.aptr(regs), ctypes.byref(nreg)),
          "chr_plan")
    return regs[: nreg.value].copy()


@dataclass
class Compressed:
    """Output of :func:`compress`: bytes on the device + the region table."""

    blob: torch.Tensor  # uint8, first `nbytes` valid
    nbytes: int
    regions: np.ndarray  # _abi.REGION_DT (codec/offset/crc filled)
    source_dtype: str
    extra: dict = field(default_factory=dict)


class Workspaces:
    """Reusable device scratch (grows on demand) so steady-state calls do
    not hit the caching allocator."""

    def __init__(self):
        self._bufs: dict[str, torch.Tensor] = {}

    def host(self, name: str, n: int, dtype) -> np.ndarray:
        a = self._bufs.get("host:" + name)
        if a is None or a.size < n or a.dtype != dtype:
            a = np.zeros(max(int(n), 1), dtype=dtype)
            self._bufs["host:" + name] = a
        return a

    def pinned(self, name: str, numel: int, dtype=torch.float64) -> torch.Tensor:
        t = self._bufs.get("pinned:" + name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(max(int(numel), 64), dtype=dtype, pin_memory=True)
            self._bufs["pinned:" + name] = t
        return t[:numel]

    def get(self, name: str, nbytes: int, dtype=torch.uint8) -> torch.Tensor:
        elem = dtype.itemsize
        n = max(1, -(-int(nbytes) // elem))
        t = self._bufs.get(name)
        if t is None or t.numel() < n or t.dtype != dtype or t.device != _abi.device():
            # drop the old buffer first: at c5 sizes old + new may not fit together
            self._bufs.pop(name, None)
            del t
            t = torch.empty(max(n, 64), dtype=dtype, device=_abi.device())
            self._bufs[name] = t
        return t

    def clear(self) -> None:
        """Drop every buffer (device, pinned and host)."""
        self._bufs.clear()


class _ThreadWorkspaces:
    """The default workspaces, one set per host thread: the reference runs
    request / decompress under a ThreadPoolExecutor (chr_archive.py:253-255),
    and a shared scratch buffer would let one thread's decode overwrite
    another's (the C library's own host state is thread-local too)."""

    def __init__(self):
        self._tls = threading.local()

    def _get(self) -> Workspaces:
        ws = getattr(self._tls, "ws", None)
        if ws is None:
            ws = self._tls.ws = Workspaces()
        return ws

    def __getattr__(self, name):
        return getattr(self._get(), name)

    def release(self) -> None:
        """Drop this thread's default workspaces."""
        ws = getattr(self._tls, "ws", None)
        if ws is not None:
            ws.clear()


def release_workspaces() -> None:
    """Free the calling thread's default scratch and the caching allocator's
    unused blocks (between full-size runs that each need most of the HBM)."""
    import gc

    _DEFAULT_WS.release()
    gc.collect()
    if torch.cuda.is_available():
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


_DEFAULT_WS = _ThreadWorkspaces()


BOUND_MODES = {"strict_vertices": 0, "paper_edges": 1}


def compress(vol: torch.Tensor, dims, regions, *, source_dtype="f32", write_file=True, spacing=(1.0, 1.0, 1.0),
             bs=0, vrange=(0.0, 0.0), cands=(0.0,), ws: Workspaces | None = None,
             out: torch.Tensor | None = None, bound_mode: str = "strict_vertices",
             accuracy: float = 1.0) -> Compressed:
    """Run chr_compress on `regions`; returns the device bytes."""
    ws = ws or _DEFAULT_WS
    L = lib()
    regions = np.ascontiguousarray(regions, dtype=_abi.REGION_DT)
    nreg = len(regions)
    rp = _abi.aptr(regions)
    cands = _cands_arr(cands)
    m = cands.size
    wsz = L.chr_compress_workspace_size(rp, nreg)
    if wsz == 0:
        raise ParameterError("invalid regions for compress")
    work = ws.get("compress", wsz)
    cap = int(L.chr_compress_capacity(rp, nreg, m, DTYPE_TAGS[source_dtype]))
    if out is None or out.numel() < cap:
        out = ws.get("compress_out", cap)
    nbytes = ctypes.c_uint64(0)
    sp = (ctypes.c_double * 3)(*[float(s) for s in spacing])
    check(L.chr_compress2(ptr(vol), _dtype_code(vol), DTYPE_TAGS[source_dtype], *dims, sp, int(bs),
                          float(vrange[0]), float(vrange[1]), _np_ptr(cands), m, rp, nreg,
                          1 if write_file else 0, BOUND_MODES[bound_mode], float(accuracy), ptr(work),
                          work.numel(), ptr(out), out.numel(), ctypes.byref(nbytes), stream_ptr()), "chr_compress")
    return Compressed(out, int(nbytes.value), regions, source_dtype)


def select_distances(vol: torch.Tensor, dims, windows, ks, accuracy: float, bound_mode: str) -> np.ndarray:
    """n-th smallest distance D(window, k) per pair (bound.py:117-147),
    -1.0 where D is empty (paper_edges, no straddling edge)."""
    npairs = len(windows)
    val = np.zeros(max(npairs, 1), np.float64)
    if npairs:
        L = lib()
        w = np.ascontiguousarray(windows, dtype=np.int32).reshape(npairs, 6)
        karr = np.ascontiguousarray(ks, dtype=np.float64)
        work = _DEFAULT_WS.get("select", L.chr_select_workspace_size(npairs))
        check(L.chr_select_distances(ptr(vol), _dtype_code(vol), *dims, _np_ptr(w), _np_ptr(karr), npairs,
                                     float(accuracy), BOUND_MODES[bound_mode], ptr(work), work.numel(),
                                     _np_ptr(val), None, None, stream_ptr()), "chr_select_distances")
    return val[:npairs]


def select_bounds(vol: torch.Tensor, dims, bs, regions: np.ndarray, block_stats: np.ndarray, cands, accuracy: float,
                  bound_mode: str, safety_factor: float, loose: float) -> np.ndarray:
    """bound.region_bound (bound.py:150-219) for accuracy < 1 / paper_edges:
    n-th smallest distance of every served (region, candidate) pair on the
    device (chr_select_distances), then per region the minimum spec over its
    served candidates (a zero distance forces lossless), the loose bound when
    nothing is served or no edge straddles, and the cap below every unserved
    candidate's margin (min |s - k|, from the region's block extrema: an
    unserved k lies outside every one of its blocks' ranges).  Returns the
    float64 bound per region."""
    cands = [float(k) for k in cands]
    nx, ny, nz = dims
    nb3 = [max(1, -(-(d - 1) // bs)) for d in dims]
    st = np.asarray(block_stats, dtype=np.float64).reshape(nb3[2], nb3[1], nb3[0], -1)
    win, kk, owner = [], [], []
    for r in range(len(regions)):
        mask = int(regions["mask"][r])
        for ci, k in enumerate(cands):
            if (mask >> ci) & 1:
                win.append(list(regions["origin"][r]) + list(regions["extent"][r]))
                kk.append(k)
                owner.append(r)
    npairs = len(win)
    val = select_distances(vol, dims, win, kk, accuracy, bound_mode)
    out = np.empty(len(regions), np.float64)
    pi = 0
    for r in range(len(regions)):
        mask = int(regions["mask"][r])
        best = None
        lossless = False
        while pi < npairs and owner[pi] == r:
            v = float(val[pi])
            pi += 1
            if lossless:
                continue
            spec = float(loose) if v < 0 else (0.0 if v == 0.0 else v * safety_factor)
            if best is None or spec < best:
                best = spec
            if v == 0.0:
                lossless = True
        if best is None:
            best = float(loose)
        if not lossless:
            lo, hi = regions["lo"][r], regions["hi"][r]
            sub = st[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
            bmin, bmax = sub[..., 0].ravel(), sub[..., 1].ravel()
            for ci, k in enumerate(cands):
                if (mask >> ci) & 1:
                    continue
                d = np.where(k < bmin, bmin - k, k - bmax)  # fl(|s - k|) at the nearer extreme
                margin = float(d.min()) * safety_factor
                if margin < best:
                    best = margin
        out[r] = best
    return out


def build_archive(vol: torch.Tensor, dims, cands, bs, *, spacing=(1.0, 1.0, 1.0), source_dtype="f32",
                  loose_fraction=LOOSE_FRACTION, safety_factor=SAFETY_FACTOR, vrange=None,
                  out_of_range="error", ws: Workspaces | None = None, on_warn=None, accuracy: float = 1.0,
                  bound_mode: str = "strict_vertices") -> Compressed:
    """stats -> plan -> compress: a complete .chr file on the device
    (chr_archive.build_chr, strict bound at accuracy 1)."""
    ws = ws or _DEFAULT_WS
    cands = _cands_arr(cands)
    if any(b <= a for a, b in zip(cands[:-1], cands[1:])) or not np.isfinite(cands).all():
        raise ParameterError(f"candidates must be finite and strictly increasing, got {list(cands)}")
    bst, bad = stats(vol, dims, bs, cands)
    host = ws.pinned("block_stats", bst.numel() + 1)
    L = lib()  # kernel copies into pinned memory: never queued behind a caller's bulk DMA
    check(L.chr_copy(host.data_ptr(), bst.data_ptr(), 8 * bst.numel(), stream_ptr()), "chr_copy")
    check(L.chr_copy(host.data_ptr() + 8 * bst.numel(), bad.data_ptr(), 8, stream_ptr()), "chr_copy")
    torch.cuda.current_stream().synchronize()
    hs = host.numpy()
    badidx = int(hs[-1:].view(np.int64)[0])
    if badidx >= 0:
        value = float(vol.reshape(-1)[badidx].item())
        raise NonFiniteSampleError(badidx, value)
    bstats = hs[:-1].reshape(-1, 3)
    if vrange is None:
        vrange = (float(bstats[:, 0].min()), float(bstats[:, 1].max()))
    vmin, vmax = vrange
    outside = [float(k) for k in cands if not vmin <= k <= vmax]
    if outside:
        msg = f"candidates outside the volume's value range [{vmin}, {vmax}]: {outside}"
        if out_of_range == "error":
            raise ParameterError(msg)
        if on_warn:
            on_warn(msg)
    if not loose_fraction > 0.0:
        raise ParameterError(f"loose_fraction must be positive, got {loose_fraction}")
    regions = plan(bstats, dims, bs, cands, vmin, vmax, loose_fraction, safety_factor)
    if accuracy != 1.0 or bound_mode != "strict_vertices":
        loose = loose_fraction * (vmax - vmin)
        regions["error_bound"] = select_bounds(vol, dims, bs, regions, bstats, cands, accuracy, bound_mode,
                                               safety_factor, loose)
    res = compress(vol, dims, regions, source_dtype=source_dtype, write_file=True, spacing=spacing, bs=bs,
                   vrange=(vmin, vmax), cands=cands, ws=ws, bound_mode=bound_mode, accuracy=accuracy)
    res.extra.update(block_stats=bstats, vrange=(vmin, vmax), cands=tuple(float(k) for k in cands))
    return res


def request_tables(regions: np.ndarray, k_index: int, spacing=(1.0, 1.0, 1.0)):
    """(decode table, marching table, selected region indices, total window
    samples) for request(k) over a ``REGION_DT`` table, built in C
    (chr_request_tables); ``k_index`` < 0 selects every region."""
    regions = np.ascontiguousarray(regions, dtype=_abi.REGION_DT)
    n = len(regions)
    dec = np.empty(n, dtype=_abi.DEC_DT)
    mct = np.empty(n, dtype=_abi.MCGRID_DT)
    sel = np.empty(n, dtype=np.int64)
    total = ctypes.c_uint64(0)
    sp = (ctypes.c_double * 3)(*[float(v) for v in spacing])
    m = lib().chr_request_tables(_abi.aptr(regions), n, int(k_index), sp, _abi.aptr(dec), _abi.aptr(mct),
                                 _np_ptr(sel), ctypes.byref(total))
    if m < 0:
        raise ParameterError("chr_request_tables: bad arguments")
    return dec[:m], mct[:m], sel[:m], int(total.value)


@dataclass
class PipelineResult:
    """chr_pipeline's outputs; the tensors are views into ``ws`` buffers
    (valid until the next pipeline call with the same workspaces)."""
    archive: torch.Tensor   # uint8 .chr file
    regions: np.ndarray     # REGION_DT (codec / offsets / CRCs filled)
    windows: torch.Tensor   # f64 selected windows, back to back
    verts: torch.Tensor     # (nv, 3) f64 world coordinates
    tris: torch.Tensor      # (nt, 3) int32
    n_selected: int
    vrange: tuple


def pipeline(vol: torch.Tensor, dims, cands, bs, *, loose_fraction=LOOSE_FRACTION, safety_factor=SAFETY_FACTOR,
             k_index: int = 0, spacing=(1.0, 1.0, 1.0), source_dtype="f32", ws: Workspaces | None = None,
             stage_events=None, after_compress=None) -> PipelineResult:
    """build_archive + request(candidate k_index) + marching cubes in one
    C call (chr_pipeline): the same bytes, windows and mesh as the separate
    calls, without the host round trips between them.  Strict bound at
    accuracy 1; candidates must lie inside the volume's range.
    ``after_compress(archive_view)`` runs as soon as the archive exists
    (the mesh is still being computed)."""
    ws = ws or _DEFAULT_WS
    L = lib()
    cands = _cands_arr(cands)
    sp = (ctypes.c_double * 3)(*[float(v) for v in spacing])
    nb = num_blocks(dims, bs)
    regions = ws.host("pipe_regions", nb, _abi.REGION_DT)
    res = np.zeros(1, dtype=_abi.PIPE_RES_DT)
    need = dict(ws=1 << 20, arch=1 << 20, tri=1 << 16, vert=1 << 16)
    for key, name in (("ws", "pipe_ws"), ("arch", "pipe_archive")):
        b = ws._bufs.get(name)
        if b is not None:
            need[key] = max(need[key], b.numel())
    for key, name, el in (("tri", "pipe_tris", 12), ("vert", "pipe_verts", 24)):
        b = ws._bufs.get(name)
        if b is not None:
            need[key] = max(need[key], b.numel() * b.element_size() // el)
    cb = _abi.AFTER_COMPRESS(0)  # NULL
    if after_compress is not None:
        def _cb(nbytes, _user):
            after_compress(ws._bufs["pipe_archive"][: int(nbytes)])
        cb = _abi.AFTER_COMPRESS(_cb)
    evs = None
    if stage_events is not None:
        for e in stage_events:
            if not e.cuda_event:  # torch creates the CUDA event lazily, on its first record
                e.record()
        evs = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(e.cuda_event) for e in stage_events])
    for _ in range(6):
        work = ws.get("pipe_ws", need["ws"])
        arch = ws.get("pipe_archive", need["arch"])
        verts = ws.get("pipe_verts", 24 * need["vert"], torch.float64)
        tris = ws.get("pipe_tris", 12 * need["tri"], torch.int32)
        rc = L.chr_pipeline(ptr(vol), _dtype_code(vol), DTYPE_TAGS[source_dtype], *dims, sp, int(bs), _np_ptr(cands),
                            cands.size, float(loose_fraction), float(safety_factor), int(k_index), ptr(work),
                            work.numel(), ptr(arch), arch.numel(), ptr(verts), verts.numel() // 3, ptr(tris),
                            tris.numel() // 3, _abi.aptr(regions), evs, cb, None, _abi.aptr(res), stream_ptr())
        r = res[0]
        if rc == _abi.CHR_E_WORKSPACE:
            need["ws"] = max(need["ws"], int(r["ws_needed"]))
            need["arch"] = max(need["arch"], int(r["archive_needed"]))
            need["tri"] = max(need["tri"], int(r["n_tri"]))
            need["vert"] = max(need["vert"], int(r["n_vert"]))
            continue
        if rc == _abi.CHR_E_NONFINITE:
            i = int(r["first_nonfinite"])
            raise NonFiniteSampleError(i, float(vol.reshape(-1)[i].item()))
        check(rc, "chr_pipeline")
        nreg, nsel = int(r["n_regions"]), int(r["n_selected"])
        nt, nv = int(r["n_tri"]), int(r["n_vert"])
        wo, tot = int(r["windows_offset"]), int(r["window_samples"])
        windows = work[wo: wo + 8 * tot].view(torch.float64)
        return PipelineResult(arch[: int(r["archive_nbytes"])], regions[:nreg].copy(), windows,
                              verts[: 3 * nv].view(nv, 3), tris[: 3 * nt].view(nt, 3), nsel,
                              (float(r["vmin"]), float(r["vmax"])))
    raise ParameterError("chr_pipeline: workspace negotiation did not converge")


def dec_table(payload_offset, payload_nbytes, codec, dims, e, crc) -> np.ndarray:
    """Vectorised chr_dec_region_t table (windows laid out back to back)."""
    n = len(payload_offset)
    t = np.zeros(n, dtype=_abi.DEC_DT)
    t["payload_offset"] = payload_offset
    t["payload_nbytes"] = payload_nbytes
    t["codec_id"] = codec
    t["dims"] = np.asarray(dims, dtype=np.int32).reshape(n, 3)
    t["error_bound"] = e
    t["crc"] = np.asarray(crc, dtype=np.uint64) & 0xFFFFFFFF
    sizes = np.prod(t["dims"].astype(np.int64), axis=1)
    t["out_offset"] = np.concatenate([[0], np.cumsum(sizes)[:-1]]) if n else []
    return t


def decode(blob: torch.Tensor, sel, ws: Workspaces | None = None, out: torch.Tensor | None = None,
           iso: float | None = None):
    """Decode CompressedBlocks of `blob` (device uint8).

    ``sel``: a ``_abi.DEC_DT`` table (see :func:`dec_table`) or a list of
    (payload_offset, payload_nbytes, codec_id, (ex,ey,ez), e, crc).
    Returns (f64 device tensor of all windows concatenated, element offsets,
    per-region status codes) -- the last two as numpy arrays.  With ``iso`` the decoder also writes every
    window's inside mask (v >= iso) into ``ws`` ("decode_mask"), which
    :func:`marching` takes as ``masks`` (fused request + extract)."""
    ws = ws or _DEFAULT_WS
    L = lib()
    if not isinstance(sel, np.ndarray):
        cols = list(zip(*sel)) if sel else [[], [], [], [], [], []]
        sel = dec_table(*[np.asarray(c) for c in cols]) if sel else np.zeros(0, dtype=_abi.DEC_DT)
    n = len(sel)
    total = int((np.prod(sel["dims"].astype(np.int64), axis=1)).sum()) if n else 0
    if out is None or out.numel() < total:
        out = ws.get("decode_out", 8 * max(total, 1), torch.float64)
    status = np.zeros(max(n, 1), dtype=np.int32)
    if n:
        sp = _abi.aptr(sel)
        wsz = L.chr_decode_workspace_size(sp, n)
        work = ws.get("decode", wsz)
        if iso is None:
            rc = L.chr_decode_regions(ptr(blob), sp, n, ptr(out), ptr(work), work.numel(), _abi.aptr(status),
                                      stream_ptr())
        else:
            dims = np.ascontiguousarray(sel["dims"], dtype=np.int32)
            mw = int(L.chr_mask_words(_np_ptr(dims), n))
            mask = ws.get("decode_mask", 4 * (mw + 8), torch.int32)
            rc = L.chr_decode_regions_mask(ptr(blob), sp, n, ptr(out), ptr(work), work.numel(),
                                           _abi.aptr(status), float(iso), ptr(mask), stream_ptr())
        if rc not in (_abi.CHR_OK, _abi.CHR_E_CORRUPT, _abi.CHR_E_UNSUPPORTED_CODEC):
            check(rc, "chr_decode_regions")
    # the windows only (the workspace may be far larger: a caller copying the
    # result to the host must not drag the whole buffer along)
    # offsets and status as numpy arrays (a Python list of ints costs ~0.1 us per region)
    offs = sel["out_offset"].astype(np.int64) if n else np.zeros(0, np.int64)
    return out[:total], offs, status[:n]


def mc_table(grid_offset, dims, origin, spacing) -> np.ndarray:
    n = len(grid_offset)
    t = np.zeros(n, dtype=_abi.MCGRID_DT)
    t["grid_offset"] = grid_offset
    t["dims"] = np.asarray(dims, dtype=np.int32).reshape(n, 3)
    t["origin"] = np.asarray(origin, dtype=np.float64).reshape(n, 3)
    t["spacing"] = np.asarray(spacing, dtype=np.float64).reshape(-1, 3)
    return t


def marching(grids: torch.Tensor, descs, k: float, ws: Workspaces | None = None, reuse_outputs: bool = False,
             masks: torch.Tensor | None = None, edges: bool = False):
    """Marching cubes over several f64 windows of `grids`, merged.

    ``descs``: a ``_abi.MCGRID_DT`` table (:func:`mc_table`) or a list of
    (element_offset, (nx,ny,nz), origin3, spacing3).
    Returns (verts f64 [nv,3], tris int32 [nt,3], ntri per grid, nvert per grid)
    (+ the int64 canonical edge of every vertex with ``edges=True``,
    chr_mc_emit_edges: grid-local ((z * ny + y) * nx + x) * 3 + axis)."""
    ws = ws or _DEFAULT_WS
    L = lib()
    dev = _abi.device()
    if not isinstance(descs, np.ndarray):
        if not descs:
            descs = np.zeros(0, dtype=_abi.MCGRID_DT)
        else:
            off, dims, org, spc = zip(*descs)
            descs = mc_table(off, dims, org, spc)
    n = len(descs)
    if n == 0:
        empty = (torch.empty((0, 3), dtype=torch.float64, device=dev),
                 torch.empty((0, 3), dtype=torch.int32, device=dev), [], [])
        return empty + (torch.empty(0, dtype=torch.int64, device=dev),) if edges else empty
    gp = _abi.aptr(descs)
    wsz = L.chr_mc_workspace_size(gp, n)
    work = ws.get("mc", wsz)
    ntri = np.zeros(n, dtype=np.int64)
    nvert = np.zeros(n, dtype=np.int64)
    tt = ctypes.c_int64(0)
    tv = ctypes.c_int64(0)
    if masks is None:
        check(L.chr_mc_count(ptr(grids), gp, n, float(k), ptr(work), work.numel(), _abi.aptr(ntri),
                             _abi.aptr(nvert), ctypes.byref(tt), ctypes.byref(tv), stream_ptr()), "chr_mc_count")
    else:  # inside masks from decode(..., iso=k) of the same windows, same order
        check(L.chr_mc_count_masked(ptr(grids), gp, n, float(k), ptr(masks), ptr(work), work.numel(),
                                    _abi.aptr(ntri), _abi.aptr(nvert), ctypes.byref(tt), ctypes.byref(tv),
                                    stream_ptr()), "chr_mc_count_masked")
    if reuse_outputs:  # outputs in the workspace: valid until the next call with this workspace
        verts = ws.get("mc_verts", 24 * tv.value, dtype=torch.float64)[: tv.value * 3].view(tv.value, 3)
        tris = ws.get("mc_tris", 12 * tt.value, dtype=torch.int32)[: tt.value * 3].view(tt.value, 3)
    else:
        verts = torch.empty((tv.value, 3), dtype=torch.float64, device=dev)
        tris = torch.empty((tt.value, 3), dtype=torch.int32, device=dev)
    if edges:
        vedge = torch.empty(tv.value, dtype=torch.int64, device=dev)
        check(L.chr_mc_emit_edges(ptr(grids), gp, n, float(k), ptr(work), work.numel(), ptr(verts), ptr(tris),
                                  ptr(vedge), stream_ptr()), "chr_mc_emit_edges")
        return verts, tris, ntri.tolist(), nvert.tolist(), vedge
    if masks is None:
        check(L.chr_mc_emit(ptr(grids), gp, n, float(k), ptr(work), work.numel(), ptr(verts), ptr(tris),
                            stream_ptr()), "chr_mc_emit")
    else:
        check(L.chr_mc_emit_masked(ptr(grids), gp, n, float(k), ptr(masks), ptr(work), work.numel(), ptr(verts),
                                   ptr(tris), stream_ptr()), "chr_mc_emit_masked")
    return verts, tris, ntri.tolist(), nvert.tolist()


def case_codes(grid: torch.Tensor, dims, k: float, binary: bool = True) -> torch.Tensor:
    nx, ny, nz = dims
    codes = torch.empty((nx - 1) * (ny - 1) * (nz - 1), dtype=torch.uint8, device=grid.device)
    check(lib().chr_case_codes(ptr(grid), nx, ny, nz, float(k), 1 if binary else 0, ptr(codes), stream_ptr()),
          "chr_case_codes")
    return codes


def stitch(windows: torch.Tensor, table: np.ndarray, dims, bs: int, fill: float = float("nan"),
           out: torch.Tensor | None = None) -> torch.Tensor:
    """chr_archive.stitch (chr_archive.py:277-294) on the device: f64
    windows (``table``: ``_abi.STITCH_DT``) -> flat f64 volume, x fastest,
    every sample written by its owner (lowest (z, y, x) origin)."""
    nx, ny, nz = dims
    n = nx * ny * nz
    if out is None:
        out = torch.full((n,), fill, dtype=torch.float64, device=_abi.device())
    else:
        out[:n].fill_(fill)
    L = lib()
    t = np.ascontiguousarray(table, dtype=_abi.STITCH_DT)
    if t.size:
        work = _DEFAULT_WS.get("stitch", L.chr_stitch_workspace_size(t.size, nx, ny, nz, int(bs)))
        check(L.chr_stitch(ptr(windows), _abi.aptr(t), t.size, nx, ny, nz, int(bs), ptr(work), work.numel(),
                           ptr(out), stream_ptr()), "chr_stitch")
    return out


def topology_compare(a: torch.Tensor, b: torch.Tensor, dims, k: float) -> tuple[int, int]:
    """Cells whose binary case codes differ at k (isosurf.verify_topology,
    isosurf.py:91-114): (count, smallest differing cell index or -1)."""
    nx, ny, nz = dims
    L = lib()
    work = _DEFAULT_WS.get("topo", 16)
    nd, first = ctypes.c_uint64(0), ctypes.c_int64(-1)
    check(L.chr_topology_compare(ptr(a), _dtype_code(a), ptr(b), _dtype_code(b), nx, ny, nz, float(k), ptr(work),
                                 work.numel(), ctypes.byref(nd), ctypes.byref(first), stream_ptr()),
          "chr_topology_compare")
    return int(nd.value), int(first.value)


@dataclass
class FileTable:
    """read_chr's parse of a device-resident .chr file (chr_read_header +
    chr_read_archive): header fields, candidates, and the region table as
    ``_abi.TABLE_ENTRY_DT`` (``entries["region"]`` is a ``REGION_DT`` table
    the decode / marching entry points take directly)."""
    info: np.ndarray
    candidates: np.ndarray
    entries: np.ndarray

    @property
    def regions(self) -> np.ndarray:
        return self.entries["region"]


def read_table(file_dev: torch.Tensor, nbytes: int) -> FileTable:
    """Validate + parse a .chr file already in HBM.  No exception is raised
    here: ``info["error"]``, the stored/actual CRCs and ``entries["status"]``
    carry the outcome so the caller can raise in the reference's order."""
    L = lib()
    info = np.zeros(1, dtype=_abi.FILE_INFO_DT)
    check(L.chr_read_header(ptr(file_dev), int(nbytes), _abi.aptr(info), stream_ptr()), "chr_read_header")
    err = int(info["error"][0])
    if err in (_abi.READ_TOO_SHORT, _abi.READ_BAD_MAGIC):
        return FileTable(info, np.zeros(0), np.zeros(0, dtype=_abi.TABLE_ENTRY_DT))
    nreg = int(info["n_regions"][0]) if err == 0 else 0
    m = int(info["m"][0])
    cands = np.zeros(m if 67 + 8 * m <= nbytes else 0, dtype=np.float64)
    entries = np.zeros(nreg, dtype=_abi.TABLE_ENTRY_DT)
    work = _DEFAULT_WS.get("read", L.chr_read_workspace_size(int(nbytes), nreg))
    if err:
        info["n_regions"] = 0
    check(L.chr_read_archive(ptr(file_dev), int(nbytes), _abi.aptr(info), _np_ptr(cands) if cands.size else None,
                             _abi.aptr(entries), ptr(work), work.numel(), stream_ptr()), "chr_read_archive")
    return FileTable(info, cands, entries)


def crc32(buf: torch.Tensor, nbytes: int | None = None) -> int:
    n = buf.numel() if nbytes is None else int(nbytes)
    L = lib()
    work = _DEFAULT_WS.get("crc", L.chr_crc32_workspace_size(n))
    out = ctypes.c_uint32(0)
    check(L.chr_crc32(ptr(buf), n, ptr(work), work.numel(), ctypes.byref(out), stream_ptr()), "chr_crc32")
    return int(out.value)


def min_abs_distance(flat: torch.Tensor, k: float) -> float:
    L = lib()
    work = _DEFAULT_WS.get("minabs", 256)
    out = ctypes.c_double(0.0)
    check(L.chr_min_abs_distance(ptr(flat), flat.numel(), float(k), ctypes.byref(out), ptr(work), work.numel(),
                                 stream_ptr()), "chr_min_abs_distance")
    return float(out.value)


def lorenzo_encode(flat: torch.Tensor, nx, ny, nz, e):
    q = torch.empty(nx * ny * nz, dtype=torch.int64, device=flat.device)
    esc = torch.empty(nx * ny * nz, dtype=torch.uint8, device=flat.device)
    check(lib().chr_lorenzo_encode(ptr(flat), nx, ny, nz, float(e), ptr(q), ptr(esc), stream_ptr()),
          "chr_lorenzo_encode")
    return q, esc


def rle_varint_encode(q: torch.Tensor) -> torch.Tensor:
    """kernels.rle_varint_encode (kernels.py:292-296): int64 quanta -> uint8
    token stream on the device (|q| <= 2^30, as every valid stream)."""
    q = q.to(device=_abi.device(), dtype=torch.int64).contiguous()
    n = q.numel()
    L = lib()
    out = torch.empty(5 * n + 16, dtype=torch.uint8, device=q.device)
    work = _DEFAULT_WS.get("rle", L.chr_rle_encode_workspace_size(n))
    nb = ctypes.c_uint64(0)
    check(L.chr_rle_encode(ptr(q), n, ptr(out), out.numel(), ptr(work), work.numel(), ctypes.byref(nb), stream_ptr()),
          "chr_rle_encode")
    return out[: nb.value]


def rle_varint_decode(buf: torch.Tensor, n: int) -> torch.Tensor:
    """kernels.rle_varint_decode (kernels.py:407-411): token stream -> int64
    quanta.  Decoded as a codec-1 stream of a (1,n,1) window with e = 1/2,
    whose reconstruction is the 1-D prefix u of q (exact in f64 for |u| < 2^53);
    q = diff(u).  Malformed streams raise ValueError with the reference's
    reasons (truncated, varint too long, missing/invalid run, trailing, count)."""
    buf = buf.to(device=_abi.device(), dtype=torch.uint8).contiguous()
    if n == 0:
        if buf.numel():
            raise ValueError("trailing bytes after the last token")
        return torch.zeros(0, dtype=torch.int64, device=buf.device)
    staging = torch.zeros(buf.numel() + 16, dtype=torch.uint8, device=buf.device)
    staging[: buf.numel()] = buf
    crc = crc32(staging, buf.numel()) if buf.numel() else 0
    u, _, status = decode(staging, [(0, buf.numel(), 1, (1, n, 1), 0.5, crc)])  # 1-D prefix along y
    if status[0]:
        raise ValueError(_abi.DEC_MESSAGES.get(int(status[0]), "corrupt token stream"))
    u = u[:n].to(torch.int64)
    return torch.diff(u, prepend=torch.zeros(1, dtype=torch.int64, device=u.device))


def lorenzo_decode(q: torch.Tensor, escaped: torch.Tensor, escape_values: torch.Tensor, e: float, nx, ny, nz):
    """kernels.lorenzo_decode (kernels.py:182-186): u = 3D inclusive prefix of
    q, recon = u * 2e, escapes overwritten in raster order.  Runs the archive
    decoder on the device: q -> token stream (rle_varint_encode) -> codec-1
    block of dims (nx, ny, nz)."""
    n = nx * ny * nz
    tok = rle_varint_encode(q)
    staging = torch.zeros(tok.numel() + 16, dtype=torch.uint8, device=tok.device)
    staging[: tok.numel()] = tok
    crc = crc32(staging, tok.numel()) if tok.numel() else 0
    recon, _, status = decode(staging, [(0, tok.numel(), 1, (nx, ny, nz), float(e), crc)])
    if status[0]:
        raise ValueError(_abi.DEC_MESSAGES.get(int(status[0]), "corrupt token stream"))
    recon = recon[:n].clone()
    esc = escaped.to(device=recon.device).reshape(-1).bool()
    if esc.any():
        recon[esc] = escape_values.to(device=recon.device, dtype=torch.float64).reshape(-1)
    return recon


def region_records(regions) -> list[dict]:
    """Plain-Python view of a chr_region_t table."""
    regions = np.asarray(regions)
    cols = {f: regions[f].tolist() for f in regions.dtype.names}
    out = []
    for i in range(len(regions)):
        out.append(dict(
            id=i, lo=tuple(cols["lo"][i]), hi=tuple(cols["hi"][i]), origin=tuple(cols["origin"][i]),
            extent=tuple(cols["extent"][i]), mask=cols["mask"][i], e=cols["error_bound"][i],
            codec=cols["codec_id"][i], crc=cols["payload_crc"][i], block_offset=cols["block_offset"][i],
            block_nbytes=cols["block_nbytes"][i], nesc=cols["n_escaped"][i],
        ))
    return out


def header_table_nbytes(m: int, nreg: int) -> int:
    return FILE_HEADER + 4 + 8 * m + 4 + nreg * (REGION_FIXED + (m + 7) // 8)


def ceil_div(a, b):
    return -(-a // b)


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("annotations", "ctypes", "math")]
