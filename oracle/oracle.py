"""CPU oracle for the CHR hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module,
and only as the checker or the timed CPU baseline.  The product package
``paper_2408_05462_b200`` never imports it.

This is a restatement of the reference ``isochr`` package's algorithm for
the path named by BASELINE.json ``north_star`` (paths below are relative to
``/root/reference/pkg/src/isochr/``):

* volume validation + value range       volume.py:54-78
* block decomposition + extrema         blocking.py:64-111
* span index                            blocking.py:114-127
* greedy region merge                   blocking.py:130-193  (C: or_merge_regions)
* region bound (strict / paper_edges,   bound.py:68-83, 117-219, chr_archive.py:168
  any accuracy)
* codec compress / decompress           codec.py:91-229
* archive build / request / stitch      chr_archive.py:132-294
* archive serialisation                 chr_archive.py:297-340 (FORMAT.md)
* marching cubes                        isosurf.py:183-225, kernels.py:428-524

Hot loops run in ``chr_oracle.c`` (built by ``oracle/Makefile`` into
``oracle/_build/``); orchestration is numpy.  The oracle is pinned against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*``, checked by
``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import struct
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libchr_oracle.so")

SAFETY_FACTOR = 1.0 - 2.0**-20  # bound.py:38
HEADER_STRUCT = struct.Struct("<B3IdBQI")  # codec.py:41
FILE_HEADER = struct.Struct("<4sH3I3dBIdd")  # chr_archive.py:50
REGION_FIXED = struct.Struct("<I3I3I3I3IBddQQ")  # chr_archive.py:51
DTYPE_TAGS = {"f32": 0, "f64": 1}  # volume.py:18

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        D = ctypes.c_double
        L.or_lorenzo_encode.argtypes = [P, I, I, I, D, P, P, P]
        L.or_lorenzo_encode.restype = I
        L.or_lorenzo_decode.argtypes = [P, P, P, D, I, I, I, P, P]
        L.or_lorenzo_decode.restype = None
        L.or_rle_encode.argtypes = [P, I, P]
        L.or_rle_encode.restype = I
        L.or_rle_decode.argtypes = [P, I, I, P]
        L.or_rle_decode.restype = ctypes.c_int
        L.or_min_abs_distance.argtypes = [P, I, D]
        L.or_min_abs_distance.restype = D
        L.or_window_min_abs_distance.argtypes = [P, I, I, I, I, I, I, I, I, D]
        L.or_window_min_abs_distance.restype = D
        L.or_gather_window.argtypes = [P, I, I, I, I, I, I, I, I, P]
        L.or_gather_window.restype = None
        L.or_decompose.argtypes = [P, I, I, I, I, P, P]
        L.or_decompose.restype = None
        L.or_merge_regions.argtypes = [P, I, I, I, P]
        L.or_merge_regions.restype = I
        L.or_crc32.argtypes = [ctypes.c_uint32, P, I]
        L.or_crc32.restype = ctypes.c_uint32
        L.or_mc_count.argtypes = [P, I, I, I, D, P]
        L.or_mc_count.restype = I
        L.or_mc_emit.argtypes = [P, I, I, I, D, P, P, P]
        L.or_mc_emit.restype = I
        L.or_case_field.argtypes = [P, I, I, I, D, P]
        L.or_case_field.restype = None
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a.size else None


# ---------------------------------------------------------------------------
# kernel-seam restatements (kernels.py)

RLE_ERRORS = {
    1: "token stream truncated",
    2: "varint too long",
    3: "zero run missing length",
    4: "zero run out of range",
    5: "trailing bytes after token stream",
}


def lorenzo_encode(flat, nx, ny, nz, e):
    flat = np.ascontiguousarray(flat, dtype=np.float64)
    n = nx * ny * nz
    q = np.empty(n, np.int64)
    esc = np.empty(n, np.uint8)
    u = np.empty(n, np.int64)
    lib().or_lorenzo_encode(_p(flat), nx, ny, nz, float(e), _p(q), _p(esc), _p(u))
    return q, esc.astype(bool)


def lorenzo_decode(q, escaped, escape_values, e, nx, ny, nz):
    q = np.ascontiguousarray(q, dtype=np.int64)
    esc = np.ascontiguousarray(escaped, dtype=np.uint8)
    ev = np.ascontiguousarray(escape_values, dtype=np.float64)
    n = nx * ny * nz
    u = np.empty(n, np.int64)
    out = np.empty(n, np.float64)
    lib().or_lorenzo_decode(_p(q), _p(esc), _p(ev) if ev.size else None, float(e), nx, ny, nz, _p(u), _p(out))
    return out


def rle_encode(vals):
    vals = np.ascontiguousarray(vals, dtype=np.int64)
    out = np.empty(6 * vals.size + 16, np.uint8)
    nb = lib().or_rle_encode(_p(vals), vals.size, _p(out))
    return out[:nb].copy()


def rle_decode(buf, n):
    """Returns (vals, err) with err 0 or a code of RLE_ERRORS."""
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    vals = np.zeros(n, np.int64)
    err = lib().or_rle_decode(_p(buf) if buf.size else None, buf.size, n, _p(vals) if n else None)
    return vals, err


def min_abs_distance(flat, k):
    flat = np.ascontiguousarray(flat, dtype=np.float64).reshape(-1)
    return float(lib().or_min_abs_distance(_p(flat), flat.size, float(k)))


def crc32(data: bytes, crc: int = 0) -> int:
    a = np.frombuffer(data, np.uint8)
    return int(lib().or_crc32(crc, _p(a) if a.size else None, a.size))


# ---------------------------------------------------------------------------
# codec (codec.py:91-229)


def _verbatim(flat, source_dtype):
    if source_dtype == "f32":
        narrow = flat.astype("<f4")
        if np.array_equal(narrow.astype(np.float64), flat):
            return 3, narrow.tobytes()
    return 0, flat.astype("<f8").tobytes()


def compress_flat(flat, dims, e, source_dtype="f64"):
    """(codec_id, payload bytes) for an x-fastest flat window."""
    nx, ny, nz = dims
    if e == 0.0:
        return _verbatim(flat, source_dtype)
    q, esc = lorenzo_encode(flat, nx, ny, nz, e)
    tokens = rle_encode(q)
    if esc.any():
        cid = 2
        payload = (
            np.packbits(esc, bitorder="little").tobytes()
            + flat[esc].astype("<f8").tobytes()
            + tokens.tobytes()
        )
    else:
        cid = 1
        payload = tokens.tobytes()
    vid, vpay = _verbatim(flat, source_dtype)
    if len(payload) >= len(vpay):
        return vid, vpay
    return cid, payload


def block_bytes(cid, dims, e, source_dtype, payload):
    return (
        HEADER_STRUCT.pack(cid, *dims, e, DTYPE_TAGS[source_dtype], len(payload), crc32(payload))
        + payload
    )


class OracleError(Exception):
    def __init__(self, kind, msg=""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def decompress_block(blob: bytes, offset: int = 0):
    """Decode one serialized CompressedBlock -> (dims, flat f64)."""
    cid, ex, ey, ez, e, tag, plen, crc = HEADER_STRUCT.unpack_from(blob, offset)
    payload = bytes(blob[offset + HEADER_STRUCT.size: offset + HEADER_STRUCT.size + plen])
    if crc32(payload) != crc:
        raise OracleError("corrupt", "payload checksum mismatch")
    n = ex * ey * ez
    if cid == 0:
        return (ex, ey, ez), np.frombuffer(payload, "<f8", count=n).astype(np.float64)
    if cid == 3:
        return (ex, ey, ez), np.frombuffer(payload, "<f4", count=n).astype(np.float64)
    buf = np.frombuffer(payload, np.uint8)
    if cid == 1:
        esc = np.zeros(n, np.uint8)
        ev = np.empty(0)
        tok = buf
    elif cid == 2:
        nbm = (n + 7) // 8
        if buf.size < nbm:
            raise OracleError("corrupt", "payload shorter than its escape bitmap")
        esc = np.unpackbits(buf[:nbm], count=n, bitorder="little")
        nesc = int(esc.sum())
        off = nbm + 8 * nesc
        if buf.size < off:
            raise OracleError("corrupt", "payload shorter than its escape values")
        ev = np.frombuffer(payload, "<f8", count=nesc, offset=nbm).astype(np.float64)
        tok = buf[off:]
    else:
        raise OracleError("codec", f"unknown codec id {cid}")
    q, err = rle_decode(tok, n)
    if err:
        raise OracleError("corrupt", RLE_ERRORS[err])
    return (ex, ey, ez), lorenzo_decode(q, esc, ev, e, ex, ey, ez)


# ---------------------------------------------------------------------------
# archive (blocking.py, bound.py, chr_archive.py)


def block_grid_shape(dims, bs):
    return tuple(max(1, -(-(d - 1) // bs)) for d in dims)


def _axis_window(bc, bs, n):
    lo = bc * bs
    return lo, min((bc + 1) * bs, n - 1) - lo + 1


class OracleArchive:
    """Plain-data archive: enough to serialise FORMAT.md bytes."""

    def __init__(self, dims, spacing, source_dtype, bs, vrange, candidates, regions):
        self.dims = dims
        self.spacing = spacing
        self.source_dtype = source_dtype
        self.block_size = bs
        self.value_range = vrange
        self.candidates = candidates
        self.regions = regions  # list of dict

    def header_table_nbytes(self):
        mb = (len(self.candidates) + 7) // 8
        return FILE_HEADER.size + 4 + 8 * len(self.candidates) + 4 + len(self.regions) * (REGION_FIXED.size + mb)

    def to_bytes(self) -> bytes:
        m = len(self.candidates)
        mb = (m + 7) // 8
        parts = [
            FILE_HEADER.pack(b"CHR1", 1, *self.dims, *self.spacing, DTYPE_TAGS[self.source_dtype],
                             self.block_size, *self.value_range),
            struct.pack("<I", m),
            struct.pack(f"<{m}d", *self.candidates),
            struct.pack("<I", len(self.regions)),
        ]
        off = self.header_table_nbytes()
        for r in self.regions:
            parts.append(REGION_FIXED.pack(r["id"], *r["lo"], *r["hi"], *r["origin"], *r["extent"],
                                           r.get("bound_mode", 0), r.get("accuracy", 1.0), r["e"], off,
                                           len(r["block"])))
            parts.append(int(r["mask"]).to_bytes(mb, "little"))
            off += len(r["block"])
        parts.extend(r["block"] for r in self.regions)
        blob = b"".join(parts)
        return blob + struct.pack("<I", crc32(blob))


def block_stats(values, dims, bs):
    nbx, nby, nbz = block_grid_shape(dims, bs)
    vmin = np.empty(nbx * nby * nbz)
    vmax = np.empty(nbx * nby * nbz)
    lib().or_decompose(_p(values), *dims, bs, _p(vmin), _p(vmax))
    return vmin, vmax


def relevance_masks(vmin, vmax, candidates):
    masks = np.zeros(vmin.size, np.uint64)
    for ci, k in enumerate(candidates):
        masks |= ((vmin <= k) & (k <= vmax)).astype(np.uint64) << np.uint64(ci)
    return masks


def merge(masks, nb3):
    nbx, nby, nbz = nb3
    out = np.empty((masks.size, 6), np.int32)
    nreg = lib().or_merge_regions(_p(np.ascontiguousarray(masks)), nbx, nby, nbz, _p(out))
    return out[:nreg]


def select_index(nd, accuracy):
    """n of the n-th-smallest rule (bound.py:117-119)."""
    return max(1, 1 + int(np.floor((1.0 - accuracy) * nd)))


def window_distances(win3, k, paper):
    """D for one window (bound.py:68-83 / 106-112): |s - k| over every
    sample, or k - s0, s1 - k over the straddling axis edges."""
    if not paper:
        return np.abs(win3.ravel() - k)
    parts = []
    for axis in range(3):
        a = np.moveaxis(win3, axis, 0)
        s0, s1 = np.minimum(a[:-1], a[1:]), np.maximum(a[:-1], a[1:])
        m = (s0 < k) & (k < s1)
        parts += [k - s0[m], s1[m] - k]
    return np.concatenate(parts) if parts else np.empty(0)


def build_chr(values, dims, candidates, bs, spacing=(1.0, 1.0, 1.0), source_dtype="f32",
              loose_fraction=0.01, out_of_range="error", workers=1, accuracy=1.0, bound_mode="strict_vertices"):
    """Archive build (chr_archive.py:132-212)."""
    paper = bound_mode == "paper_edges"
    values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    nx, ny, nz = dims
    if not np.isfinite(values).all():
        idx = int(np.argmin(np.isfinite(values)))
        raise OracleError("nonfinite", f"{idx}")
    vrange = (float(values.min()), float(values.max()))
    cands = [float(k) for k in candidates]
    if not cands or any(b <= a for a, b in zip(cands, cands[1:])) or not all(np.isfinite(cands)):
        raise OracleError("param", "bad candidates")
    if any(not vrange[0] <= k <= vrange[1] for k in cands) and out_of_range == "error":
        raise OracleError("param", "candidate outside value range")
    nb3 = block_grid_shape(dims, bs)
    vmin, vmax = block_stats(values, dims, bs)
    masks = relevance_masks(vmin, vmax, cands)
    boxes = merge(masks, nb3)
    loose = loose_fraction * (vrange[1] - vrange[0])
    nbx, nby, _ = nb3
    L = lib()

    def one(rid):
        bx, by, bz, hx, hy, hz = (int(v) for v in boxes[rid])
        lo_o = (bx * bs, by * bs, bz * bs)
        hi_w = [_axis_window(c, bs, n) for c, n in zip((hx, hy, hz), dims)]
        ext = tuple(hi_w[a][0] + hi_w[a][1] - lo_o[a] for a in range(3))
        mask = int(masks[bx + nbx * (by + nby * bz)])
        served = [cands[ci] for ci in range(len(cands)) if (mask >> ci) & 1]
        unserved = [k for k in cands if k not in served]
        win = (ctypes.c_void_p(values.ctypes.data), nx, ny, *lo_o, *ext)
        # region_bound (bound.py:150-219)
        best = None
        lossless = False
        w3 = None
        if paper or accuracy != 1.0:
            w3 = np.empty(ext[0] * ext[1] * ext[2])
            L.or_gather_window(*win, _p(w3))
            w3 = w3.reshape(ext[2], ext[1], ext[0])
        for k in served:
            if w3 is None:
                val = L.or_window_min_abs_distance(*win, k)
            else:
                d = window_distances(w3, k, paper)
                if d.size == 0:
                    best = loose if best is None or loose < best else best
                    continue
                n = select_index(d.size, accuracy)
                val = float(np.partition(d, n - 1)[n - 1])
            cand = 0.0 if val == 0.0 else val * SAFETY_FACTOR
            if best is None or cand < best:
                best = cand
            if val == 0.0:
                lossless = True
                break
        if best is None:
            best = loose
        if not lossless:
            cap = best
            for k in unserved:
                margin = L.or_window_min_abs_distance(*win, k) * SAFETY_FACTOR
                if margin < cap:
                    cap = margin
            best = min(best, cap)
        flat = np.empty(ext[0] * ext[1] * ext[2])
        L.or_gather_window(*win, _p(flat))
        cid, payload = compress_flat(flat, ext, best, source_dtype)
        return {
            "id": rid, "lo": (bx, by, bz), "hi": (hx, hy, hz), "origin": lo_o, "extent": ext,
            "mask": mask, "e": best, "codec": cid, "bound_mode": 1 if paper else 0, "accuracy": float(accuracy),
            "block": block_bytes(cid, ext, best, source_dtype, payload),
        }

    if workers > 1:
        with ThreadPoolExecutor(workers) as pool:
            regions = list(pool.map(one, range(len(boxes))))
    else:
        regions = [one(r) for r in range(len(boxes))]
    return OracleArchive(tuple(dims), tuple(float(s) for s in spacing), source_dtype, bs, vrange,
                         tuple(cands), regions)


def request(arch: OracleArchive, k, drop_pruned=True, workers=1):
    """(chr_archive.py:226-274) -> list of (region dict, (ex,ey,ez) f64 flat window)."""
    ci = arch.candidates.index(float(k))
    sel = [r for r in arch.regions if (not drop_pruned) or ((r["mask"] >> ci) & 1)]

    def dec(r):
        return decompress_block(r["block"])[1]

    if workers > 1:
        with ThreadPoolExecutor(workers) as pool:
            wins = list(pool.map(dec, sel))
    else:
        wins = [dec(r) for r in sel]
    return list(zip(sel, wins))


def stitch(sel, dims, fill=np.nan):
    """(chr_archive.py:277-294): windows written in descending (z, y, x)
    origin order, so the lowest origin lands last.  Flat x-fastest f64."""
    nx, ny, nz = dims
    out = np.full((nz, ny, nx), fill, dtype=np.float64)
    for r, w in sorted(sel, key=lambda p: tuple(reversed(p[0]["origin"])), reverse=True):
        (ox, oy, oz), (ex, ey, ez) = r["origin"], r["extent"]
        out[oz:oz + ez, oy:oy + ey, ox:ox + ex] = np.asarray(w).reshape(ez, ey, ex)
    return out.reshape(-1)


def verify_topology(a, b, dims, k):
    """(isosurf.py:91-114): (preserved_fraction, differing, total, first
    differing cell (cx, cy, cz) or None) from binary case codes."""
    ca, cb = case_field(a, dims, k), case_field(b, dims, k)
    diff = ca != cb
    nd = int(diff.sum())
    total = ca.size
    first = None
    if nd:
        flat = int(np.argmax(diff))
        ncx, ncy = dims[0] - 1, dims[1] - 1
        cz, rem = divmod(flat, ncx * ncy)
        cy, cx = divmod(rem, ncx)
        first = [cx, cy, cz]
    return [(total - nd) / total, nd, total, first]


def bytes_touched(arch: OracleArchive, sel):
    return arch.header_table_nbytes() + sum(len(r["block"]) for r, _ in sel)


# ---------------------------------------------------------------------------
# marching cubes (isosurf.py:183-225, kernels.py:428-524)


def mc_lattice(flat, dims, k):
    """(verts lattice f64 (nv,3), tris int32 (nt,3), bourke codes) of one grid."""
    nx, ny, nz = dims
    flat = np.ascontiguousarray(flat, dtype=np.float64).reshape(-1)
    L = lib()
    codes = np.empty(max(0, (nx - 1) * (ny - 1) * (nz - 1)), np.uint8)
    total = L.or_mc_count(_p(flat), nx, ny, nz, float(k), _p(codes))
    verts = np.empty((3 * total, 3), np.float64)
    tris = np.empty((total, 3), np.int32)
    vids = np.empty(3 * flat.size, np.int32)
    nv = L.or_mc_emit(_p(flat), nx, ny, nz, float(k), _p(verts), _p(tris), _p(vids))
    return verts[:nv].copy(), tris, codes


def marching_cubes(flat, dims, k, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)):
    lat, tris, _ = mc_lattice(flat, dims, k)
    verts = np.empty_like(lat)
    for ax in range(3):
        verts[:, ax] = origin[ax] + lat[:, ax] * spacing[ax]
    return verts, tris


def extract_regions(sel, spacing, k):
    """Per-region MC + merge_meshes (pipeline.py:93-103, isosurf.py:207-225)."""
    verts, tris, off = [], [], 0
    for r, win in sel:
        origin = tuple(o * s for o, s in zip(r["origin"], spacing))
        v, t = marching_cubes(win, r["extent"], k, spacing, origin)
        verts.append(v)
        tris.append(t + off)
        off += v.shape[0]
    if not verts:
        return np.empty((0, 3)), np.empty((0, 3), np.int32)
    return np.concatenate(verts), np.concatenate(tris).astype(np.int32)


def case_field(flat, dims, k):
    nx, ny, nz = dims
    flat = np.ascontiguousarray(flat, dtype=np.float64).reshape(-1)
    codes = np.empty((nx - 1) * (ny - 1) * (nz - 1), np.uint8)
    lib().or_case_field(_p(flat), nx, ny, nz, float(k), _p(codes))
    return codes


def bourke_to_binary(codes):
    """Swap bits 2<->3 and 6<->7 (Bourke corner order -> binary order)."""
    c = codes.astype(np.uint8)
    b2 = (c >> 2) & 1
    b3 = (c >> 3) & 1
    b6 = (c >> 6) & 1
    b7 = (c >> 7) & 1
    c = c & np.uint8(0b00110011)
    return c | (b3 << 2) | (b2 << 3) | (b7 << 6) | (b6 << 7)
