"""CHR archive API on the GPU (reference: isochr/chr_archive.py:54-407,
FORMAT.md).

``build_chr`` runs stats -> plan -> compress on the device and keeps the
finished file resident (``CHRArchive._device``), so a following ``request``
decodes straight from HBM; the returned dataclasses are the reference's
(frozen, compared with ``==``), materialised from one device->host copy.
"""

from __future__ import annotations

import struct
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi, device
from .blockcodec import HEADER_SIZE, CompressedBlock, decompress_many
from .exceptions import (
    BadMagicError,
    ChecksumError,
    CorruptPayloadError,
    InsufficientAccuracyError,
    NoSuchIsovalueError,
    ParameterError,
    UnsupportedCodecError,
)
from .field import DTYPE_TAGS, Volume, as_volume_like

MODE_STRICT = "strict_vertices"
MODE_PAPER = "paper_edges"
MAGIC = b"CHR1"
VERSION = 1
BOUND_MODE_TAGS = {MODE_STRICT: 0, MODE_PAPER: 1}
_MODES = {v: k for k, v in BOUND_MODE_TAGS.items()}
_FILE_HDR = struct.Struct("<4sH3I3dBIdd")
_REC = struct.Struct("<I3I3I3I3IBddQQ")
DEFAULT_SAFETY_FACTOR = device.SAFETY_FACTOR
DEFAULT_LOOSE_FRACTION = device.LOOSE_FRACTION


@dataclass(frozen=True)
class ArchiveRegion:
    region_id: int
    block_span: tuple[tuple[int, int, int], tuple[int, int, int]]
    sample_origin: tuple[int, int, int]
    sample_extent: tuple[int, int, int]
    relevance: frozenset
    bound_mode: str
    accuracy: float
    error_bound: float
    block: CompressedBlock

    @property
    def payload_nbytes(self) -> int:
        return self.block.nbytes

    def is_relevant(self, candidate_index: int) -> bool:
        return candidate_index in self.relevance


@dataclass(frozen=True)
class CHRArchive:
    dims: tuple[int, int, int]
    spacing: tuple[float, float, float]
    source_dtype: str
    block_size: int
    value_range: tuple[float, float]
    candidates: tuple[float, ...]
    regions: tuple[ArchiveRegion, ...]
    # device copy of the serialised file (built here or uploaded on demand)
    _device: dict = field(default=None, compare=False, repr=False, hash=False)

    @property
    def stored_accuracy(self) -> float:
        return self.regions[0].accuracy

    @property
    def bound_mode(self) -> str:
        return self.regions[0].bound_mode

    def header_table_nbytes(self) -> int:
        return device.header_table_nbytes(len(self.candidates), len(self.regions))

    def payload_nbytes(self) -> int:
        return sum(r.payload_nbytes for r in self.regions)

    def file_nbytes(self) -> int:
        return self.header_table_nbytes() + self.payload_nbytes() + 4


@dataclass(frozen=True)
class RequestReport:
    requested_isovalue: float
    isovalue: float
    snapped: bool
    candidate_index: int
    requested_accuracy: float
    stored_accuracy: float
    drop_pruned: bool
    regions_returned: int
    regions_total: int
    bytes_touched: int
    bytes_total: int


@dataclass(frozen=True)
class ReconstructionSet:
    regions: tuple
    report: RequestReport
    # the decoded windows still on the device (f64, element offsets) and the
    # archive's block size, when produced by request(): stitch reuses them
    _device: tuple | None = field(default=None, compare=False, repr=False)


def _check_build_args(accuracy, bound_mode, safety_factor, loose_fraction, out_of_range):
    if not 0.0 < accuracy <= 1.0:
        raise ParameterError(f"accuracy must be in (0, 1], got {accuracy}")
    if not 0.0 < safety_factor < 1.0:
        raise ParameterError(f"safety_factor must be in (0, 1), got {safety_factor}")
    if bound_mode not in BOUND_MODE_TAGS:
        raise ParameterError(f"mode must be one of {tuple(BOUND_MODE_TAGS)}, got {bound_mode!r}")
    if out_of_range not in ("error", "warn"):
        raise ParameterError(f"out_of_range must be 'error' or 'warn', got {out_of_range!r}")
    if not 0.0 < loose_fraction:
        raise ParameterError(f"loose_fraction must be positive, got {loose_fraction}")


def _pinned_host(t: torch.Tensor) -> np.ndarray:
    """A device tensor copied into page-locked host memory (torch's caching
    host allocator recycles the buffers), as numpy: ~55 GB/s instead of the
    few GB/s of a pageable .cpu() (1 GB of c3 windows: 20 ms, not 0.45 s)."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def _regions_from_device(res: device.Compressed, host_blob, cands, source_dtype, bound_mode=MODE_STRICT,
                         accuracy=1.0):
    out = []
    for rec in device.region_records(res.regions):
        blk = CompressedBlock.from_bytes(host_blob, rec["block_offset"])
        mask = rec["mask"]
        out.append(ArchiveRegion(
            region_id=rec["id"], block_span=(rec["lo"], rec["hi"]), sample_origin=rec["origin"],
            sample_extent=rec["extent"], relevance=frozenset(ci for ci in range(len(cands)) if (mask >> ci) & 1),
            bound_mode=bound_mode, accuracy=float(accuracy), error_bound=rec["e"], block=blk))
    return tuple(out)


def build_chr(volume, candidates, block_size: int, accuracy: float = 1.0, bound_mode: str = MODE_STRICT,
              safety_factor: float = DEFAULT_SAFETY_FACTOR, loose_fraction: float = DEFAULT_LOOSE_FRACTION,
              out_of_range: str = "error", workers: int = 1, codec=None) -> CHRArchive:
    """chr_archive.build_chr (chr_archive.py:132-212) on the GPU."""
    del workers  # one device pass; kept for signature compatibility
    _check_build_args(accuracy, bound_mode, safety_factor, loose_fraction, out_of_range)
    if block_size < 2:
        raise ParameterError(f"block_size must be >= 2, got {block_size}")
    vol = as_volume_like(volume)
    if any(d < 2 for d in vol.dims):
        raise ParameterError(f"volume dims must be >= 2 per axis, got {vol.dims}")
    cands = [float(k) for k in candidates]
    if not cands:
        raise ParameterError("candidates must be non-empty")
    if any(not np.isfinite(k) for k in cands):
        raise ParameterError("candidates must be finite")
    if any(b <= a for a, b in zip(cands, cands[1:])):
        raise ParameterError(f"candidates must be strictly increasing, got {cands}")
    dvals = vol.device_values()
    res = device.build_archive(dvals, vol.dims, cands, block_size, spacing=vol.spacing,
                               source_dtype=vol.source_dtype, loose_fraction=loose_fraction,
                               safety_factor=safety_factor, vrange=vol.known_range(), out_of_range=out_of_range,
                               on_warn=lambda m: warnings.warn(m, stacklevel=3), accuracy=accuracy,
                               bound_mode=bound_mode)
    if vol.known_range() is None:  # a device field: the range comes from the stats pass just run
        vol._set_range(res.extra["vrange"])
    if codec is not None:
        return _rebuild_with_plugin(vol, res, cands, block_size, codec, bound_mode, accuracy)
    host = _pinned_host(res.blob[: res.nbytes])  # the file bytes (serialize() makes `bytes` on demand)
    regions = _regions_from_device(res, host, cands, vol.source_dtype, bound_mode, accuracy)
    # own copy: res.blob is reusable workspace; +16 slack for aligned word reads
    dev = {"blob": res.blob[: min(res.blob.numel(), res.nbytes + 16)].clone(), "file": host}
    return CHRArchive(vol.dims, vol.spacing, vol.source_dtype, int(block_size), tuple(res.extra["vrange"]),
                      tuple(cands), regions, dev)


def _rebuild_with_plugin(vol, res, cands, bs, codec, bound_mode=MODE_STRICT, accuracy=1.0):
    """build_chr(codec=...) seam (chr_archive.py:142,185): GPU bounds, plugin bytes."""
    grid = vol.grid
    regions = []
    for rec in device.region_records(res.regions):
        (ox, oy, oz), (ex, ey, ez) = rec["origin"], rec["extent"]
        blk = codec(grid[ox:ox + ex, oy:oy + ey, oz:oz + ez], rec["e"], vol.source_dtype)
        mask = rec["mask"]
        regions.append(ArchiveRegion(rec["id"], (rec["lo"], rec["hi"]), rec["origin"], rec["extent"],
                                     frozenset(ci for ci in range(len(cands)) if (mask >> ci) & 1),
                                     bound_mode, float(accuracy), rec["e"], blk))
    return CHRArchive(vol.dims, vol.spacing, vol.source_dtype, int(bs), tuple(res.extra["vrange"]),
                      tuple(cands), tuple(regions))


def _select_candidate(archive: CHRArchive, k: float, snap: bool):
    c = np.asarray(archive.candidates)
    hit = np.flatnonzero(c == k)
    if hit.size:
        return int(hit[0]), False
    if not snap:
        raise NoSuchIsovalueError(k, archive.candidates)
    return int(np.argmin(np.abs(c - k))), True


def _device_file(archive: CHRArchive):
    """The archive's serialised bytes on the device (uploading once if needed)."""
    d = archive._device
    if d is not None and "blob" in d:
        return d["blob"]
    blob = serialize(archive) + bytes(16)  # slack for aligned word reads at the end
    t = torch.from_numpy(np.frombuffer(blob, dtype=np.uint8).copy()).to(_abi.device())
    if d is not None:
        d["blob"] = t
    return t


def _block_offsets(archive: CHRArchive):
    off = archive.header_table_nbytes()
    out = []
    for r in archive.regions:
        out.append(off)
        off += r.payload_nbytes
    return out


def request_device(archive: CHRArchive, k: float, accuracy=None, drop_pruned=True, snap=False):
    """request() keeping the windows on the device: returns
    (selected regions, f64 device tensor of windows, element offsets, report)."""
    k = float(k)
    ci, snapped = _select_candidate(archive, k, snap)
    stored = archive.stored_accuracy
    req = stored if accuracy is None else float(accuracy)
    if req > stored:
        raise InsufficientAccuracyError(req, stored)
    offs = _block_offsets(archive)
    sel = [(r, o) for r, o in zip(archive.regions, offs) if (not drop_pruned) or r.is_relevant(ci)]
    builtin = all(r.block.codec_id in (0, 1, 2, 3) for r, _ in sel)
    windows, woffs = None, []
    if builtin and sel:
        blob = _device_file(archive)
        desc = [(o + HEADER_SIZE, len(r.block.payload), r.block.codec_id, r.block.dims, r.block.error_bound,
                 r.block.checksum) for r, o in sel]
        # the windows get their own buffer: a ReconstructionSet keeps them for
        # stitch(), so they must not alias the decoder's reusable workspace
        total = sum(int(r.block.dims[0]) * int(r.block.dims[1]) * int(r.block.dims[2]) for r, _ in sel)
        own = torch.empty(max(total, 1), dtype=torch.float64, device=blob.device)
        windows, woffs, status = device.decode(blob, desc, out=own)
        for (r, _), st in zip(sel, status):
            if st == 10:
                raise UnsupportedCodecError(f"unknown codec id {r.block.codec_id}")
            if st:
                raise CorruptPayloadError(_abi.DEC_MESSAGES.get(st, "corrupt payload"))
    touched = archive.header_table_nbytes() + sum(r.payload_nbytes for r, _ in sel)
    report = RequestReport(k, archive.candidates[ci], snapped, ci, req, stored, drop_pruned, len(sel),
                           len(archive.regions), touched, archive.file_nbytes())
    return [r for r, _ in sel], windows, woffs, report, builtin


def request(archive: CHRArchive, k: float, accuracy=None, drop_pruned: bool = True, snap: bool = False,
            workers: int = 1) -> ReconstructionSet:
    """chr_archive.request (chr_archive.py:226-274) on the GPU."""
    del workers
    regs, windows, woffs, report, builtin = request_device(archive, k, accuracy, drop_pruned, snap)
    if not builtin:
        arrays = decompress_many([r.block for r in regs])
    else:
        # one D2H of every window; each region's array is a read-only
        # Fortran-order view of it, and marching_cubes on such a view reads
        # the device copy instead of uploading it again (device.host_window)
        host = _pinned_host(windows) if regs else None
        arrays = []
        if regs:
            host.setflags(write=False)
            device.register_host_windows(host, windows)
        for r, o in zip(regs, woffs):
            d = r.block.dims
            n = d[0] * d[1] * d[2]
            arrays.append(host[o:o + n].reshape(d, order="F"))
    dev = (windows, list(woffs), archive.block_size) if builtin and regs else None
    return ReconstructionSet(tuple(zip(regs, arrays)), report, dev)


def _stitch_bs(regions, dims) -> tuple[int, bool]:
    """Block size from the regions' spans (origin = lo * bs); (max dim, True)
    when no region starts past block 0 (one region: spans are irrelevant)."""
    for r in regions:
        for a in range(3):
            lo = r.block_span[0][a]
            if lo > 0:
                return r.sample_origin[a] // lo, False
    return max(max(dims) - 1, 1), True


def stitch_device(recon: ReconstructionSet, dims, fill: float = np.nan) -> torch.Tensor:
    """stitch() leaving the volume on the device: a (nx, ny, nz) float64
    view of an x-fastest buffer (chr_stitch; every sample written once by
    its owner, the region with the lowest (z, y, x) origin)."""
    dims = tuple(int(d) for d in dims)
    regs = [r for r, _ in recon.regions]
    if recon._device is not None:
        windows, woffs, bs = recon._device
        single = False
    else:
        arrays = [np.asarray(a, dtype=np.float64) for _, a in recon.regions]
        woffs = list(np.cumsum([0] + [a.size for a in arrays])[:-1])
        flat = np.concatenate([a.ravel(order="F") for a in arrays]) if arrays else np.zeros(1)
        windows = torch.from_numpy(flat).to(_abi.device())
        bs, single = _stitch_bs(regs, dims)
    t = np.zeros(len(regs), dtype=_abi.STITCH_DT)
    for i, (r, o) in enumerate(zip(regs, woffs)):
        t[i] = (o, r.sample_origin, r.sample_extent, (0, 0, 0) if single else r.block_span[0],
                (0, 0, 0) if single else r.block_span[1])
    out = device.stitch(windows, t, dims, bs, fill)
    return out.view(dims[2], dims[1], dims[0]).permute(2, 1, 0)


def stitch(recon: ReconstructionSet, dims, fill: float = np.nan) -> np.ndarray:
    """chr_archive.stitch (chr_archive.py:277-294) on the GPU: owner-wins
    reassembly, the lower (z, y, x) origin wins; returns the numpy grid."""
    v = stitch_device(recon, dims, fill)
    return v.permute(2, 1, 0).cpu().numpy().reshape(-1).reshape(tuple(int(d) for d in dims), order="F")


def serialize(archive: CHRArchive) -> bytes:
    """FORMAT.md bytes of an archive (header, candidates, table, blocks, CRC)."""
    d = archive._device
    if d is not None and "file" in d:
        if not isinstance(d["file"], bytes):  # build_chr keeps the pinned host copy
            d["file"] = d["file"].tobytes()
        return d["file"]
    m = len(archive.candidates)
    mb = (m + 7) // 8
    parts = [_FILE_HDR.pack(MAGIC, VERSION, *archive.dims, *archive.spacing, DTYPE_TAGS[archive.source_dtype],
                            archive.block_size, *archive.value_range),
             struct.pack("<I", m), struct.pack(f"<{m}d", *archive.candidates),
             struct.pack("<I", len(archive.regions))]
    off = archive.header_table_nbytes()
    for r in archive.regions:
        mask = sum(1 << ci for ci in r.relevance)
        parts.append(_REC.pack(r.region_id, *r.block_span[0], *r.block_span[1], *r.sample_origin,
                               *r.sample_extent, BOUND_MODE_TAGS[r.bound_mode], r.accuracy, r.error_bound, off,
                               r.payload_nbytes))
        parts.append(mask.to_bytes(mb, "little"))
        off += r.payload_nbytes
    parts.extend(r.block.to_bytes() for r in archive.regions)
    body = b"".join(parts)
    return body + struct.pack("<I", _gpu_crc(body))


def _gpu_crc(b: bytes) -> int:
    if not b:
        return 0
    t = torch.from_numpy(np.frombuffer(b, dtype=np.uint8).copy()).to(_abi.device())
    return device.crc32(t)


def write_chr(archive: CHRArchive, path) -> None:
    """chr_archive.write_chr (chr_archive.py:297-340)."""
    with open(path, "wb") as fh:
        fh.write(serialize(archive))


def _upload_file(blob: bytes) -> torch.Tensor:
    """The file in HBM (+16 zero bytes of slack for aligned word reads)."""
    host = torch.empty(len(blob) + 16, dtype=torch.uint8, pin_memory=True)
    host[: len(blob)].numpy()[:] = np.frombuffer(blob, dtype=np.uint8)
    host[len(blob):] = 0
    return host.to(_abi.device(), non_blocking=True)


def read_chr(path) -> CHRArchive:
    """chr_archive.read_chr (chr_archive.py:343-407): the file goes to HBM
    once; the whole-file CRC, the header and every region record + block
    header are validated there (device.read_table); the same exceptions
    are raised in the reference's order.  The device copy stays attached,
    so a following request() decodes without another upload."""
    with open(path, "rb") as fh:
        blob = fh.read()
    n = len(blob)
    if n < _FILE_HDR.size + 4:
        raise ChecksumError(f"{path}: file too short to be a CHR archive")
    if blob[:4] != MAGIC:
        raise BadMagicError(f"{path}: bad magic {blob[:4]!r}, expected {MAGIC!r}")
    file_dev = _upload_file(blob)
    ft = device.read_table(file_dev, n)
    info = ft.info[0]
    if int(info["stored_crc"]) != int(info["actual_crc"]):
        raise ChecksumError(f"{path}: checksum mismatch (stored {int(info['stored_crc']):#010x}, "
                            f"computed {int(info['actual_crc']):#010x})")
    if int(info["version"]) != VERSION:
        from .exceptions import VersionError

        raise VersionError(f"{path}: unsupported CHR version {int(info['version'])}")
    if int(info["error"]) == _abi.READ_TABLE_PAST_END:
        raise struct.error(f"{path}: region table extends past the end of the file")
    m = int(info["m"])
    mb = (m + 7) // 8
    ent = ft.entries
    bad = np.nonzero(ent["status"])[0]
    if bad.size:
        e = ent[int(bad[0])]
        rid, st = int(e["region_id"]), int(e["status"])
        if st == _abi.READ_PAYLOAD_PAST_END:
            raise ChecksumError(f"{path}: region {rid} payload exceeds file size")
        if st == _abi.READ_BLOCK_HEADER_TRUNCATED:
            raise struct.error(f"{path}: region {rid} block header truncated")
        if st == _abi.READ_PAYLOAD_TRUNCATED:
            avail = n - int(e["region"]["block_offset"]) - HEADER_SIZE
            raise CorruptPayloadError(f"payload truncated: header says {int(e['payload_len'])} bytes, "
                                      f"{avail} available")
        raise ChecksumError(f"{path}: region {rid} payload length mismatch (table {int(e['region']['block_nbytes'])}, "
                            f"block {HEADER_SIZE + int(e['payload_len'])})")
    names = {0: "f32", 1: "f64"}
    table0 = int(info["table_nbytes"]) - len(ent) * (_REC.size + mb)
    regions = []
    for i, e in enumerate(ent):
        r = e["region"]
        if m <= 64:
            mask = int(r["mask"])
        else:  # wider masks than the device entry holds: from the record bytes
            p = table0 + i * (_REC.size + mb) + _REC.size
            mask = int.from_bytes(blob[p:p + mb], "little")
        off = int(r["block_offset"]) + HEADER_SIZE
        blk = CompressedBlock(int(r["codec_id"]), tuple(int(d) for d in e["block_dims"]),
                              float(e["block_error_bound"]), names[int(e["block_dtype"])],
                              blob[off:off + int(e["payload_len"])], int(r["payload_crc"]))
        regions.append(ArchiveRegion(int(e["region_id"]), (tuple(int(v) for v in r["lo"]), tuple(int(v) for v in r["hi"])),
                                     tuple(int(v) for v in r["origin"]), tuple(int(v) for v in r["extent"]),
                                     frozenset(ci for ci in range(m) if (mask >> ci) & 1),
                                     _MODES[int(e["bound_mode"])], float(e["accuracy"]), float(r["error_bound"]), blk))
    dtype = {v: k for k, v in DTYPE_TAGS.items()}[int(info["dtype"])]
    return CHRArchive(tuple(int(d) for d in info["dims"]), tuple(float(s) for s in info["spacing"]), dtype,
                      int(info["block_size"]), (float(info["vmin"]), float(info["vmax"])),
                      tuple(float(c) for c in ft.candidates), tuple(regions), {"file": blob, "blob": file_dev})


__all__ = ["ArchiveRegion", "CHRArchive", "RequestReport", "ReconstructionSet", "build_chr", "request",
           "request_device", "stitch", "write_chr", "read_chr", "serialize", "MODE_STRICT", "MODE_PAPER", "Volume"]
