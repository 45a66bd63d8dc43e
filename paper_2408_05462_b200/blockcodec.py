"""Single-block codec API (reference: isochr/codec.py:45-229, CODEC.md).

``compress`` / ``decompress`` run the same CUDA kernels as the archive
path, on one region covering the whole array.  The 34-byte header layout,
codec ids 0-3 and the plugin registry (``register_codec``) match the
reference so blocks are interchangeable byte for byte.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi, device
from .exceptions import CorruptPayloadError, NonFiniteSampleError, ParameterError, UnsupportedCodecError

CODEC_VERBATIM = 0
CODEC_LORENZO = 1
CODEC_LORENZO_ESCAPED = 2
CODEC_VERBATIM_F32 = 3

_HDR = struct.Struct("<B3IdBQI")  # codec | dims | bound | dtype | length | crc
HEADER_SIZE = _HDR.size
_TAGS = {"f32": 0, "f64": 1}
_NAMES = {v: k for k, v in _TAGS.items()}

_REGISTRY: dict[int, tuple[str, object]] = {
    CODEC_VERBATIM: ("verbatim", None),
    CODEC_LORENZO: ("lorenzo", None),
    CODEC_LORENZO_ESCAPED: ("lorenzo+escapes", None),
    CODEC_VERBATIM_F32: ("verbatim-f32", None),
}


@dataclass(frozen=True)
class CompressedBlock:
    """Header fields + payload of one compressed region."""

    codec_id: int
    dims: tuple[int, int, int]
    error_bound: float
    source_dtype: str
    payload: bytes
    checksum: int

    @property
    def nbytes(self) -> int:
        return HEADER_SIZE + len(self.payload)

    def to_bytes(self) -> bytes:
        return _HDR.pack(self.codec_id, *self.dims, self.error_bound, _TAGS[self.source_dtype],
                         len(self.payload), self.checksum) + self.payload

    @classmethod
    def from_bytes(cls, buf, offset: int = 0) -> "CompressedBlock":
        cid, ex, ey, ez, eb, tag, plen, crc = _HDR.unpack_from(buf, offset)
        body = bytes(buf[offset + HEADER_SIZE: offset + HEADER_SIZE + plen])
        if len(body) != plen:
            raise CorruptPayloadError(f"payload truncated: header says {plen} bytes, {len(body)} available")
        return cls(cid, (ex, ey, ez), eb, _NAMES[tag], body, crc)


def register_codec(codec_id: int, name: str, decompress_fn) -> None:
    """Plug in an extra codec id (codec.py:207-211); ids 0-3 are built in."""
    if codec_id in _REGISTRY:
        raise ParameterError(f"codec id {codec_id} is already registered")
    _REGISTRY[codec_id] = (name, decompress_fn)


def codec_name(codec_id: int) -> str:
    if codec_id not in _REGISTRY:
        raise UnsupportedCodecError(f"unknown codec id {codec_id}")
    return _REGISTRY[codec_id][0]


def _grid_to_device(samples) -> tuple[torch.Tensor, tuple[int, int, int]]:
    if isinstance(samples, torch.Tensor):
        if samples.ndim != 3:
            raise ParameterError(f"samples must be a 3D array, got ndim={samples.ndim}")
        dims = tuple(int(d) for d in samples.shape)
        t = samples.to(device=_abi.device(), dtype=torch.float64).permute(2, 1, 0).contiguous().reshape(-1)
        return t, dims
    g = np.asarray(samples, dtype=np.float64)
    if g.ndim != 3:
        raise ParameterError(f"samples must be a 3D array, got ndim={g.ndim}")
    flat = g.ravel(order="F")
    fin = np.isfinite(flat)
    if not fin.all():
        i = int(np.argmin(fin))
        raise NonFiniteSampleError(i, float(flat[i]))
    return torch.from_numpy(np.require(flat, requirements=["C", "W"])).to(_abi.device()), tuple(int(d) for d in g.shape)


def compress(samples, error_bound: float, source_dtype: str = "f64") -> CompressedBlock:
    """codec.compress on the GPU (codec.py:91-143)."""
    e = float(error_bound)
    if e < 0 or not np.isfinite(e):
        raise ParameterError(f"error_bound must be finite and >= 0, got {error_bound}")
    if source_dtype not in _TAGS:
        raise ParameterError(f"unknown dtype tag {source_dtype!r}")
    vol, dims = _grid_to_device(samples)
    if isinstance(samples, torch.Tensor):
        fin = torch.isfinite(vol)
        if not bool(fin.all()):
            i = int(torch.argmin(fin.to(torch.uint8)))
            raise NonFiniteSampleError(i, float(vol[i]))
    regs = np.zeros(1, dtype=_abi.REGION_DT)
    regs["extent"][0] = dims
    regs["error_bound"][0] = e
    res = device.compress(vol, dims, regs, source_dtype=source_dtype, write_file=False)
    blob = res.blob[: res.nbytes].cpu().numpy().tobytes()
    return CompressedBlock.from_bytes(blob, 0)


def decompress_many(blocks) -> list[np.ndarray]:
    """Decode several blocks in one device pass; raises for the first bad one
    in order, with the reference's precedence (checksum, codec, payload)."""
    blocks = list(blocks)
    builtin = [i for i, b in enumerate(blocks) if b.codec_id in (0, 1, 2, 3)]
    out: list[np.ndarray | None] = [None] * len(blocks)
    if builtin:
        sizes = [len(blocks[i].payload) for i in builtin]
        # +16 bytes: the tokenizer reads whole aligned words around the last token
        staging = np.frombuffer(b"".join(blocks[i].payload for i in builtin) + bytes(16), dtype=np.uint8)
        dev = torch.from_numpy(staging.copy()).to(_abi.device())
        sel, off = [], 0
        for i, sz in zip(builtin, sizes):
            b = blocks[i]
            sel.append((off, sz, b.codec_id, b.dims, b.error_bound, b.checksum))
            off += sz
        flat, offs, status = device.decode(dev, sel)
        host = flat.cpu().numpy() if sel else None
        for j, i in enumerate(builtin):
            st = status[j]
            if st:
                msg = _abi.DEC_MESSAGES.get(st, "corrupt payload")
                if st == 10:
                    raise UnsupportedCodecError(f"unknown codec id {blocks[i].codec_id}")
                out[i] = CorruptPayloadError(msg)
                continue
            d = blocks[i].dims
            n = d[0] * d[1] * d[2]
            out[i] = host[offs[j]: offs[j] + n].reshape(d, order="F").copy()
    for i, b in enumerate(blocks):
        if out[i] is None:
            import zlib  # plugin codecs: checksum check as the reference does

            actual = zlib.crc32(b.payload)
            if actual != b.checksum:
                out[i] = CorruptPayloadError(
                    f"payload checksum mismatch: header {b.checksum:#010x}, computed {actual:#010x}")
            elif b.codec_id not in _REGISTRY:
                out[i] = UnsupportedCodecError(f"unknown codec id {b.codec_id}")
            else:
                out[i] = _REGISTRY[b.codec_id][1](b)
    for o in out:
        if isinstance(o, Exception):
            raise o
    return out  # type: ignore[return-value]


def decompress(block: CompressedBlock) -> np.ndarray:
    """codec.decompress (codec.py:220-229): CRC check, registry, decode."""
    return decompress_many([block])[0]
