"""ctypes binding of libchr.so (include/chr.h).

The library is built in-tree (``paper_2408_05462_b200/libchr.so``, see
``csrc/Makefile`` and ``__graft_entry__.build``).  There is deliberately no
CPU fallback: importing the compute entry points without the library or
without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import exceptions as errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHR_LIB_PATH") or os.path.join(_HERE, "libchr.so")

CHR_OK = 0
CHR_E_PARAMETER = 1
CHR_E_NONFINITE = 2
CHR_E_CORRUPT = 3
CHR_E_UNSUPPORTED_CODEC = 4
CHR_E_CUDA = 5
CHR_E_WORKSPACE = 6

DEC_MESSAGES = {
    1: "token stream truncated",
    2: "varint too long",
    3: "zero run missing length",
    4: "zero run out of range",
    5: "trailing bytes after token stream",
    6: "token stream produced wrong count",
    7: "payload checksum mismatch",
    8: "payload shorter than its escape bitmap",
    9: "payload shorter than its escape values",
    10: "unknown codec id",
}

P = ctypes.c_void_p
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
D = ctypes.c_double
INT = ctypes.c_int
SZ = ctypes.c_size_t


class Region(ctypes.Structure):
    """chr_region_t"""

    _fields_ = [
        ("lo", ctypes.c_int32 * 3),
        ("hi", ctypes.c_int32 * 3),
        ("origin", ctypes.c_int32 * 3),
        ("extent", ctypes.c_int32 * 3),
        ("mask", ctypes.c_uint64),
        ("error_bound", ctypes.c_double),
        ("codec_id", ctypes.c_int32),
        ("payload_crc", ctypes.c_uint32),
        ("block_offset", ctypes.c_uint64),
        ("block_nbytes", ctypes.c_uint64),
        ("n_escaped", ctypes.c_uint64),
    ]


class DecRegion(ctypes.Structure):
    """chr_dec_region_t"""

    _fields_ = [
        ("payload_offset", ctypes.c_uint64),
        ("payload_nbytes", ctypes.c_uint64),
        ("codec_id", ctypes.c_int32),
        ("dims", ctypes.c_int32 * 3),
        ("error_bound", ctypes.c_double),
        ("crc", ctypes.c_uint32),
        ("_pad", ctypes.c_uint32),
        ("out_offset", ctypes.c_uint64),
    ]


class McGrid(ctypes.Structure):
    """chr_mc_grid_t"""

    _fields_ = [
        ("grid_offset", ctypes.c_uint64),
        ("dims", ctypes.c_int32 * 3),
        ("zoff", ctypes.c_int32),
        ("origin", ctypes.c_double * 3),
        ("spacing", ctypes.c_double * 3),
    ]


# numpy mirrors of the ABI structs (vectorised fill / read, no per-field ctypes)
REGION_DT = np.dtype([("lo", "<i4", 3), ("hi", "<i4", 3), ("origin", "<i4", 3), ("extent", "<i4", 3),
                      ("mask", "<u8"), ("error_bound", "<f8"), ("codec_id", "<i4"), ("payload_crc", "<u4"),
                      ("block_offset", "<u8"), ("block_nbytes", "<u8"), ("n_escaped", "<u8")], align=True)
PORTION_DT = np.dtype([("len", "<i8"), ("lead", "<i8"), ("trail", "<i8"), ("bytes", "<i8"), ("nesc", "<i8"),
                       ("nz", "<i4"), ("f32ok", "<i4")])  # chr_portion_t
DEC_DT = np.dtype([("payload_offset", "<u8"), ("payload_nbytes", "<u8"), ("codec_id", "<i4"), ("dims", "<i4", 3),
                   ("error_bound", "<f8"), ("crc", "<u4"), ("_pad", "<u4"), ("out_offset", "<u8")], align=True)
MCGRID_DT = np.dtype([("grid_offset", "<u8"), ("dims", "<i4", 3), ("zoff", "<i4"), ("origin", "<f8", 3),
                      ("spacing", "<f8", 3)], align=True)
AFTER_COMPRESS = ctypes.CFUNCTYPE(None, ctypes.c_uint64, ctypes.c_void_p)  # chr_after_compress_fn
STITCH_DT = np.dtype([("window_offset", "<u8"), ("origin", "<i4", 3), ("extent", "<i4", 3), ("block_lo", "<i4", 3),
                      ("block_hi", "<i4", 3)])  # chr_stitch_t
assert STITCH_DT.itemsize == 56
FILE_INFO_DT = np.dtype([("magic", "S4"), ("version", "<u4"), ("dims", "<u4", 3), ("spacing", "<f8", 3),
                         ("dtype", "<u4"), ("block_size", "<u4"), ("vmin", "<f8"), ("vmax", "<f8"), ("m", "<u4"),
                         ("n_regions", "<u4"), ("table_nbytes", "<u8"), ("stored_crc", "<u4"),
                         ("actual_crc", "<u4"), ("error", "<i4"), ("_pad", "<i4")], align=True)  # chr_file_info_t
TABLE_ENTRY_DT = np.dtype([("region", REGION_DT), ("region_id", "<u4"), ("status", "<i4"), ("bound_mode", "<u4"),
                           ("block_dtype", "<u4"), ("accuracy", "<f8"), ("block_dims", "<u4", 3), ("_pad", "<u4"),
                           ("block_error_bound", "<f8"), ("payload_len", "<u8")], align=True)  # chr_table_entry_t
assert FILE_INFO_DT.itemsize == 104 and TABLE_ENTRY_DT.itemsize == 152
PIPE_RES_DT = np.dtype([("n_regions", "<i8"), ("n_selected", "<i8"), ("archive_nbytes", "<u8"),
                        ("archive_needed", "<u8"), ("n_tri", "<i8"), ("n_vert", "<i8"), ("window_samples", "<u8"),
                        ("windows_offset", "<u8"), ("masks_offset", "<u8"), ("ws_needed", "<u8"),
                        ("first_nonfinite", "<i8"), ("vmin", "<f8"), ("vmax", "<f8")])  # chr_pipeline_result_t
READ_TOO_SHORT, READ_BAD_MAGIC, READ_TABLE_PAST_END, READ_PAYLOAD_PAST_END = 1, 2, 3, 4
READ_BLOCK_HEADER_TRUNCATED, READ_PAYLOAD_TRUNCATED, READ_LENGTH_MISMATCH = 5, 6, 7
assert REGION_DT.itemsize == ctypes.sizeof(Region)
assert DEC_DT.itemsize == ctypes.sizeof(DecRegion)
assert MCGRID_DT.itemsize == ctypes.sizeof(McGrid)


def aptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else None


_lib = None


def lib():
    """The loaded library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libchr.so not found at {LIB_PATH}: run __graft_entry__.build() "
                "(make -C paper_2408_05462_b200/csrc); there is no CPU fallback"
            )
        L = ctypes.CDLL(LIB_PATH)
        L.chr_abi_version.restype = INT
        L.chr_status_string.argtypes = [INT]
        L.chr_status_string.restype = ctypes.c_char_p
        L.chr_num_blocks.argtypes = [I64, I64, I64, I64]
        L.chr_num_blocks.restype = I64
        L.chr_stats.argtypes = [P, INT, I64, I64, I64, I64, P, INT, P, P, P]
        L.chr_stats.restype = INT
        L.chr_plan.argtypes = [P, I64, I64, I64, I64, P, INT, D, D, D, D, P, P]
        L.chr_plan.restype = INT
        L.chr_merge_keys.argtypes = [P, I64, I64, I64, P, P]
        L.chr_merge_keys.restype = INT
        L.chr_value_range.argtypes = [P, INT, I64, P, SZ, P, P, P]
        L.chr_value_range.restype = INT
        L.chr_compress_workspace_size.argtypes = [P, I64]
        L.chr_compress_workspace_size.restype = SZ
        L.chr_compress_capacity.argtypes = [P, I64, INT, INT]
        L.chr_compress_capacity.restype = U64
        L.chr_compress.argtypes = [P, INT, INT, I64, I64, I64, P, I64, D, D, P, INT, P, I64, INT, P, SZ,
                                   P, U64, P, P]
        L.chr_compress.restype = INT
        L.chr_decode_workspace_size.argtypes = [P, I64]
        L.chr_decode_workspace_size.restype = SZ
        L.chr_decode_regions.argtypes = [P, P, I64, P, P, SZ, P, P]
        L.chr_decode_regions.restype = INT
        L.chr_mc_workspace_size.argtypes = [P, I64]
        L.chr_mc_workspace_size.restype = SZ
        L.chr_mc_count.argtypes = [P, P, I64, D, P, SZ, P, P, P, P, P]
        L.chr_mc_count.restype = INT
        L.chr_mc_emit.argtypes = [P, P, I64, D, P, SZ, P, P, P]
        L.chr_mc_emit.restype = INT
        L.chr_case_codes.argtypes = [P, I64, I64, I64, D, INT, P, P]
        L.chr_case_codes.restype = INT
        L.chr_crc32_workspace_size.argtypes = [U64]
        L.chr_crc32_workspace_size.restype = SZ
        L.chr_crc32.argtypes = [P, U64, P, SZ, P, P]
        L.chr_crc32.restype = INT
        L.chr_crc32_segments_workspace_size.argtypes = [I64]
        L.chr_crc32_segments_workspace_size.restype = SZ
        L.chr_crc32_segments.argtypes = [P, P, I64, P, SZ, P, P, P]
        L.chr_crc32_segments.restype = INT
        L.chr_crc32_shift.argtypes = [ctypes.c_uint32, U64]
        L.chr_crc32_shift.restype = ctypes.c_uint32
        L.chr_crc32_shift_many.argtypes = [P, P, I64, P]
        L.chr_crc32_shift_many.restype = None
        L.chr_mc_emit_edges.argtypes = [P, P, I64, D, P, SZ, P, P, P, P]
        L.chr_mc_emit_edges.restype = INT
        L.chr_portion_finish.argtypes = [P, P, P, P, P, P, I64, P, P, SZ, P]
        L.chr_portion_finish.restype = INT
        L.chr_copy_segments.argtypes = [P, P, P, P, I64, INT, P, SZ, P]
        L.chr_copy_segments.restype = INT
        L.chr_slab_classify.argtypes = [P, I64, P, INT, P, P, P, P, SZ, P]
        L.chr_slab_classify.restype = INT
        L.chr_slab_gid.argtypes = [P, I64, P, INT, P, P, SZ, P]
        L.chr_slab_gid.restype = INT
        L.chr_crc32_combine.argtypes = [ctypes.c_uint32, ctypes.c_uint32, U64]
        L.chr_crc32_combine.restype = ctypes.c_uint32
        L.chr_min_abs_distance.argtypes = [P, I64, D, P, P, SZ, P]
        L.chr_min_abs_distance.restype = INT
        L.chr_lorenzo_encode.argtypes = [P, I64, I64, I64, D, P, P, P]
        L.chr_lorenzo_encode.restype = INT
        L.chr_dcompress_workspace_size.argtypes = [P, I64, I64, I64, I64, I64]
        L.chr_dcompress_workspace_size.restype = SZ
        L.chr_dcompress_local.argtypes = [P, INT, INT, I64, I64, I64, I64, I64, I64, P, I64, P, SZ, P, P]
        L.chr_dcompress_local.restype = INT
        L.chr_dcompress_finish.argtypes = [P, INT, INT, I64, I64, I64, I64, I64, I64, P, I64, D, D, P, INT, P, I64,
                                           P, INT, INT, P, SZ, P, U64, P, P, P]
        L.chr_dcompress_finish.restype = INT
        L.chr_dcompress_headers.argtypes = [I64, I64, I64, INT, P, I64, D, D, P, INT, P, I64, P, P, SZ, P, P]
        L.chr_dcompress_headers.restype = INT
        L.chr_select_workspace_size.argtypes = [I64]
        L.chr_select_workspace_size.restype = SZ
        L.chr_select_distances.argtypes = [P, INT, I64, I64, I64, P, P, I64, D, INT, P, SZ, P, P, P, P]
        L.chr_select_distances.restype = INT
        L.chr_compress2.argtypes = [P, INT, INT, I64, I64, I64, P, I64, D, D, P, INT, P, I64, INT, INT, D, P, SZ,
                                    P, U64, P, P]
        L.chr_compress2.restype = INT
        L.chr_stitch_workspace_size.argtypes = [I64, I64, I64, I64, I64]
        L.chr_stitch_workspace_size.restype = SZ
        L.chr_stitch.argtypes = [P, P, I64, I64, I64, I64, I64, P, SZ, P, P]
        L.chr_stitch.restype = INT
        L.chr_topology_compare.argtypes = [P, INT, P, INT, I64, I64, I64, D, P, SZ, P, P, P]
        L.chr_topology_compare.restype = INT
        L.chr_read_header.argtypes = [P, U64, P, P]
        L.chr_read_header.restype = INT
        L.chr_read_workspace_size.argtypes = [U64, I64]
        L.chr_read_workspace_size.restype = SZ
        L.chr_read_archive.argtypes = [P, U64, P, P, P, P, SZ, P]
        L.chr_read_archive.restype = INT
        L.chr_mask_words.argtypes = [P, I64]
        L.chr_mask_words.restype = U64
        L.chr_decode_regions_mask.argtypes = [P, P, I64, P, P, SZ, P, D, P, P]
        L.chr_decode_regions_mask.restype = INT
        L.chr_mc_count_masked.argtypes = [P, P, I64, D, P, P, SZ, P, P, P, P, P]
        L.chr_mc_count_masked.restype = INT
        L.chr_mc_emit_masked.argtypes = [P, P, I64, D, P, P, SZ, P, P, P]
        L.chr_mc_emit_masked.restype = INT
        L.chr_sm_copy.argtypes = [P, P, U64, INT, P]
        L.chr_sm_copy.restype = INT
        L.chr_rle_encode_workspace_size.argtypes = [I64]
        L.chr_rle_encode_workspace_size.restype = SZ
        L.chr_rle_encode.argtypes = [P, I64, P, U64, P, SZ, P, P]
        L.chr_rle_encode.restype = INT
        L.chr_prof_enable.argtypes = [INT]
        L.chr_prof_enable.restype = None
        L.chr_launch_count.argtypes = []
        L.chr_launch_count.restype = ctypes.c_longlong
        L.chr_prof_report.argtypes = [ctypes.c_char_p, SZ]
        L.chr_prof_report.restype = INT
        L.chr_prof_timeline.argtypes = [ctypes.c_char_p, SZ]
        L.chr_prof_timeline.restype = INT
        L.chr_prof_mark.argtypes = [ctypes.c_char_p, P]
        L.chr_prof_mark.restype = None
        L.chr_copy.argtypes = [P, P, U64, P]
        L.chr_copy.restype = INT
        L.chr_request_tables.argtypes = [P, I64, INT, P, P, P, P, P]
        L.chr_request_tables.restype = I64
        L.chr_pipeline.argtypes = [P, INT, INT, I64, I64, I64, P, I64, P, INT, D, D, INT, P, SZ, P, U64, P, I64, P,
                                   I64, P, P, AFTER_COMPRESS, P, P, P]
        L.chr_pipeline.restype = INT
        _lib = L
    return _lib


EXPORTS = [
    "chr_rle_encode_workspace_size", "chr_rle_encode", "chr_sm_copy",
    "chr_mask_words", "chr_decode_regions_mask", "chr_mc_count_masked", "chr_mc_emit_masked",
    "chr_select_workspace_size", "chr_select_distances", "chr_compress2",
    "chr_stitch_workspace_size", "chr_stitch", "chr_topology_compare",
    "chr_read_header", "chr_read_workspace_size", "chr_read_archive", "chr_prof_timeline",
    "chr_prof_mark", "chr_copy", "chr_request_tables", "chr_pipeline",
    "chr_dcompress_workspace_size", "chr_dcompress_local", "chr_dcompress_finish", "chr_dcompress_headers",
    "chr_abi_version", "chr_status_string", "chr_num_blocks", "chr_stats", "chr_plan", "chr_merge_keys",
    "chr_value_range", "chr_crc32_segments_workspace_size", "chr_crc32_segments", "chr_crc32_shift", "chr_crc32_shift_many",
    "chr_mc_emit_edges", "chr_portion_finish", "chr_copy_segments", "chr_slab_classify", "chr_slab_gid",
    "chr_compress_workspace_size", "chr_compress_capacity", "chr_compress",
    "chr_decode_workspace_size", "chr_decode_regions", "chr_mc_workspace_size", "chr_mc_count",
    "chr_mc_emit", "chr_case_codes", "chr_crc32_workspace_size", "chr_crc32", "chr_crc32_combine",
    "chr_min_abs_distance", "chr_lorenzo_encode", "chr_prof_enable", "chr_launch_count", "chr_prof_report",
]


def prof_report() -> dict[str, tuple[int, float]]:
    """{kernel: (launches, total_ms)} since the last call (CUDA events)."""
    L = lib()
    buf = ctypes.create_string_buffer(1 << 16)
    L.chr_prof_report(buf, 1 << 16)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.rsplit(" ", 2)
        out[name] = (int(cnt), float(ms))
    return out


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2408_05462_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())


def check(rc: int, what: str = ""):
    if rc == CHR_OK:
        return
    msg = lib().chr_status_string(rc).decode()
    if what:
        msg = f"{what}: {msg}"
    if rc == CHR_E_PARAMETER:
        raise errors.ParameterError(msg)
    if rc == CHR_E_CORRUPT:
        raise errors.CorruptPayloadError(msg)
    if rc == CHR_E_UNSUPPORTED_CODEC:
        raise errors.UnsupportedCodecError(msg)
    raise RuntimeError(msg)
