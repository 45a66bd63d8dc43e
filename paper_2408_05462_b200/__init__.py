"""paper_2408_05462_b200 -- B200-native (sm_100a) CHR hot path of arXiv 2408.05462.

Drop-in for the reference package ``isochr`` on the path BASELINE.json
``north_star`` names: block decomposition + min/max index, topology-preserving
error-bounded quantisation, the CODEC.md token stream + FORMAT.md archive,
selective reconstruction and marching cubes -- all as hand-written CUDA
kernels in ``libchr.so`` (include/chr.h), driven through ctypes with torch
tensors as device buffers.  There is no CPU fallback.

The names below mirror ``isochr/__init__.py:9-86``.
"""

from .archive import (
    MODE_PAPER,
    MODE_STRICT,
    ArchiveRegion,
    CHRArchive,
    ReconstructionSet,
    RequestReport,
    build_chr,
    read_chr,
    request,
    request_device,
    stitch,
    stitch_device,
    write_chr,
)
from .blockcodec import CompressedBlock, compress, decompress, register_codec
from .field import Volume, load_raw, save_raw
from .index import BlockMeta, IsoIndex, Region, build_index, decompose, merge_regions
from .surface import (
    CaseField,
    TopologyReport,
    TriangleMesh,
    case_field,
    cell_case,
    export_obj,
    extract_device,
    marching_cubes,
    merge_meshes,
    verify_topology,
)

__version__ = "0.1.0"

__all__ = [
    "ArchiveRegion", "BlockMeta", "CHRArchive", "CaseField", "CompressedBlock", "IsoIndex", "MODE_PAPER",
    "MODE_STRICT", "ReconstructionSet", "Region", "RequestReport", "TopologyReport", "TriangleMesh", "Volume",
    "build_chr", "build_index", "case_field", "cell_case", "compress", "decompose", "decompress", "export_obj",
    "extract_device", "load_raw", "marching_cubes", "merge_meshes", "merge_regions", "read_chr",
    "register_codec", "request", "request_device", "save_raw", "stitch", "stitch_device", "verify_topology", "write_chr",
]
