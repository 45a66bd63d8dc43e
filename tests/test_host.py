"""CPU-only checks of the host side: the C-ABI library loads and exports every
symbol include/chr.h declares, the host C++ planner (chr_plan) reproduces the
reference's regions and strict bounds (through the pinned oracle), CRC
combine algebra, multi-rank placement over gloo.  No CUDA compute here."""

import ctypes
import os
import re
import zlib

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2408_05462_b200 import _abi

    return _abi, _abi.lib()


def test_library_exports_every_declared_symbol():
    _abi, L = _lib()
    hdr = open(os.path.join(ROOT, "include", "chr.h")).read()
    names = set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(chr_\w+)\s*\(", hdr, flags=re.M))
    assert len(names) >= 20
    for n in sorted(names):
        assert hasattr(L, n), n
    assert set(_abi.EXPORTS) <= names
    assert L.chr_abi_version() == 1
    assert L.chr_status_string(3) == b"corrupt payload"


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2408_05462_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f), encoding="utf-8", errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "chr_oracle" not in txt, f


def _block_stats_numpy(vals, dims, bs, cands):
    from oracle import oracle as O

    vmin, vmax = O.block_stats(vals, dims, bs)
    nbx, nby, nbz = O.block_grid_shape(dims, bs)
    L = O.lib()
    dmin = np.empty(vmin.size)
    for b in range(vmin.size):
        bz, rem = divmod(b, nbx * nby)
        by, bx = divmod(rem, nbx)
        w = [O._axis_window(c, bs, n) for c, n in zip((bx, by, bz), dims)]
        dmin[b] = min(L.or_window_min_abs_distance(ctypes.c_void_p(vals.ctypes.data), dims[0], dims[1],
                                                   w[0][0], w[1][0], w[2][0], w[0][1], w[1][1], w[2][1], float(k))
                      for k in cands)
    return np.stack([vmin, vmax, dmin], axis=1)


@pytest.mark.parametrize("name", ["c1", "sphere", "smooth", "exactk", "oor"])
def test_plan_matches_reference_regions_and_bounds(golden, golden_meta, name):
    """chr_plan (greedy merge + closed-form strict bound from per-block dmin)
    == the reference's merge_regions + region_bound (via the pinned oracle)."""
    from oracle import oracle as O
    from paper_2408_05462_b200 import device

    info = golden_meta["archive_" + name]
    vals = np.ascontiguousarray(golden[name + "_in"], dtype=np.float64)
    dims, bs, cands = tuple(info["dims"]), info["bs"], info["cands"]
    kw = info["kw"]
    lf = kw.get("loose_fraction", 0.01)
    arch = O.build_chr(vals, dims, cands, bs, tuple(info["spacing"]), info["dtype"], loose_fraction=lf,
                       out_of_range=kw.get("out_of_range", "error"))
    st = _block_stats_numpy(vals, dims, bs, cands)
    regs = device.plan(st, dims, bs, cands, arch.value_range[0], arch.value_range[1], lf)
    recs = device.region_records(regs)
    assert len(recs) == len(arch.regions)
    for r, o in zip(recs, arch.regions):
        assert (r["lo"], r["hi"], r["origin"], r["extent"]) == (o["lo"], o["hi"], o["origin"], o["extent"])
        assert r["mask"] == o["mask"]
        assert r["e"] == o["e"], (r["e"], o["e"])  # bit-exact closed form


def test_plan_closed_form_on_random_fields():
    from oracle import oracle as O
    from paper_2408_05462_b200 import device

    rng = np.random.default_rng(5)
    for trial in range(6):
        dims = tuple(int(d) for d in rng.integers(9, 30, size=3))
        bs = int(rng.integers(3, 9))
        vals = rng.normal(size=dims[0] * dims[1] * dims[2]).cumsum().astype(np.float32).astype(np.float64)
        m = int(rng.integers(1, 5))
        cands = sorted(set(float(v) for v in rng.choice(vals, size=m, replace=False)))
        if trial % 2:  # candidates off the samples
            cands = [c + 1e-3 for c in cands]
        arch = O.build_chr(vals, dims, cands, bs, source_dtype="f32", loose_fraction=0.02, out_of_range="warn")
        st = _block_stats_numpy(vals, dims, bs, cands)
        recs = device.region_records(device.plan(st, dims, bs, cands, *arch.value_range, 0.02))
        assert [r["e"] for r in recs] == [o["e"] for o in arch.regions]
        assert [r["mask"] for r in recs] == [o["mask"] for o in arch.regions]


def test_plan_rejects_bad_candidates():
    from paper_2408_05462_b200 import device, exceptions

    st = np.zeros((8, 3))
    with pytest.raises(exceptions.ParameterError):
        device.plan(st, (5, 5, 5), 2, [1.0, 1.0], 0.0, 1.0)
    with pytest.raises(exceptions.ParameterError):
        device.plan(st, (5, 5, 5), 2, [float("nan")], 0.0, 1.0)


def test_crc32_combine_matches_zlib():
    _abi, L = _lib()
    rng = np.random.default_rng(0)
    for _ in range(20):
        a = rng.integers(0, 256, size=int(rng.integers(0, 300)), dtype=np.uint8).tobytes()
        b = rng.integers(0, 256, size=int(rng.integers(0, 5000)), dtype=np.uint8).tobytes()
        assert L.chr_crc32_combine(zlib.crc32(a), zlib.crc32(b), len(b)) == zlib.crc32(a + b)


def test_block_header_roundtrip(golden):
    from paper_2408_05462_b200.blockcodec import CompressedBlock

    raw = golden["codec_example_block"].tobytes()
    blk = CompressedBlock.from_bytes(raw)
    assert blk.to_bytes() == raw and blk.nbytes == len(raw) and blk.codec_id == 1
    assert blk.checksum == 0xD71089FD


def _gloo_worker(rank, world, port, sizes, out):
    import torch.distributed as dist

    from paper_2408_05462_b200 import multi

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = multi.place(*sizes[rank], device="cpu")
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_multi_rank_placement_gloo():
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    sizes = [(1000, 10, 7), (250, 3, 2)]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gloo_worker, args=(2, port, sizes, out), nprocs=2, join=True)
    assert out[0]["archive_offset"] == 0 and out[1]["archive_offset"] == 1000
    assert out[1]["tri_offset"] == 10 and out[1]["vert_offset"] == 7
    assert out[0]["archive_total"] == 1250 and out[1]["tri_total"] == 13


@pytest.mark.parametrize("nz,bs,world", [(512, 32, 8), (65, 16, 2), (97, 32, 3), (33, 32, 4), (1024, 32, 7), (17, 8, 1)])
def test_slab_geometry_partitions_planes_and_blocks(nz, bs, world):
    """z-slabs: encode planes partition [0, nz); each rank holds
    the plane below its first (Lorenzo z-1) and its blocks' ghost plane; the
    block layers partition the block grid."""
    from paper_2408_05462_b200 import multi

    nbz = max(1, -(-(nz - 1) // bs))
    covered, layers = [], []
    for r in range(world):
        s = multi.slab_of(nz, bs, world, r)
        if s.zs == s.ze:
            continue
        covered.append((s.zs, s.ze))
        layers.extend(range(s.bz0, s.bz1))
        assert s.z_base <= max(s.zs - 1, 0) and s.ze <= s.z_base + s.nz_local
        assert s.z_base + s.nz_local - 1 == min(s.bz1 * bs, nz - 1)  # ghost plane of the last layer
        assert s.nz_stats - 1 == min(s.bz1 * bs, nz - 1) - s.zs
    covered.sort()
    assert covered[0][0] == 0 and covered[-1][1] == nz
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
    assert layers == list(range(nbz))


def test_request_tables_match_selection():
    """chr_request_tables (host C) == the numpy selection + table build of
    request(k) (chr_archive.py:249-259)."""
    from paper_2408_05462_b200 import _abi, device

    rng = np.random.default_rng(4)
    n = 57
    regs = np.zeros(n, dtype=_abi.REGION_DT)
    regs["extent"] = rng.integers(2, 40, size=(n, 3))
    regs["origin"] = rng.integers(0, 500, size=(n, 3))
    regs["mask"] = rng.integers(0, 8, size=n).astype(np.uint64)
    regs["block_offset"] = np.cumsum(rng.integers(40, 4000, size=n))
    regs["block_nbytes"] = rng.integers(34, 3000, size=n)
    regs["codec_id"] = rng.integers(0, 4, size=n)
    regs["error_bound"] = rng.random(n)
    regs["payload_crc"] = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    spacing = (0.5, 2.0, 1.25)
    for ki in (-1, 0, 1, 2):
        dec, mct, sel_idx, total = device.request_tables(regs, ki, spacing)
        want = np.arange(n) if ki < 0 else np.nonzero((regs["mask"] >> np.uint64(ki)) & np.uint64(1))[0]
        assert np.array_equal(sel_idx, want)
        s = regs[want]
        ref = device.dec_table(s["block_offset"] + device.BLOCK_HEADER, s["block_nbytes"] - device.BLOCK_HEADER,
                               s["codec_id"], s["extent"], s["error_bound"], s["payload_crc"])
        assert dec.tobytes() == ref.tobytes()
        mref = device.mc_table(ref["out_offset"], s["extent"], s["origin"] * np.asarray(spacing), spacing)
        assert mct.tobytes() == mref.tobytes()
        assert total == int(np.prod(s["extent"].astype(np.int64), axis=1).sum())
