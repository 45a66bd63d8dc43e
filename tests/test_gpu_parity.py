"""Parity of the CUDA path (libchr.so through the C-ABI) with the oracle and
the reference's golden vectors.  Bit-exact for bytes / integers / case codes /
triangle indices; vertices and reconstructions are bit-exact too (the kernels
do the reference's f64 operations without FMA), which is stricter than the
north_star tolerances (1 ulp recon, 1e-5 * spacing vertices)."""

import hashlib
import struct

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_05462_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2408_05462_b200 import device, exceptions, synth  # noqa: E402
from paper_2408_05462_b200.blockcodec import CompressedBlock  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ----------------------------------------------------------------- blocks
def test_codec_md_worked_example(golden):
    g = golden["codec_example_in"].reshape((2, 2, 2), order="F")
    blk = G.compress(g, 0.25)
    assert blk.to_bytes() == golden["codec_example_block"].tobytes()
    assert blk.payload == bytes.fromhex("0500050908") and blk.checksum == 0xD71089FD
    assert np.array_equal(G.decompress(blk).ravel(order="F"), [1, 1, 1, 1, 1, 1, 3, 1])


def test_random_blocks_bit_exact(golden, golden_meta):
    for name, shape, e in golden_meta["rand_cases"]:
        g = golden[name + "_in"].reshape(shape, order="F")
        blk = G.compress(g, e)
        assert blk.to_bytes() == golden[name + "_block"].tobytes(), name
        out = G.decompress(CompressedBlock.from_bytes(golden[name + "_block"].tobytes()))
        assert np.array_equal(out.ravel(order="F"), golden[name + "_out"]), name


def test_verbatim_blocks(golden):
    g = golden["incompressible_in"].reshape((8, 8, 8), order="F")
    blk = G.compress(g, 1e-12)
    assert blk.codec_id == 0 and blk.to_bytes() == golden["incompressible_block"].tobytes()
    assert np.array_equal(G.decompress(blk), g)
    g32 = golden["f32src_in"].reshape((5, 4, 3), order="F")
    for tag, e in (("e0", 0.0), ("tiny", 1e-15), ("1e-2", 1e-2)):
        blk = G.compress(g32, e, source_dtype="f32")
        assert blk.to_bytes() == golden[f"f32src_block_{tag}"].tobytes(), tag


def test_lorenzo_seam_matches_reference(golden, golden_meta):
    for name, shape, e in golden_meta["rand_cases"]:
        flat = torch.from_numpy(golden[name + "_in"]).cuda()
        q, esc = device.lorenzo_encode(flat, *shape, e)
        assert np.array_equal(q.cpu().numpy(), golden[name + "_q"]), name
        assert np.array_equal(esc.cpu().numpy().astype(bool), golden[name + "_esc"]), name
    for e in (0.25, 0.001):
        q, esc = device.lorenzo_encode(torch.from_numpy(golden["tie_in"]).cuda(), 4, 2, 2, e)
        assert np.array_equal(q.cpu().numpy(), golden[f"tie_e{e}_q"])


def test_corrupt_and_unknown_codec():
    g = np.random.default_rng(1).normal(size=(9, 8, 7))
    blk = G.compress(g, 1e-3)
    for pos in (0, len(blk.payload) // 2, len(blk.payload) - 1):
        bad = bytearray(blk.payload)
        bad[pos] ^= 0x41
        with pytest.raises(exceptions.CorruptPayloadError):
            G.decompress(CompressedBlock(blk.codec_id, blk.dims, blk.error_bound, blk.source_dtype, bytes(bad),
                                         blk.checksum))
    with pytest.raises(exceptions.UnsupportedCodecError):
        G.decompress(CompressedBlock(77, blk.dims, blk.error_bound, blk.source_dtype, blk.payload, blk.checksum))


def test_crc_valid_malformed_streams(golden_meta):
    import zlib

    for hexbuf, n, msg in golden_meta["tok_errors"]:
        payload = bytes.fromhex(hexbuf)
        blk = CompressedBlock(1, (n, 1, 1), 0.5, "f64", payload, zlib.crc32(payload))
        with pytest.raises(exceptions.CorruptPayloadError):
            G.decompress(blk)


def test_token_stream_edge_runs(golden):
    # long runs (multi-byte run lengths) and extreme quanta through a full
    # compress/decompress: a field whose quanta are exactly tok_vals
    vals = golden["tok_vals"]
    n = vals.size
    q = vals.astype(np.int64)
    u = np.cumsum(q)  # 1D: x-only Lorenzo
    e = 0.5
    g = (u.astype(np.float64) * (2 * e)).reshape((n, 1, 1), order="F")
    if np.abs(u).max() <= 2**27:
        blk = G.compress(g, e)
        ref_cid, ref_payload = O.compress_flat(g.ravel(order="F"), (n, 1, 1), e, "f64")
        assert blk.payload == ref_payload and blk.codec_id == ref_cid
        assert np.array_equal(G.decompress(blk).ravel(order="F"), O.decompress_block(blk.to_bytes())[1])


# ----------------------------------------------------------------- MC
def test_mc_all_256_cases(golden):
    corners = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
    for code in range(256):
        g = np.zeros((2, 2, 2))
        for i, (ox, oy, oz) in enumerate(corners):
            g[ox, oy, oz] = 1.0 if (code >> i) & 1 else 0.0
        m = G.marching_cubes(g, k=0.5)
        assert np.array_equal(m.vertices, golden[f"mc256_{code}_v"]), code
        assert np.array_equal(m.triangles, golden[f"mc256_{code}_t"]), code


def test_mc_random_grids(golden):
    for seed in range(5):
        g = golden[f"mcrand{seed}_in"].reshape((8, 7, 9), order="F")
        m = G.marching_cubes(g, spacing=(1.0, 2.0, 0.5), origin=(3.0, -1.0, 2.5), k=0.1)
        assert np.array_equal(m.vertices, golden[f"mcrand{seed}_v"])
        assert np.array_equal(m.triangles, golden[f"mcrand{seed}_t"])
        assert np.array_equal(G.case_field(g, 0.1).codes, golden[f"mcrand{seed}_case"])
    g = golden["mcsmooth_in"].reshape((12, 11, 13), order="F")
    m = G.marching_cubes(g, k=0.0)
    assert np.array_equal(m.vertices, golden["mcsmooth_v"]) and np.array_equal(m.triangles, golden["mcsmooth_t"])


@pytest.mark.parametrize("shape", [(70, 9, 5), (5, 70, 9), (9, 5, 70), (130, 17, 19), (2, 2, 2), (66, 2, 3)])
def test_mc_shapes_vs_oracle(shape):
    g = np.random.default_rng(sum(shape)).normal(size=shape)
    m = G.marching_cubes(g, k=0.05)
    v, t = O.marching_cubes(g.ravel(order="F"), shape, 0.05)
    assert np.array_equal(m.vertices, v) and np.array_equal(m.triangles, t)


# ----------------------------------------------------------------- archives
@pytest.mark.parametrize("name", ["c1", "sphere", "smooth", "exactk", "oor", "c1_acc95", "sphere_paper",
                                  "smooth_paper80", "smooth_acc90", "exactk_paper"])
def test_golden_archives(golden, golden_meta, name, tmp_path):
    import warnings

    info = golden_meta["archive_" + name]
    vals = golden[info["input"] + "_in"]
    vol = G.Volume(tuple(info["dims"]), tuple(info["spacing"]), vals.astype(np.float64), info["dtype"])
    kw = dict(info["kw"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        arch = G.build_chr(vol, info["cands"], info["bs"], **kw)
    p = tmp_path / "a.chr"
    G.write_chr(arch, p)
    assert p.read_bytes() == golden[name + "_chr"].tobytes()
    back = G.read_chr(p)
    assert back == arch
    for k in arch.candidates:
        ref = info["requests"][repr(k)]
        rs = G.request(arch, k)
        assert [r.region_id for r, _ in rs.regions] == ref["regions"]
        assert [sha(np.asarray(w).ravel(order="F")) for _, w in rs.regions] == ref["recon_sha"]
        assert rs.report.bytes_touched == ref["bytes_touched"]
        # the same request decoded from the re-read (host) archive
        rs2 = G.request(back, k)
        assert all(np.array_equal(a, b) for (_, a), (_, b) in zip(rs.regions, rs2.regions))
        # stitch + verify_topology on the device
        st = G.stitch(rs, vol.dims)
        assert sha(st.ravel(order="F")) == ref["stitch_sha"]
        full = G.stitch_device(G.request(arch, k, drop_pruned=False), vol.dims)
        assert sha(full.permute(2, 1, 0).cpu().numpy()) == ref["full_stitch_sha"]
        for rep, want in ((G.verify_topology(vol.grid, full, k), ref["topo_full"]),
                          (G.verify_topology(vol.grid, st, k), ref["topo_pruned"])):
            assert [rep.preserved_fraction, rep.differing_cells, rep.total_cells,
                    list(rep.first_diff) if rep.first_diff else None] == want
        # the host-array path (windows re-uploaded, block size inferred)
        rs_host = G.ReconstructionSet(rs.regions, rs.report)
        assert sha(G.stitch(rs_host, vol.dims).ravel(order="F")) == ref["stitch_sha"]
        regs, wins, offs, _, _ = G.request_device(arch, k)
        v, t, nt, nv = G.extract_device(wins, regs, offs, vol.spacing, k) if regs else (None, None, [], [])
        if regs:
            assert sha(v.cpu().numpy()) == ref["merged_v_sha"] and sha(t.cpu().numpy()) == ref["merged_t_sha"]
            assert nt == ref["ntri"] and nv == ref["nvert"]


def _config_parity(name, n, quantile=None, r=None, accuracy=1.0, bound_mode="strict_vertices"):
    vals, dims, bs, cands, rr = synth.make_config(name, device="cuda", n=n, quantile=quantile, r=r)
    host = vals.cpu().numpy()
    res = device.build_archive(vals, dims, cands, bs, loose_fraction=rr, accuracy=accuracy, bound_mode=bound_mode)
    got = res.blob[: res.nbytes].cpu().numpy().tobytes()
    ref = O.build_chr(host.astype(np.float64), dims, cands, bs, source_dtype="f32", loose_fraction=rr, workers=8,
                      accuracy=accuracy, bound_mode=bound_mode)
    want = ref.to_bytes()
    assert len(got) == len(want)
    assert got == want
    return res, ref, dims, cands


@pytest.mark.parametrize("name,n", [("c1", 64), ("c2", 96), ("c3", 96), ("c4", 80), ("c5", 72)])
def test_config_recipes_archive_request_mc(name, n):
    res, ref, dims, cands = _config_parity(name, n)
    blob = ref.to_bytes()
    for k in cands[:3]:
        sel = O.request(ref, k)
        if not sel:
            continue
        desc = []
        table = _block_offsets(ref)
        for r, _ in sel:
            o = table[r["id"]]
            cid, ex, ey, ez, e, _, plen, crc = O.HEADER_STRUCT.unpack_from(blob, o)
            desc.append((o + 34, plen, cid, (ex, ey, ez), e, crc))
        wins, offs, status = device.decode(res.blob, desc)
        assert not any(status)
        host = wins.cpu().numpy()
        for (r, w), o in zip(sel, offs):
            assert np.array_equal(host[o:o + w.size], w)
        v, t, nt, nv = device.marching(wins, [(o, r["extent"], tuple(float(a) for a in r["origin"]), (1.0, 1.0, 1.0))
                                              for (r, _), o in zip(sel, offs)], k)
        rv, rt = O.extract_regions(sel, (1.0, 1.0, 1.0), k)
        assert np.array_equal(v.cpu().numpy(), rv) and np.array_equal(t.cpu().numpy(), rt)


def _block_offsets(ref):
    off = ref.header_table_nbytes()
    out = []
    for r in ref.regions:
        out.append(off)
        off += len(r["block"])
    return out


def test_stats_kernel_vs_oracle():
    vals, dims, bs, cands, _ = synth.make_config("c5", device="cuda", n=70)
    st, bad = device.stats(vals, dims, bs, cands)
    assert int(bad.item()) == -1
    st = st.cpu().numpy()
    host = vals.cpu().numpy().astype(np.float64)
    vmin, vmax = O.block_stats(host, dims, bs)
    assert np.array_equal(st[:, 0], vmin) and np.array_equal(st[:, 1], vmax)
    nbx, nby, nbz = O.block_grid_shape(dims, bs)
    L = O.lib()
    import ctypes

    for b in range(0, nbx * nby * nbz, 7):
        bz, rem = divmod(b, nbx * nby)
        by, bx = divmod(rem, nbx)
        w = [O._axis_window(c, bs, n) for c, n in zip((bx, by, bz), dims)]
        d = min(L.or_window_min_abs_distance(ctypes.c_void_p(host.ctypes.data), dims[0], dims[1], w[0][0], w[1][0],
                                             w[2][0], w[0][1], w[1][1], w[2][1], k) for k in cands)
        assert st[b, 2] == d


def test_nonfinite_detected():
    vals, dims, bs, cands, _ = synth.make_config("c1", device="cuda", n=32)
    vals = vals.clone()
    vals[12345] = float("nan")
    vals[20000] = float("inf")
    with pytest.raises(exceptions.NonFiniteSampleError) as ei:
        device.build_archive(vals, dims, cands, bs)
    assert ei.value.index == 12345


def test_crc_kernel_matches_zlib():
    import zlib

    rng = np.random.default_rng(3)
    for n in (1, 3, 4, 5, 1000, 65537, 3 * 2**20 + 7):
        a = rng.integers(0, 256, size=n, dtype=np.uint8)
        t = torch.from_numpy(a).cuda()
        assert device.crc32(t) == zlib.crc32(a.tobytes()), n
        if n > 8:
            assert device.crc32(t[3:], n - 3) == zlib.crc32(a[3:].tobytes())


def test_noncanonical_stream_uses_generic_path():
    """CRC-valid hand-made streams with non-minimal varints (e.g. 0x81 0x00 for
    the literal 1) must decode exactly like the reference (kernels.py:304-342);
    the fast canonical tokenizer hands such regions to the generic path."""
    import zlib

    g = np.random.default_rng(9).normal(size=(20, 9, 7))
    blk = G.compress(g, 0.05)
    assert blk.codec_id == 1
    tok = blk.payload
    # rewrite every single-byte literal 0x02..0x7f (end byte, after an end byte)
    # into a 2-byte non-minimal form b|0x80, 0x00
    out = bytearray()
    prev_end = True
    changed = 0
    for b in tok:
        if prev_end and 2 <= b < 0x80 and changed < 40:
            out += bytes([b | 0x80, 0x00])
            changed += 1
        else:
            out.append(b)
        prev_end = b < 0x80
    assert changed
    crafted = CompressedBlock(1, blk.dims, blk.error_bound, "f64", bytes(out), zlib.crc32(bytes(out)))
    want = O.decompress_block(crafted.to_bytes())[1]
    got = G.decompress(crafted).ravel(order="F")
    assert np.array_equal(got, want)
    assert np.array_equal(got, G.decompress(blk).ravel(order="F"))


@pytest.mark.parametrize("shape", [(64, 8, 8), (65, 9, 17), (130, 3, 2), (1, 1, 300), (200, 1, 1), (3, 70, 40),
                                   (33, 33, 300), (65, 161, 12), (300, 40, 9), (1, 300, 300), (97, 2, 500),
                                   (8200, 2, 2), (33, 200, 60), (64, 40, 100), (32, 32, 400)])
def test_decode_tile_shapes(shape):
    """Band tiles: whole planes, bands x chunks, warp-per-row prefixes, and
    rows too wide for a tile (generic path)."""
    g = np.random.default_rng(sum(shape) + 1).normal(size=shape).cumsum(axis=0)
    for e in (1e-3, 0.3):
        blk = G.compress(g, e)
        ref = O.decompress_block(blk.to_bytes())[1]
        assert np.array_equal(G.decompress(blk).ravel(order="F"), ref), (shape, e)


def test_decode_wide_quanta_use_int64_path():
    """A tile whose sum |q| >= 2^31: the int32 band pass flags its region and
    the int64 band pass (k_band<int64_t>) decodes it again (|u| < 2^27
    still, so no escapes)."""
    g = np.random.default_rng(5).uniform(-1e7, 1e7, size=(20, 20, 20))
    blk = G.compress(g, 0.5)
    assert blk.codec_id == 1
    ref = O.decompress_block(blk.to_bytes())[1]
    assert np.array_equal(G.decompress(blk).ravel(order="F"), ref)


@pytest.mark.parametrize("shape", [(40, 50, 60), (33, 33, 200), (130, 70, 3)])
def test_decode_escapes_in_band_tiles(shape):
    rng = np.random.default_rng(sum(shape))
    g = rng.normal(size=shape).cumsum(axis=2)
    idx = rng.choice(g.size, size=40, replace=False)
    g.reshape(-1)[idx] = rng.uniform(1e11, 1e12, size=40)
    blk = G.compress(g, 1e-2)
    assert blk.codec_id == 2
    ref = O.decompress_block(blk.to_bytes())[1]
    assert np.array_equal(G.decompress(blk).ravel(order="F"), ref)


@pytest.mark.parametrize("n,kind", [(1, "zeros"), (5, "zeros"), (300, "mixed"), (100000, "mixed"), (64, "ones"),
                                    (777, "wide"), (4096, "runs")])
def test_kernel_seam_rle_round_trip(n, kind):
    """rle_varint_encode / rle_varint_decode shims (kernels.py:292-296,
    407-411) against the oracle's restatement, byte for byte."""
    import torch

    rng = np.random.default_rng(n)
    if kind == "zeros":
        q = np.zeros(n, dtype=np.int64)
    elif kind == "ones":
        q = np.ones(n, dtype=np.int64)
    elif kind == "wide":
        q = rng.integers(-(1 << 30), (1 << 30) + 1, size=n).astype(np.int64)
    elif kind == "runs":
        q = np.where(rng.random(n) < 0.9, 0, rng.integers(-50, 50, size=n)).astype(np.int64)
    else:
        q = np.where(rng.random(n) < 0.4, 0, rng.integers(-70000, 70000, size=n)).astype(np.int64)
    want = O.rle_encode(q)
    got = device.rle_varint_encode(torch.from_numpy(q)).cpu().numpy()
    assert bytes(got) == bytes(want)
    back = device.rle_varint_decode(torch.from_numpy(np.frombuffer(bytes(want), dtype=np.uint8).copy()), n)
    assert np.array_equal(back.cpu().numpy(), q)


def test_kernel_seam_rle_decode_errors():
    import torch

    good = O.rle_encode(np.array([0, 0, 0, 5, -3], dtype=np.int64))
    with pytest.raises(ValueError):  # truncated varint
        device.rle_varint_decode(torch.tensor(list(good[:-1]) + [0x80], dtype=torch.uint8), 5)
    with pytest.raises(ValueError):  # wrong count
        device.rle_varint_decode(torch.tensor(list(good), dtype=torch.uint8), 6)
    with pytest.raises(ValueError):  # missing run length
        device.rle_varint_decode(torch.tensor([0x00], dtype=torch.uint8), 3)


@pytest.mark.parametrize("dims", [(9, 7, 5), (33, 33, 40), (1, 1, 1)])
def test_kernel_seam_lorenzo_decode(dims):
    import torch

    nx, ny, nz = dims
    g = np.random.default_rng(sum(dims)).normal(size=dims).cumsum(axis=1).ravel(order="F")
    e = 1e-2
    q, esc = O.lorenzo_encode(g, nx, ny, nz, e)
    escv = g[esc.astype(bool)]
    want = O.lorenzo_decode(q, esc, escv, e, nx, ny, nz)
    got = device.lorenzo_decode(torch.from_numpy(q), torch.from_numpy(esc.astype(np.uint8)),
                                torch.from_numpy(escv), e, nx, ny, nz)
    assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("name,n", [("c3", 96), ("c2", 80), ("c1", 64)])
def test_fused_request_extract_masks(name, n):
    """decode(..., iso=k) writes the windows' inside masks; marching cubes on
    those masks gives exactly the mesh of the unfused path, and every mask
    bit equals (window value >= k)."""
    import torch

    vals, dims, bs, cands, r = synth.make_config(name, device="cuda", n=n)
    res = device.build_archive(vals, dims, cands, bs, loose_fraction=r)
    regs = res.regions
    sel = regs[(regs["mask"] & np.uint64(1)) != 0]
    dec = device.dec_table(sel["block_offset"] + device.BLOCK_HEADER, sel["block_nbytes"] - device.BLOCK_HEADER,
                           sel["codec_id"], sel["extent"], sel["error_bound"], sel["payload_crc"])
    ws = device.Workspaces()
    k = cands[0]
    wins, offs, st = device.decode(res.blob, dec, ws=ws, iso=k)
    assert not any(st)
    masks = ws.get("decode_mask", 4, torch.int32).clone()
    w = wins.cpu().numpy()
    mw = masks.cpu().numpy().view(np.uint32)
    base = 0
    for i, (ex, ey, ez) in enumerate(sel["extent"].tolist()):
        pw = -(-(ex * ey) // 32)
        win = w[offs[i]: offs[i] + ex * ey * ez].reshape(ez, ex * ey)
        bits = np.unpackbits(mw[base: base + pw * ez].view(np.uint8), bitorder="little").reshape(ez, pw * 32)
        assert np.array_equal(bits[:, : ex * ey].astype(bool), win >= k), i
        base += pw * ez
    mct = device.mc_table(dec["out_offset"], sel["extent"], sel["origin"] * 1.0, (1.0, 1.0, 1.0))
    v0, t0, _, _ = device.marching(wins, mct, k)
    v1, t1, _, _ = device.marching(wins, mct, k, masks=masks)
    assert torch.equal(t0, t1) and torch.equal(v0, v1)


# ----------------------------------------------------------------- SURVEY 8(f2)
@pytest.mark.parametrize("name,n,acc,mode", [
    ("c1", 64, 0.95, "strict_vertices"), ("c2", 96, 0.9, "paper_edges"), ("c3", 96, 0.999, "strict_vertices"),
    ("c4", 80, 1.0, "paper_edges"), ("c5", 72, 0.5, "paper_edges"), ("c2", 96, 1e-9, "strict_vertices")])
def test_config_accuracy_and_paper_bounds(name, n, acc, mode):
    """accuracy < 1 / paper_edges archives byte-identical to the oracle's
    restatement of bound.region_bound (itself pinned by the reference's
    archives in tests/golden: c1_acc95, sphere_paper, smooth_paper80 ...)."""
    _config_parity(name, n, accuracy=acc, bound_mode=mode)


@pytest.mark.parametrize("mode", ["strict_vertices", "paper_edges"])
def test_select_distances_vs_numpy(mode):
    """n-th smallest distance of every (window, k) pair: windows larger than
    one histogram chunk, duplicated values (ties across the select digits),
    k on a sample, windows with no straddling edge (|D| = 0 -> -1)."""
    rng = np.random.default_rng(5)
    dims = (70, 50, 40)
    vol = np.round(rng.normal(size=dims[::-1]) * 8) / 8  # many exact ties
    vol[:, :, :10] = 3.0  # constant slab: no straddles
    flat = torch.from_numpy(vol.ravel()).cuda()
    wins, ks = [], []
    for o, e, k in [((0, 0, 0), (70, 50, 40), 0.0), ((0, 0, 0), (10, 50, 40), 0.0), ((5, 3, 2), (33, 17, 9), 0.25),
                    ((10, 0, 0), (60, 50, 40), 0.3), ((1, 1, 1), (1, 1, 1), 2.0), ((0, 0, 0), (2, 1, 1), -1.0),
                    ((20, 20, 20), (50, 30, 20), -0.0625)]:
        wins.append(list(o) + list(e))
        ks.append(k)
    for acc in (1.0, 0.9, 0.5, 0.01):
        got = device.select_distances(flat, dims, wins, ks, acc, mode)
        for (ox, oy, oz, ex, ey, ez), k, v in zip(wins, ks, got):
            w = vol[oz:oz + ez, oy:oy + ey, ox:ox + ex]
            d = O.window_distances(w, k, mode == "paper_edges")
            if d.size == 0:
                assert v == -1.0
                continue
            nn = O.select_index(d.size, acc)
            assert v == np.partition(d, nn - 1)[nn - 1], (acc, k)


# ----------------------------------------------------------------- SURVEY 8(f3)
@pytest.mark.parametrize("shape", [(2, 2, 2), (33, 9, 17), (70, 3, 40), (5, 130, 2), (64, 64, 33)])
def test_topology_compare_vs_oracle(shape):
    rng = np.random.default_rng(sum(shape))
    a = rng.normal(size=shape)
    b = a.copy()
    flip = rng.random(size=shape) < 0.01
    b[flip] = -b[flip]
    b.reshape(-1)[-1] = np.nan  # NaN is "outside" on both sides of >=
    want = O.verify_topology(a.ravel(order="F"), b.ravel(order="F"), shape, 0.0)
    for x, y in ((a, b), (torch.from_numpy(a).cuda().float(), torch.from_numpy(b).cuda())):
        rep = G.verify_topology(x, y, 0.0) if isinstance(x, np.ndarray) else None
        if rep is None:  # f32 original resident on the device vs f64 reconstruction
            rep = G.verify_topology(x, y, 0.0)
            want = O.verify_topology(a.astype(np.float32).astype(np.float64).ravel(order="F"),
                                     b.ravel(order="F"), shape, 0.0)
        assert [rep.preserved_fraction, rep.differing_cells, rep.total_cells,
                list(rep.first_diff) if rep.first_diff else None] == want


@pytest.mark.parametrize("name,n", [("c2", 96), ("c5", 72)])
def test_stitch_and_topology_at_config(name, n):
    """Full (unpruned) request stitched on the device == the oracle's
    stitch, and strict accuracy-1 archives preserve every cell case."""
    vals, dims, bs, cands, rr = synth.make_config(name, device="cuda", n=n)
    vol = G.Volume(dims, (1.0, 1.0, 1.0), vals.cpu().numpy().astype(np.float64), "f32")
    arch = G.build_chr(vol, cands, bs, loose_fraction=rr)
    ref = O.build_chr(vals.cpu().numpy().astype(np.float64), dims, cands, bs, loose_fraction=rr, workers=8)
    for k in cands[:2]:
        full = G.stitch_device(G.request(arch, k, drop_pruned=False), dims)
        want = O.stitch(O.request(ref, k, drop_pruned=False), dims)
        assert np.array_equal(full.permute(2, 1, 0).reshape(-1).cpu().numpy(), want)
        resident = vals.view(dims[2], dims[1], dims[0]).permute(2, 1, 0)  # f32, no widening copy
        rep = G.verify_topology(resident, full, k)
        assert rep.preserved_fraction == 1.0 and rep.differing_cells == 0


# ----------------------------------------------------------------- SURVEY 8(f1)
def _fix_crc(b: bytearray) -> bytes:
    import struct
    import zlib

    b[-4:] = struct.pack("<I", zlib.crc32(bytes(b[:-4])))
    return bytes(b)


def test_read_chr_errors_in_reference_order(golden, tmp_path):
    """read_chr validated on the device raises what chr_archive.read_chr
    raises (chr_archive.py:343-407; test_chr.py:90-137)."""
    import struct

    blob = golden["smooth_chr"].tobytes()
    p = tmp_path / "x.chr"
    cases = [
        (blob[:50], exceptions.ChecksumError, "too short"),
        (b"XHR1" + blob[4:], exceptions.BadMagicError, "bad magic"),
        (blob[:-1] + bytes([blob[-1] ^ 1]), exceptions.ChecksumError, "checksum mismatch"),
        (blob[:-100] + blob[-4:], exceptions.ChecksumError, "checksum mismatch"),
    ]
    b = bytearray(blob)
    b[4] = 99
    cases.append((_fix_crc(b), exceptions.VersionError, "unsupported CHR version 99"))
    m = struct.unpack_from("<I", blob, 63)[0]
    rec0 = 63 + 4 + 8 * m + 4
    b = bytearray(blob)  # region 0: payload offset far past the end
    struct.pack_into("<Q", b, rec0 + 69, len(blob))
    cases.append((_fix_crc(b), exceptions.ChecksumError, "region 0 payload exceeds file size"))
    b = bytearray(blob)  # region 0: table length one byte short of the block
    plen = struct.unpack_from("<Q", b, rec0 + 77)[0]
    struct.pack_into("<Q", b, rec0 + 77, plen - 1)
    cases.append((_fix_crc(b), exceptions.ChecksumError, f"(table {plen - 1}, block {plen})"))
    for data, exc, msg in cases:
        p.write_bytes(data)
        with pytest.raises(exc, match=msg.replace("(", r"\(").replace(")", r"\)")):
            G.read_chr(p)


def test_read_chr_single_byte_corruption(tmp_path):
    vol = G.Volume((10, 10, 10), (1.0, 1.0, 1.0), np.random.default_rng(3).normal(size=1000), "f64")
    arch = G.build_chr(vol, [0.0], 4)
    p = tmp_path / "c.chr"
    G.write_chr(arch, p)
    blob = p.read_bytes()
    rng = np.random.default_rng(0)
    positions = set(range(0, 64)) | {int(x) for x in rng.integers(0, len(blob), 150)} | set(range(len(blob) - 8, len(blob)))
    q = tmp_path / "bad.chr"
    for pos in sorted(positions):
        t = bytearray(blob)
        t[pos] ^= 1
        q.write_bytes(bytes(t))
        with pytest.raises(exceptions.IsochrError):
            G.read_chr(q)
    back = G.read_chr(p)
    assert back == arch
    # the device copy from read_chr serves the request without another upload
    assert back._device["blob"].is_cuda
    rs = G.request(back, 0.0)
    rs0 = G.request(arch, 0.0)
    assert all(np.array_equal(a, b) for (_, a), (_, b) in zip(rs.regions, rs0.regions))


def test_read_table_at_config_size(tmp_path):
    """The device parse of a device-built file matches the builder's table."""
    vals, dims, bs, cands, rr = synth.make_config("c5", device="cuda", n=96)
    res = device.build_archive(vals, dims, cands, bs, loose_fraction=rr)
    ft = device.read_table(res.blob, res.nbytes)
    info = ft.info[0]
    assert int(info["stored_crc"]) == int(info["actual_crc"]) and int(info["error"]) == 0
    assert list(ft.candidates) == list(cands)
    assert not ft.entries["status"].any()
    got, want = ft.regions, res.regions
    for f in ("lo", "hi", "origin", "extent", "mask", "error_bound", "codec_id", "payload_crc", "block_offset",
              "block_nbytes"):
        assert np.array_equal(got[f], want[f]), f


# ----------------------------------------------------------------- reentrancy (no global mutable state)
def test_concurrent_threads_on_separate_streams():
    """Two host threads, each on its own stream and workspaces, run compress ->
    request -> marching cubes at the same time (ctypes drops the GIL inside
    the library): results identical to a sequential run.  Exercises the
    thread-local transfer ring and decoder plan cache."""
    import threading

    jobs = []
    for name, n in (("c2", 80), ("c5", 64)):
        vals, dims, bs, cands, r = synth.make_config(name, device="cuda", n=n)
        jobs.append((vals, dims, bs, cands, r))

    def run(job, ws, stream):
        vals, dims, bs, cands, r = job
        with torch.cuda.stream(stream):
            res = device.build_archive(vals, dims, cands, bs, loose_fraction=r, ws=ws)
            regs = res.regions
            sel = regs[(regs["mask"] & np.uint64(1)) != 0]
            dec = device.dec_table(sel["block_offset"] + device.BLOCK_HEADER, sel["block_nbytes"] - device.BLOCK_HEADER,
                                   sel["codec_id"], sel["extent"], sel["error_bound"], sel["payload_crc"])
            wins, offs, st = device.decode(res.blob, dec, ws=ws, iso=cands[0])
            mct = device.mc_table(dec["out_offset"], sel["extent"], sel["origin"].astype(np.float64), (1.0, 1.0, 1.0))
            v, t, _, _ = device.marching(wins, mct, cands[0], ws=ws, masks=ws.get("decode_mask", 4, torch.int32))
            stream.synchronize()
            return (res.blob[: res.nbytes].cpu().numpy().tobytes(), sha(wins[: int(np.prod(sel["extent"].astype(np.int64), axis=1).sum())].cpu().numpy()),
                    sha(v.cpu().numpy()), sha(t.cpu().numpy()), list(st))

    want = [run(j, device.Workspaces(), torch.cuda.Stream()) for j in jobs]
    for _ in range(3):
        got = [None, None]

        def worker(i):
            got[i] = run(jobs[i], device.Workspaces(), torch.cuda.Stream())

        th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        assert got == want


def test_decode_returns_only_the_windows():
    """decode() hands back a view of exactly the decoded samples, never the
    (possibly much larger) workspace buffer: a small decompress after a big
    request must not copy the big buffer to the host."""
    ws = device.Workspaces()
    big = torch.zeros(1 << 24, dtype=torch.float64, device="cuda")
    ws._bufs["decode_out"] = big
    g = np.random.default_rng(3).normal(size=(6, 5, 4))
    b = G.compress(g, 0.01).to_bytes()
    blob = torch.from_numpy(np.frombuffer(b + bytes(16), dtype=np.uint8).copy()).cuda()
    cid, ex, ey, ez, e, _, plen, crc = struct.unpack_from("<B3IdBQI", b, 0)
    wins, offs, st = device.decode(blob, [(34, plen, cid, (ex, ey, ez), e, crc)], ws=ws)
    assert not any(st) and wins.numel() == 6 * 5 * 4 and wins.data_ptr() == big.data_ptr()


@pytest.mark.parametrize("case", ["dense64", "close_pairs", "wide_range", "on_samples"])
def test_stats_rows_many_candidates_exact(case):
    """The row-streaming stats kernel (f32, nx % 4 == 0) finds each sample's
    bracketing candidates from a bucket table: exact against the oracle for
    candidate sets that defeat the buckets (pairs closer than a bucket, two
    doubles rounding to one float, extreme ranges, candidates on samples)."""
    rng = np.random.default_rng(11)
    dims, bs = (64, 40, 36), 8
    vals = (rng.normal(size=dims[::-1]) * 3.0).astype(np.float32).reshape(-1)
    if case == "dense64":
        cands = np.sort(rng.normal(size=64) * 3.0)
    elif case == "close_pairs":
        base = np.sort(rng.normal(size=20) * 3.0)
        f = np.float32(1.2345)
        cands = np.concatenate([base, [float(f), float(f) + 1e-12, float(f) + 2e-12, 0.5, 0.5 + 1e-9]])
    elif case == "wide_range":
        cands = np.array([-1e30, -1e3, -1.0, -1e-7, 1e-30, 0.3, 2.0, 1e5, 1e30])
    else:
        cands = np.sort(vals[rng.choice(vals.size, size=24, replace=False)].astype(np.float64))
    cands = np.unique(cands)
    st, bad = device.stats(torch.from_numpy(vals).cuda(), dims, bs, list(cands))
    st = st.cpu().numpy()
    host = vals.astype(np.float64)
    nbx, nby, nbz = O.block_grid_shape(dims, bs)
    L = O.lib()
    import ctypes

    for b in range(nbx * nby * nbz):
        bz, rem = divmod(b, nbx * nby)
        by, bx = divmod(rem, nbx)
        w = [O._axis_window(c, bs, n) for c, n in zip((bx, by, bz), dims)]
        d = min(L.or_window_min_abs_distance(ctypes.c_void_p(host.ctypes.data), dims[0], dims[1], w[0][0], w[1][0],
                                             w[2][0], w[0][1], w[1][1], w[2][1], float(k)) for k in cands)
        assert st[b, 2] == d, (case, b)


@pytest.mark.parametrize("name,n", [("c1", 64), ("c3", 96), ("c5", 72)])
def test_pipeline_one_call_matches_separate_calls(name, n):
    """chr_pipeline (stats -> plan -> compress -> request -> decode -> MC in
    one call) produces the same archive, windows and mesh as the separate
    entry points; the after-compress hook sees the finished archive."""
    vals, dims, bs, cands, r = synth.make_config(name, device="cuda", n=n)
    seen = {}
    ws = device.Workspaces()
    p = device.pipeline(vals, dims, cands, bs, loose_fraction=r, ws=ws,
                        after_compress=lambda a: seen.setdefault("a", a.cpu().numpy().tobytes()))
    ref = device.build_archive(vals, dims, cands, bs, loose_fraction=r)
    want = ref.blob[: ref.nbytes].cpu().numpy().tobytes()
    assert p.archive.cpu().numpy().tobytes() == want and seen["a"] == want
    assert np.array_equal(p.regions.view(np.uint8), ref.regions.view(np.uint8))
    dec, mct, sel_idx, total = device.request_tables(ref.regions, 0)
    wins, offs, st = device.decode(ref.blob, dec, iso=cands[0])
    assert not any(st) and p.n_selected == len(sel_idx)
    assert torch.equal(p.windows, wins)
    v, t, _, _ = device.marching(wins, mct, cands[0])
    assert torch.equal(p.verts, v) and torch.equal(p.tris, t)
    # a second call reuses the negotiated buffers
    p2 = device.pipeline(vals, dims, cands, bs, loose_fraction=r, ws=ws)
    assert torch.equal(p2.tris, t)


def test_decode_payload_crc_mismatch_per_region():
    """Payload CRCs are checked on a side stream while the band decoder runs:
    a region whose payload bytes were flipped reports the checksum status
    (before any token error, as decompress() checks the CRC first,
    codec.py:220-226), an unknown codec with a bad CRC reports the checksum
    too, and every intact region still decodes bit-identically to the oracle."""
    import torch

    vals, dims, bs, cands, r = synth.make_config("c2", device="cuda", n=160)
    res = device.build_archive(vals, dims, cands, bs, loose_fraction=r)
    regs = res.regions
    host = res.blob[: res.nbytes].cpu().numpy().tobytes()
    sel = regs[(regs["mask"] & np.uint64(1)) != 0]
    assert len(sel) >= 6, len(sel)
    codec = sel["codec_id"].copy()
    blob = bytearray(host)
    hit = [1, 3, len(sel) - 1]  # flip a payload byte in these regions
    for j in hit:
        o = int(sel["block_offset"][j]) + device.BLOCK_HEADER
        ln = int(sel["block_nbytes"][j]) - device.BLOCK_HEADER
        blob[o + ln // 2] ^= 0x5A
    codec[4] = 77  # unknown codec, intact CRC
    dev = torch.tensor(np.frombuffer(bytes(blob), np.uint8), device="cuda")
    dec = device.dec_table(sel["block_offset"] + device.BLOCK_HEADER, sel["block_nbytes"] - device.BLOCK_HEADER,
                           codec, sel["extent"], sel["error_bound"], sel["payload_crc"])
    for iso in (None, cands[0]):
        wins, offs, st = device.decode(dev, dec, iso=iso)
        w = wins.cpu().numpy()
        for j in range(len(sel)):
            if j in hit:
                assert st[j] == 7, (j, st[j])  # CHR_DEC_CHECKSUM
            elif j == 4:
                assert st[j] == 10, st[j]  # unknown codec
            else:
                assert st[j] == 0, (j, st[j])
                _, ref = O.decompress_block(host, int(sel["block_offset"][j]))
                assert np.array_equal(w[int(offs[j]): int(offs[j]) + ref.size], ref), j
    # an unknown codec whose payload CRC is also wrong: the checksum wins
    codec2 = sel["codec_id"].copy()
    codec2[hit[0]] = 77
    dec2 = device.dec_table(sel["block_offset"] + device.BLOCK_HEADER, sel["block_nbytes"] - device.BLOCK_HEADER,
                            codec2, sel["extent"], sel["error_bound"], sel["payload_crc"])
    _, _, st2 = device.decode(dev, dec2)
    assert st2[hit[0]] == 7
