"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_codec_md_worked_example(golden):
    # CODEC.md:64-90: 2x2x2 at bound 0.25 -> tokens 05 00 05 09 08, crc 0xd71089fd
    flat = golden["codec_example_in"]
    cid, payload = O.compress_flat(flat, (2, 2, 2), 0.25, "f64")
    blk = O.block_bytes(cid, (2, 2, 2), 0.25, "f64", payload)
    assert payload == bytes.fromhex("0500050908")
    assert O.crc32(payload) == 0xD71089FD
    assert blk == golden["codec_example_block"].tobytes()


@pytest.mark.parametrize("e", [0.25, 0.001])
def test_ties_round_to_odd(golden, e):
    q, esc = O.lorenzo_encode(golden["tie_in"], 4, 2, 2, e)
    assert np.array_equal(q, golden[f"tie_e{e}_q"])
    assert np.array_equal(esc, golden[f"tie_e{e}_esc"])


def test_random_blocks_bit_exact(golden, golden_meta):
    saw = set()
    for name, shape, e in golden_meta["rand_cases"]:
        flat = golden[name + "_in"]
        q, esc = O.lorenzo_encode(flat, *shape, e)
        assert np.array_equal(q, golden[name + "_q"]), name
        assert np.array_equal(esc, golden[name + "_esc"]), name
        cid, payload = O.compress_flat(flat, tuple(shape), e, "f64")
        blk = O.block_bytes(cid, tuple(shape), e, "f64", payload)
        assert blk == golden[name + "_block"].tobytes(), name
        saw.add(cid)
        dims, out = O.decompress_block(blk)
        assert np.array_equal(out, golden[name + "_out"]), name
    assert {1, 2} <= saw


def test_verbatim_paths(golden):
    g = golden["incompressible_in"]
    cid, payload = O.compress_flat(g, (8, 8, 8), 1e-12, "f64")
    assert cid == 0
    assert O.block_bytes(cid, (8, 8, 8), 1e-12, "f64", payload) == golden["incompressible_block"].tobytes()
    g32 = golden["f32src_in"]
    for tag, e in (("e0", 0.0), ("tiny", 1e-15), ("1e-2", 1e-2)):
        cid, payload = O.compress_flat(g32, (5, 4, 3), e, "f32")
        assert O.block_bytes(cid, (5, 4, 3), e, "f32", payload) == golden[f"f32src_block_{tag}"].tobytes()


def test_token_codec(golden, golden_meta):
    vals = golden["tok_vals"]
    assert np.array_equal(O.rle_encode(vals), golden["tok_bytes"])
    back, err = O.rle_decode(golden["tok_bytes"], vals.size)
    assert err == 0 and np.array_equal(back, vals)
    for hexbuf, n, msg in golden_meta["tok_errors"]:
        _, err = O.rle_decode(np.frombuffer(bytes.fromhex(hexbuf), np.uint8), n)
        assert O.RLE_ERRORS.get(err, "") == msg, (hexbuf, n)


def test_mc_all_256_cases(golden):
    for code in range(256):
        g = np.zeros((2, 2, 2))
        for i, (ox, oy, oz) in enumerate([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
                                          (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]):
            g[ox, oy, oz] = 1.0 if (code >> i) & 1 else 0.0
        v, t = O.marching_cubes(g.ravel(order="F"), (2, 2, 2), 0.5)
        assert np.array_equal(v, golden[f"mc256_{code}_v"]), code
        assert np.array_equal(t, golden[f"mc256_{code}_t"]), code


def test_mc_random_grids(golden):
    for seed in range(5):
        g = golden[f"mcrand{seed}_in"]
        v, t = O.marching_cubes(g, (8, 7, 9), 0.1, (1.0, 2.0, 0.5), (3.0, -1.0, 2.5))
        assert np.array_equal(v, golden[f"mcrand{seed}_v"])
        assert np.array_equal(t, golden[f"mcrand{seed}_t"])
        assert np.array_equal(O.case_field(g, (8, 7, 9), 0.1), golden[f"mcrand{seed}_case"])
        _, _, bourke = O.mc_lattice(g, (8, 7, 9), 0.1)
        assert np.array_equal(O.bourke_to_binary(bourke), golden[f"mcrand{seed}_case"])
    v, t = O.marching_cubes(golden["mcsmooth_in"], (12, 11, 13), 0.0)
    assert np.array_equal(v, golden["mcsmooth_v"]) and np.array_equal(t, golden["mcsmooth_t"])


@pytest.mark.parametrize("name", ["c1", "sphere", "smooth", "exactk", "oor", "c1_acc95", "sphere_paper",
                                  "smooth_paper80", "smooth_acc90", "exactk_paper"])
def test_archives_byte_identical(golden, golden_meta, name):
    info = golden_meta["archive_" + name]
    vals = golden[info["input"] + "_in"].astype(np.float64)
    kw = dict(info["kw"])
    arch = O.build_chr(vals, tuple(info["dims"]), info["cands"], info["bs"], tuple(info["spacing"]),
                       info["dtype"], loose_fraction=kw.get("loose_fraction", 0.01),
                       out_of_range=kw.get("out_of_range", "error"), accuracy=kw.get("accuracy", 1.0),
                       bound_mode=kw.get("bound_mode", "strict_vertices"))
    blob = arch.to_bytes()
    assert blob == golden[name + "_chr"].tobytes()
    for k in arch.candidates:
        ref = info["requests"][repr(k)]
        sel = O.request(arch, k)
        assert [r["id"] for r, _ in sel] == ref["regions"]
        assert [sha(w) for _, w in sel] == ref["recon_sha"]
        assert O.bytes_touched(arch, sel) == ref["bytes_touched"]
        v, t = O.extract_regions(sel, tuple(info["spacing"]), k)
        assert sha(v) == ref["merged_v_sha"] and sha(t) == ref["merged_t_sha"]
        # stitch + verify_topology
        dims = tuple(info["dims"])
        st = O.stitch(sel, dims)
        assert sha(st) == ref["stitch_sha"]
        full = O.stitch(O.request(arch, k, drop_pruned=False), dims)
        assert sha(full) == ref["full_stitch_sha"]
        assert O.verify_topology(vals, full, dims, k) == ref["topo_full"]
        assert O.verify_topology(vals, st, dims, k) == ref["topo_pruned"]
