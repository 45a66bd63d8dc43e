"""BASELINE configs at their own sizes, pinned to the REFERENCE's outputs.

tests/golden/golden_large.json holds, for c2 256^3 (all 9 (r, k) variants)
and c3 512^3, SHA-256s of what the reference package produced
(make_golden_large.py: build_chr -> write_chr, request(k) windows,
marching_cubes per region + merge_meshes; chr_archive.py:132-274,
isosurf.py:183-225) on inputs from the bit-reproducible CPU recipes
(tests/golden/recipes.py).  Each test regenerates its input, checks the
input's SHA-256 against the fixture FIRST, then compares the CUDA path's
outputs with the reference's -- bit-exact archive bytes, windows and mesh.

c2 runs through the drop-in API (build_chr -> serialize, request,
marching_cubes per region -> merge_meshes); c3 runs through chr_pipeline,
the one-call path bench.py times, and through the separate entry points.
"""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_05462_b200 as G  # noqa: E402
from paper_2408_05462_b200 import archive, device  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import recipes as R  # noqa: E402

with open(os.path.join(HERE, "golden", "golden_large.json")) as fh:
    LARGE = json.load(fh)["configs"]


def sha(b) -> str:
    return hashlib.sha256(b if isinstance(b, bytes) else np.ascontiguousarray(b).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def c2_field():
    f = R.c2_field()
    assert R.sha(f) == LARGE["c2_q50_r0.001"]["input_sha"], "c2 recipe is not bit-reproducible on this host"
    return f


@pytest.fixture(scope="module")
def c3_field():
    f = R.c3_field()
    assert R.sha(f) == LARGE["c3"]["input_sha"], "c3 recipe is not bit-reproducible on this host"
    return f


C2_NAMES = [f"c2_q{int(q)}_r{r:g}" for q in R.C2_Q for r in R.C2_R]


@pytest.mark.parametrize("name", C2_NAMES)
def test_c2_256_variants_match_reference(c2_field, name):
    ref = LARGE[name]
    dims, bs, k, r = tuple(ref["dims"]), ref["bs"], ref["k"], ref["r"]
    assert R.percentile(c2_field, float(name.split("_q")[1].split("_")[0])) == k
    vol = G.Volume(dims, values=torch.from_numpy(c2_field).cuda(), source_dtype="f32")
    arch = G.build_chr(vol, [k], bs, loose_fraction=r)
    blob = archive.serialize(arch)
    assert len(blob) == ref["archive_nbytes"] and sha(blob) == ref["archive_sha"]
    rs = G.request(arch, k)
    assert [reg.region_id for reg, _ in rs.regions] == ref["selected"]
    assert rs.report.bytes_touched == ref["bytes_touched"]
    h = hashlib.sha256()
    meshes = []
    for reg, win in rs.regions:
        h.update(np.asarray(win).ravel(order="F").tobytes())
        meshes.append(G.marching_cubes(win, vol.spacing, tuple(o * s for o, s in zip(reg.sample_origin, vol.spacing)),
                                       k))
    assert h.hexdigest() == ref["windows_sha"]
    m = G.merge_meshes(meshes)
    assert (m.num_triangles, m.num_vertices) == (ref["n_tri"], ref["n_vert"])
    assert sha(np.ascontiguousarray(m.vertices, dtype=np.float64)) == ref["verts_sha"]
    assert sha(np.ascontiguousarray(m.triangles, dtype=np.int32)) == ref["tris_sha"]


def test_c3_512_pipeline_matches_reference(c3_field):
    ref = LARGE["c3"]
    dims, bs, k, r = tuple(ref["dims"]), ref["bs"], ref["k"], ref["r"]
    vals = torch.from_numpy(c3_field).cuda()
    ws = device.Workspaces()
    p = device.pipeline(vals, dims, [k], bs, loose_fraction=r, ws=ws)
    torch.cuda.synchronize()
    blob = p.archive.cpu().numpy().tobytes()
    assert len(blob) == ref["archive_nbytes"] and sha(blob) == ref["archive_sha"]
    assert len(p.regions) == ref["n_regions"]
    assert np.bincount(p.regions["codec_id"], minlength=4).tolist() == ref["codecs"]
    assert p.n_selected == len(ref["selected"])
    assert p.windows.numel() == ref["window_samples"]
    assert sha(p.windows.cpu().numpy()) == ref["windows_sha"]
    assert (p.tris.shape[0], p.verts.shape[0]) == (ref["n_tri"], ref["n_vert"])
    assert sha(p.verts.cpu().numpy()) == ref["verts_sha"]
    assert sha(p.tris.cpu().numpy()) == ref["tris_sha"]


def test_c3_512_separate_calls_match_reference(c3_field):
    ref = LARGE["c3"]
    dims, bs, k, r = tuple(ref["dims"]), ref["bs"], ref["k"], ref["r"]
    vals = torch.from_numpy(c3_field).cuda()
    res = device.build_archive(vals, dims, [k], bs, loose_fraction=r)
    assert sha(res.blob[: res.nbytes].cpu().numpy().tobytes()) == ref["archive_sha"]
    regs = res.regions
    sel = np.nonzero((regs["mask"] & np.uint64(1)) != 0)[0]
    assert sel.tolist() == ref["selected"]
    mine = regs[sel]
    dec = device.dec_table(mine["block_offset"] + device.BLOCK_HEADER, mine["block_nbytes"] - device.BLOCK_HEADER,
                           mine["codec_id"], mine["extent"], mine["error_bound"], mine["payload_crc"])
    wins, offs, st = device.decode(res.blob, dec)  # unfused decode (no inside masks)
    assert not any(st)
    assert sha(wins.cpu().numpy()) == ref["windows_sha"]
    mct = device.mc_table(dec["out_offset"], mine["extent"], mine["origin"].astype(np.float64), (1.0, 1.0, 1.0))
    v, t, _, _ = device.marching(wins, mct, k)  # masks recomputed from the windows
    assert sha(v.cpu().numpy()) == ref["verts_sha"] and sha(t.cpu().numpy()) == ref["tris_sha"]


def test_bourke_case_codes_match_reference(golden):
    """Per-cell case IDs in mc_extract's Bourke corner order
    (kernels.py:448-470; the reference never returns them, so the fixture
    forms them from the reference's CORNER_OFFSETS exactly as
    _mc_vectorized does, isosurf.py:126-131) and in case_field's binary
    order (isosurf.py:77-88) -- chr_case_codes, both conventions."""
    with open(os.path.join(HERE, "golden", "golden_large.json")) as fh:
        bourke = json.load(fh)["bourke"]
    for seed in range(5):
        grid = torch.from_numpy(golden[f"mcrand{seed}_in"]).cuda()
        codes = device.case_codes(grid, (8, 7, 9), 0.1, binary=False).cpu().numpy()
        assert codes.tolist() == bourke[f"mcrand{seed}"], seed
        binary = device.case_codes(grid, (8, 7, 9), 0.1, binary=True).cpu().numpy()
        assert np.array_equal(binary, golden[f"mcrand{seed}_case"]), seed
