"""Generate golden vectors by running the REFERENCE itself (isochr).

Run in the build container, where the reference is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes tests/golden/golden.npz (+ golden_meta.json).  The fixtures pin the
oracle (oracle/) and, through it, the CUDA path.  Inputs are stored with the
outputs (no generator has to be reproduced on another machine).  Nothing on
the GPU box reads /root/reference: only these committed files travel.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, os.environ.get("ISOCHR_SRC", "/root/reference/pkg/src"))

import isochr  # noqa: E402
from isochr import kernels  # noqa: E402
from isochr.codec import compress  # noqa: E402
from isochr.isosurf import case_field, marching_cubes  # noqa: E402
from isochr.mc_tables import CORNER_OFFSETS  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
G: dict[str, np.ndarray] = {}
META: dict[str, object] = {}


def put(name, arr):
    G[name] = np.asarray(arr)


def put_bytes(name, b: bytes):
    G[name] = np.frombuffer(b, dtype=np.uint8).copy()


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --- 1. CODEC.md:64-90 worked example --------------------------------------
ex = np.array([1.0, 1.2, 0.9, 1.1, 1.0, 1.0, 3.0, 1.05]).reshape((2, 2, 2), order="F")
put("codec_example_in", ex.ravel(order="F"))
put_bytes("codec_example_block", compress(ex, 0.25).to_bytes())

# --- 2. kernel seam: quantiser ties, escapes, random windows ----------------
# ties: v = (j + 1/2) * 2e exactly -> the ties-to-odd rule (kernels.py:62-68)
tie = (np.arange(-6, 6, dtype=np.float64) + 0.5) * 0.5
tie = np.concatenate([tie, [0.375, 0.125, -0.375, 1e-3 * 187.5 * 2]])
tie3 = np.resize(tie, 4 * 2 * 2)
for e in (0.25, 0.001):
    q, esc = kernels.lorenzo_encode(tie3, 4, 2, 2, e)
    put(f"tie_e{e}_q", q)
    put(f"tie_e{e}_esc", esc)
put("tie_in", tie3)

cases = []
for seed in range(6):
    rng = np.random.default_rng(seed)
    shape = tuple(int(s) for s in rng.integers(2, 11, size=3))
    g = rng.normal(size=shape) * (10.0 ** rng.integers(-3, 4))
    if seed == 4:  # extreme outliers escape on magnitude
        flat = g.reshape(-1)
        flat[rng.choice(flat.size, size=5, replace=False)] = 1e18
    for frac in (1e-1, 1e-3, 1e-6):
        e = float(frac * (g.max() - g.min()))
        q, esc = kernels.lorenzo_encode(g.ravel(order="F"), *shape, e)
        blk = compress(g, e)
        name = f"rand{seed}_f{frac}"
        put(name + "_in", g.ravel(order="F"))
        put(name + "_q", q)
        put(name + "_esc", esc)
        put_bytes(name + "_block", blk.to_bytes())
        put(name + "_out", isochr.decompress(blk).ravel(order="F"))
        cases.append([name, list(shape), e])
# codec 2: outliers that overflow the lattice, and an f64 tie that lands
# 4 ulp outside the bound, at a fixed small bound
rng = np.random.default_rng(11)
g = rng.normal(size=(8, 8, 8))
flat = g.reshape(-1)
flat[rng.choice(flat.size, size=5, replace=False)] = 1e18
g.reshape(-1)[7] = 0.375
for name, e in (("esc_outlier", 1e-3),):
    blk = compress(g, e)
    assert blk.codec_id == 2
    q, esc = kernels.lorenzo_encode(g.ravel(order="F"), 8, 8, 8, e)
    put(name + "_in", g.ravel(order="F"))
    put(name + "_q", q)
    put(name + "_esc", esc)
    put_bytes(name + "_block", blk.to_bytes())
    put(name + "_out", isochr.decompress(blk).ravel(order="F"))
    cases.append([name, [8, 8, 8], e])
META["rand_cases"] = cases

# incompressible -> verbatim (codec 0) and f32-source verbatim (codec 3)
rng = np.random.default_rng(99)
g = rng.uniform(-1e9, 1e9, size=(8, 8, 8))
put("incompressible_in", g.ravel(order="F"))
put_bytes("incompressible_block", compress(g, 1e-12).to_bytes())
g32 = rng.normal(size=(5, 4, 3)).astype("<f4").astype(np.float64)
put("f32src_in", g32.ravel(order="F"))
put_bytes("f32src_block_e0", compress(g32, 0.0, source_dtype="f32").to_bytes())
put_bytes("f32src_block_tiny", compress(g32, 1e-15, source_dtype="f32").to_bytes())
put_bytes("f32src_block_1e-2", compress(g32, 1e-2, source_dtype="f32").to_bytes())

# --- 3. token codec ----------------------------------------------------------
rng = np.random.default_rng(7)
tok_vals = np.concatenate([
    np.zeros(1), [5, -5, 0, 0, 0], np.zeros(200), [2**30, -(2**30), 63, -64, 64],
    np.zeros(20000), [1], np.zeros(1), [-1], rng.integers(-300, 300, size=500),
    np.zeros(2**14 + 3), [7], np.zeros(3),
]).astype(np.int64)
put("tok_vals", tok_vals)
put("tok_bytes", kernels.rle_varint_encode(tok_vals))
bad = []
for buf, n in [
    (b"", 1), (b"\x85", 1), (b"\x80\x80\x80\x80\x80\x01", 1), (b"\x00", 3),
    (b"\x00\x00", 3), (b"\x00\x05", 3), (b"\x02\x02", 1), (b"\x02", 2),
]:
    try:
        kernels.rle_varint_decode(np.frombuffer(buf, np.uint8).copy(), n)
        msg = ""
    except ValueError as exc:
        msg = str(exc)
    bad.append([buf.hex(), n, msg])
META["tok_errors"] = bad

# --- 4. marching cubes -------------------------------------------------------
mc_cases = []
for code in range(256):
    g = np.zeros((2, 2, 2))
    for i in range(8):
        ox, oy, oz = CORNER_OFFSETS[i]
        g[ox, oy, oz] = 1.0 if (code >> i) & 1 else 0.0
    m = marching_cubes(g, k=0.5)
    put(f"mc256_{code}_v", m.vertices)
    put(f"mc256_{code}_t", m.triangles)
for seed in range(5):
    g = np.random.default_rng(seed).normal(size=(8, 7, 9))
    m = marching_cubes(g, k=0.1, spacing=(1.0, 2.0, 0.5), origin=(3.0, -1.0, 2.5))
    put(f"mcrand{seed}_in", g.ravel(order="F"))
    put(f"mcrand{seed}_v", m.vertices)
    put(f"mcrand{seed}_t", m.triangles)
    put(f"mcrand{seed}_case", case_field(g, 0.1).codes)
    mc_cases.append(seed)
g = isochr.gen_smooth_random((12, 11, 13), seed=21, num_modes=3).grid
m = marching_cubes(g, k=0.0)
put("mcsmooth_in", g.ravel(order="F"))
put("mcsmooth_v", m.vertices)
put("mcsmooth_t", m.triangles)

# --- 5. whole archives -------------------------------------------------------


def archive_case(name, vol, cands, bs, input_from=None, **kw):
    arch = isochr.build_chr(vol, cands, block_size=bs, **kw)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "a.chr")
        isochr.write_chr(arch, p)
        blob = open(p, "rb").read()
    if input_from is None:  # else: the same samples as archive ``input_from``
        put(name + "_in", vol.values.astype(np.float32) if vol.source_dtype == "f32" else vol.values)
    put_bytes(name + "_chr", blob)
    info = {
        "input": input_from or name,
        "dims": list(vol.dims), "spacing": list(vol.spacing), "dtype": vol.source_dtype,
        "cands": list(arch.candidates), "bs": bs, "kw": kw,
        "codecs": [r.block.codec_id for r in arch.regions],
        "requests": {},
    }
    for k in arch.candidates:
        rs = isochr.request(arch, k, drop_pruned=True)
        meshes = []
        for region, samples in rs.regions:
            mm = marching_cubes(samples, spacing=vol.spacing,
                                origin=tuple(o * s for o, s in zip(region.sample_origin, vol.spacing)),
                                k=k)
            meshes.append(mm)
        merged = isochr.merge_meshes(meshes)
        st = isochr.stitch(rs, vol.dims)  # pruned request: NaN outside the selection
        full = isochr.stitch(isochr.request(arch, k, drop_pruned=False), vol.dims)
        topo = isochr.verify_topology(vol.grid, full, k)
        topo_p = isochr.verify_topology(vol.grid, st, k)
        info["requests"][repr(k)] = {
            "stitch_sha": sha(st.ravel(order="F")),
            "full_stitch_sha": sha(full.ravel(order="F")),
            "topo_full": [topo.preserved_fraction, topo.differing_cells, topo.total_cells,
                          list(topo.first_diff) if topo.first_diff else None],
            "topo_pruned": [topo_p.preserved_fraction, topo_p.differing_cells, topo_p.total_cells,
                            list(topo_p.first_diff) if topo_p.first_diff else None],
            "regions": [r.region_id for r, _ in rs.regions],
            "recon_sha": [sha(np.asarray(s).ravel(order="F")) for _, s in rs.regions],
            "bytes_touched": rs.report.bytes_touched,
            "ntri": [int(mm.num_triangles) for mm in meshes],
            "nvert": [int(mm.num_vertices) for mm in meshes],
            "merged_v_sha": sha(merged.vertices),
            "merged_t_sha": sha(merged.triangles),
        }
    META["archive_" + name] = info
    return arch


# c1 recipe: 64^3, 8 blobs, noise, bs16, r=1e-3, k=0.5*max, f32 raw
rng = np.random.default_rng(0)
n = 64
x = np.arange(n, dtype=np.float64)
X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
f = np.zeros((n, n, n))
for _ in range(8):
    c = rng.uniform(0, n, size=3)
    s = rng.uniform(4, 12)
    a = rng.uniform(0.5, 1.0)
    f += a * np.exp(-((X - c[0]) ** 2 + (Y - c[1]) ** 2 + (Z - c[2]) ** 2) / (2 * s * s))
f += rng.uniform(-1e-3, 1e-3, size=f.shape)
f32 = f.astype("<f4")
vol = isochr.Volume(dims=(n, n, n), values=f32.ravel(order="F"), source_dtype="f32")
archive_case("c1", vol, [0.5 * vol.value_range[1]], 16, loose_fraction=1e-3)

# small multi-candidate archives, f64 source (most reference tests use f64)
sph = isochr.gen_sphere((24, 24, 24), radius=8.0)
archive_case("sphere", sph, [-4.0, 0.0, 5.0], 8)
sm = isochr.gen_smooth_random((20, 21, 19), seed=8, num_modes=3)
archive_case("smooth", sm, [-1.0, float(np.median(sm.values)), 1.5], 6, loose_fraction=0.05)
# a candidate equal to a sample value -> e == 0 regions (verbatim codec 3)
rng = np.random.default_rng(3)
v32 = rng.normal(size=(17, 18, 16)).astype("<f4")
vq = isochr.Volume(dims=(17, 18, 16), values=v32.ravel(order="F"), source_dtype="f32")
archive_case("exactk", vq, [float(np.sort(vq.values)[vq.values.size // 2])], 5)
# out-of-range candidate kept with warn: everything pruned, loose bound
import warnings  # noqa: E402

with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    archive_case("oor", isochr.Volume(dims=(9, 8, 10), values=np.linspace(0, 1, 720)), [7.0], 4,
                 out_of_range="warn")

# accuracy < 1 and paper_edges bounds (bound.py:68-219)
archive_case("c1_acc95", vol, [0.5 * vol.value_range[1]], 16, "c1", loose_fraction=1e-3, accuracy=0.95)
archive_case("sphere_paper", sph, [-4.0, 0.0, 5.0], 8, "sphere", bound_mode="paper_edges")
archive_case("smooth_paper80", sm, [-1.0, float(np.median(sm.values)), 1.5], 6, "smooth", loose_fraction=0.05,
             bound_mode="paper_edges", accuracy=0.8)
archive_case("smooth_acc90", sm, [-1.0, float(np.median(sm.values)), 1.5], 6, "smooth", loose_fraction=0.05,
             accuracy=0.9)
# k on a sample: strict -> lossless regions; paper -> edges ending on k do not straddle
archive_case("exactk_paper", vq, [float(np.sort(vq.values)[vq.values.size // 2])], 5, "exactk",
             bound_mode="paper_edges", accuracy=0.7)

np.savez_compressed(os.path.join(HERE, "golden.npz"), **G)
with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
    json.dump(META, fh, indent=1, sort_keys=True)
print("golden arrays:", len(G), "bytes:", os.path.getsize(os.path.join(HERE, "golden.npz")))
