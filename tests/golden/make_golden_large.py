"""Reference-pinned fixtures at BASELINE sizes + the blocking API, made by
running the REFERENCE itself (isochr) -- TEST INFRASTRUCTURE.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_large.py

Writes tests/golden/golden_large.json:

* ``configs``: for c2 (256^3, all 9 (r, k) variants) and c3 (512^3), the
  SHA-256 of the bit-reproducible input (recipes.py), then the reference's
  outputs as SHA-256s: the .chr file (write_chr), the request(k) windows
  (drop_pruned=True, each window raveled x-fastest, concatenated in
  selection order), the merged mesh (marching_cubes per selected region with
  origin = sample_origin * spacing, merge_meshes: vertices f64, triangles
  int32), plus sizes, selected region ids and bytes_touched
  (chr_archive.py:132-274, isosurf.py:183-225).
* ``blocking``: decompose / build_index / merge_regions outputs
  (blocking.py:77-193) on small volumes, including a hand-made IsoIndex.
* ``bourke``: Bourke-order case codes of the mcrand grids of golden.npz,
  formed with the reference's CORNER_OFFSETS exactly as mc_extract /
  _mc_vectorized form them (kernels.py:448-470, isosurf.py:126-131).

Nothing on the GPU box reads /root/reference: only this JSON travels.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, os.environ.get("ISOCHR_SRC", "/root/reference/pkg/src"))
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import isochr  # noqa: E402
from isochr.blocking import IsoIndex, build_index, decompose, merge_regions  # noqa: E402
from isochr.mc_tables import CORNER_OFFSETS  # noqa: E402

import recipes as R  # noqa: E402

WORKERS = len(os.sched_getaffinity(0))
OUT: dict = {"configs": {}, "blocking": {}, "bourke": {}}


def sha_bytes(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def run_config(name, vals, dims, bs, k, r):
    vol = isochr.Volume(dims=dims, values=vals, source_dtype="f32")
    t0 = time.time()
    arch = isochr.build_chr(vol, [k], block_size=bs, loose_fraction=r, workers=WORKERS)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "a.chr")
        isochr.write_chr(arch, p)
        blob = open(p, "rb").read()
    rs = isochr.request(arch, k, drop_pruned=True, workers=WORKERS)
    h = hashlib.sha256()
    meshes = []
    nsel = 0
    for region, samples in rs.regions:
        h.update(np.asarray(samples, dtype=np.float64).ravel(order="F").tobytes())
        nsel += samples.size
        meshes.append(isochr.marching_cubes(samples, spacing=vol.spacing,
                                            origin=tuple(o * s for o, s in zip(region.sample_origin, vol.spacing)),
                                            k=k))
    merged = isochr.merge_meshes(meshes)
    OUT["configs"][name] = {
        "input_sha": R.sha(vals), "dims": list(dims), "bs": bs, "k": k, "r": r,
        "archive_sha": sha_bytes(blob), "archive_nbytes": len(blob), "n_regions": len(arch.regions),
        "codecs": np.bincount([rg.block.codec_id for rg in arch.regions], minlength=4).tolist(),
        "selected": [rg.region_id for rg, _ in rs.regions], "bytes_touched": rs.report.bytes_touched,
        "windows_sha": h.hexdigest(), "window_samples": int(nsel),
        "n_tri": int(merged.num_triangles), "n_vert": int(merged.num_vertices),
        "verts_sha": hashlib.sha256(np.ascontiguousarray(merged.vertices, dtype=np.float64).tobytes()).hexdigest(),
        "tris_sha": hashlib.sha256(np.ascontiguousarray(merged.triangles, dtype=np.int32).tobytes()).hexdigest(),
    }
    print(name, f"{time.time() - t0:.1f}s", len(arch.regions), "regions", len(blob), "B",
          merged.num_triangles, "tris", flush=True)


# --- c2 256^3: one field, 9 (r, k) variants ------------------------------------
f2 = R.c2_field()
for q in R.C2_Q:
    k = R.percentile(f2, q)
    for r in R.C2_R:
        run_config(f"c2_q{int(q)}_r{r:g}", f2, (256, 256, 256), 16, k, r)
del f2
# --- c3 512^3 -------------------------------------------------------------------
f3 = R.c3_field()
run_config("c3", f3, (512, 512, 512), 32, R.percentile(f3, 99.0), 1e-3)
del f3

# --- blocking API -----------------------------------------------------------------


def blocking_case(name, vol, cands, bs, custom=None):
    blocks = decompose(vol, bs)
    idx = build_index(blocks, cands) if custom is None else custom(blocks)
    regs = merge_regions(blocks, idx)
    OUT["blocking"][name] = {
        "dims": list(vol.dims), "bs": bs, "cands": list(idx.candidates),
        "values_sha": R.sha(vol.values),
        "blocks": [[b.block_id, list(b.block_coords), list(b.sample_origin), list(b.sample_extent), b.vmin, b.vmax]
                   for b in blocks],
        "relevant": [sorted(s) for s in idx.relevant],
        "regions": [[rg.region_id, [list(rg.block_span[0]), list(rg.block_span[1])], list(rg.sample_origin),
                     list(rg.sample_extent), sorted(rg.relevance_key)] for rg in regs],
    }


sph = isochr.gen_sphere((24, 24, 24), radius=8.0)
blocking_case("sphere", sph, [-4.0, 0.0, 5.0], 8)
sm = isochr.gen_smooth_random((20, 21, 19), seed=8, num_modes=3)
blocking_case("smooth", sm, [-1.0, float(np.median(sm.values)), 1.5], 6)
rng = np.random.default_rng(5)
odd = isochr.Volume(dims=(23, 17, 30), values=rng.normal(size=23 * 17 * 30))
blocking_case("odd_dims", odd, [-0.5, 0.0, 0.7], 4)


def checkerboard(blocks):
    # a hand-made index whose keys are not a span test (merge must use them as given)
    rel = (frozenset(b.block_id for b in blocks if sum(b.block_coords) % 2 == 0),
           frozenset(b.block_id for b in blocks if b.block_coords[2] >= 1))
    return IsoIndex(candidates=(0.0, 1.0), relevant=rel)


blocking_case("custom_keys", sph, [0.0, 1.0], 8, custom=checkerboard)

# --- Bourke-order case codes (kernels.py:448-470) -----------------------------------
g = np.load(os.path.join(HERE, "golden.npz"))
for seed in range(5):
    grid = g[f"mcrand{seed}_in"].reshape((8, 7, 9), order="F")
    inside = grid >= 0.1
    ncx, ncy, ncz = (n - 1 for n in grid.shape)
    codes = np.zeros((ncx, ncy, ncz), dtype=np.uint8)
    for i in range(8):
        ox, oy, oz = (int(v) for v in CORNER_OFFSETS[i])
        codes |= inside[ox:ox + ncx, oy:oy + ncy, oz:oz + ncz].astype(np.uint8) << i
    OUT["bourke"][f"mcrand{seed}"] = codes.ravel(order="F").tolist()

with open(os.path.join(HERE, "golden_large.json"), "w") as fh:
    json.dump(OUT, fh, indent=0, sort_keys=True)
print("wrote golden_large.json")
