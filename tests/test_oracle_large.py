"""The oracle (oracle/) against the REFERENCE's own outputs at BASELINE
sizes: c2 256^3 (all 9 (r, k) variants) and c3 512^3
(tests/golden/golden_large.json, made by make_golden_large.py running
isochr).  Pins the oracle beyond the small golden vectors, so the GPU tests
that compare against the oracle at c4/c5 sizes rest on a checked checker.
CPU only (no GPU needed)."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import recipes as R  # noqa: E402

with open(os.path.join(HERE, "golden", "golden_large.json")) as fh:
    LARGE = json.load(fh)["configs"]
WORKERS = len(os.sched_getaffinity(0))


def _check(name, f):
    ref = LARGE[name]
    assert R.sha(f) == ref["input_sha"]
    arch = O.build_chr(f.astype(np.float64), tuple(ref["dims"]), [ref["k"]], ref["bs"], source_dtype="f32",
                       loose_fraction=ref["r"], workers=WORKERS)
    blob = arch.to_bytes()
    assert len(blob) == ref["archive_nbytes"] and hashlib.sha256(blob).hexdigest() == ref["archive_sha"]
    sel = O.request(arch, ref["k"], workers=WORKERS)
    assert [s["id"] for s, _ in sel] == ref["selected"]
    h = hashlib.sha256()
    for _, w in sel:
        h.update(np.ascontiguousarray(w).tobytes())
    assert h.hexdigest() == ref["windows_sha"]
    v, t = O.extract_regions(sel, (1.0, 1.0, 1.0), ref["k"])
    assert hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() == ref["verts_sha"]
    assert hashlib.sha256(np.ascontiguousarray(t, dtype=np.int32).tobytes()).hexdigest() == ref["tris_sha"]


@pytest.fixture(scope="module")
def c2():
    return R.c2_field()


@pytest.mark.parametrize("name", [f"c2_q{int(q)}_r{r:g}" for q in R.C2_Q for r in R.C2_R])
def test_oracle_c2_variants_match_reference(c2, name):
    _check(name, c2)


def test_oracle_c3_matches_reference():
    _check("c3", R.c3_field())
