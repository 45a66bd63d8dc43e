"""The reference's documented behaviours, checked on the GPU package.

Each test restates one behaviour the reference's own suite asserts
(pkg/tests/test_codec.py, test_chr.py, test_isosurf.py; file:line in the
docstrings) against ``paper_2408_05462_b200`` used as a drop-in for
``isochr``: same calls, same exceptions, same guarantees.  The byte-level
parity lives in test_gpu_parity.py / test_gpu_fullsize.py; these are the
semantic contracts around it.
"""

import struct
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_05462_b200 as G  # noqa: E402
from paper_2408_05462_b200 import exceptions as X  # noqa: E402
from paper_2408_05462_b200.blockcodec import HEADER_SIZE, CompressedBlock  # noqa: E402


def sphere(dims, radius):
    """Signed distance to a centred sphere (the reference's gen_sphere shape)."""
    axes = [np.arange(n, dtype=np.float64) - (n - 1) / 2.0 for n in dims]
    X_, Y_, Z_ = np.meshgrid(*axes, indexing="ij")
    g = np.sqrt(X_ ** 2 + Y_ ** 2 + Z_ ** 2) - radius
    return G.Volume(dims=dims, values=g.ravel(order="F"))


def smooth(dims, seed, modes=3):
    """A few random cosine modes (a smooth band-limited field)."""
    rng = np.random.default_rng(seed)
    axes = [np.linspace(0.0, 1.0, n) for n in dims]
    X_, Y_, Z_ = np.meshgrid(*axes, indexing="ij")
    g = np.zeros(dims)
    for _ in range(modes):
        kx, ky, kz = rng.uniform(1.0, 4.0, 3)
        g += rng.uniform(0.5, 1.0) * np.cos(2 * np.pi * (kx * X_ + ky * Y_ + kz * Z_) + rng.uniform(0, 2 * np.pi))
    return G.Volume(dims=dims, values=g.ravel(order="F"))


def size_cap(n):
    return 8 * n + HEADER_SIZE + (n + 7) // 8


# ------------------------------------------------------------------ codec (test_codec.py)
def test_constant_field_is_tiny_and_within_bound():
    """test_codec.py:28-33"""
    g = np.full((32, 32, 32), 5.0)
    b = G.compress(g, 0.1)
    assert b.codec_id == 1 and len(b.payload) < 512
    assert np.abs(G.decompress(b) - g).max() <= 0.1


def test_zero_bound_is_verbatim_and_exact():
    """test_codec.py:36-40"""
    g = np.random.default_rng(1).normal(size=(7, 5, 9))
    b = G.compress(g, 0.0)
    assert b.codec_id == 0 and np.array_equal(G.decompress(b), g)


def test_random_fields_round_trip_within_bound():
    """test_codec.py:50-58, 77-88 (escapes), 102-107 (size cap)"""
    for seed in range(6):
        g = np.random.default_rng(seed).normal(size=(9, 8, 7))
        for frac in (1e-1, 1e-2, 1e-3):
            e = frac * (g.max() - g.min())
            b = G.compress(g, e)
            assert np.abs(G.decompress(b) - g).max() <= e
            assert b.nbytes <= size_cap(g.size)
    rng = np.random.default_rng(2)
    g = rng.normal(size=(8, 8, 8))
    g.reshape(-1)[rng.choice(512, size=5, replace=False)] = 1e18
    b = G.compress(g, 1e-3)
    assert b.codec_id == 2 and np.abs(G.decompress(b) - g).max() <= 1e-3 and b.nbytes <= size_cap(512)


def test_hard_bound_property():
    """test_codec.py:61-74 (hypothesis): any finite field, three bounds"""
    hyp = pytest.importorskip("hypothesis")
    from hypothesis import given, settings
    from hypothesis import strategies as st
    from hypothesis.extra import numpy as hnp

    @given(hnp.arrays(np.float64, st.tuples(st.integers(2, 6), st.integers(2, 6), st.integers(2, 6)),
                      elements=st.floats(min_value=-1e12, max_value=1e12, allow_nan=False)),
           st.sampled_from([1e-1, 1e-2, 1e-3]))
    @settings(max_examples=60, deadline=None)
    def check(g, frac):
        e = frac * max(g.max() - g.min(), 1e-12)
        assert np.abs(G.decompress(G.compress(g, e)) - g).max() <= e

    del hyp
    check()


def test_incompressible_is_verbatim_and_deterministic_and_idempotent():
    """test_codec.py:91-99, 110-120"""
    rng = np.random.default_rng(3)
    g = rng.uniform(-1e9, 1e9, size=(8, 8, 8))
    b = G.compress(g, 1e-12)
    assert b.codec_id == 0 and np.array_equal(G.decompress(b), g)
    h = rng.normal(size=(12, 10, 8))
    assert G.compress(h, 0.01).to_bytes() == G.compress(h, 0.01).to_bytes()
    first = G.decompress(G.compress(h, 0.05))
    assert np.abs(G.decompress(G.compress(first, 0.05)) - first).max() <= 0.05


def test_checksum_catches_every_payload_flip():
    """test_codec.py:123-132"""
    g = np.random.default_rng(4).normal(size=(6, 6, 6))
    raw = bytearray(G.compress(g, 0.01).to_bytes())
    for pos in range(HEADER_SIZE, len(raw)):
        raw[pos] ^= 0x40
        with pytest.raises(X.CorruptPayloadError):
            G.decompress(CompressedBlock.from_bytes(bytes(raw)))
        raw[pos] ^= 0x40


def test_header_fields_and_parameter_errors():
    """test_codec.py:135-183"""
    rng = np.random.default_rng(5)
    b = G.compress(rng.normal(size=(4, 5, 6)), 0.25, source_dtype="f32")
    back = CompressedBlock.from_bytes(b.to_bytes())
    assert back == b and back.dims == (4, 5, 6) and back.error_bound == 0.25 and back.source_dtype == "f32"
    g = np.zeros((3, 3, 3))
    g[1, 2, 0] = np.inf
    with pytest.raises(X.NonFiniteSampleError):
        G.compress(g, 0.1)
    for bad in (-1.0, np.nan):
        with pytest.raises(X.ParameterError):
            G.compress(rng.normal(size=(3, 3, 3)), bad)
    weird = CompressedBlock(250, b.dims, b.error_bound, b.source_dtype, b.payload, b.checksum)
    with pytest.raises(X.UnsupportedCodecError):
        G.decompress(weird)
    with pytest.raises(X.ParameterError):
        G.register_codec(0, "dup", lambda blk: None)


def test_f32_sources_verbatim():
    """test_codec.py:186-205"""
    rng = np.random.default_rng(6)
    g32 = rng.normal(size=(4, 4, 4)).astype("<f4").astype(np.float64)
    b = G.compress(g32, 0.0, source_dtype="f32")
    assert b.codec_id == 3 and len(b.payload) == 4 * 64 and np.array_equal(G.decompress(b), g32)
    g = rng.normal(size=(4, 4, 4))  # mislabelled doubles stay exact
    b = G.compress(g, 0.0, source_dtype="f32")
    assert b.codec_id == 0 and np.array_equal(G.decompress(b), g)


def test_payload_shrinks_as_bound_grows():
    """test_codec.py:208-211"""
    g = smooth((24, 24, 24), seed=9).grid
    sizes = [len(G.compress(g, e).payload) for e in (1e-4, 1e-3, 1e-2, 1e-1)]
    assert sizes == sorted(sizes, reverse=True)


# ------------------------------------------------------------------ archive (test_chr.py)
@pytest.fixture(scope="module")
def sphere_archive():
    vol = sphere((24, 24, 24), 8.0)
    return vol, G.build_chr(vol, [-4.0, 0.0, 5.0], block_size=8, accuracy=1.0)


def test_relevant_regions_cover_every_mixed_cell(sphere_archive):
    """test_chr.py:34-46"""
    vol, arch = sphere_archive
    ci = arch.candidates.index(0.0)
    cf = G.case_field(vol.grid, 0.0)
    mixed = (cf.codes != 0) & (cf.codes != 255)
    covered = np.zeros(cf.cell_dims, dtype=bool, order="F")
    for r in arch.regions:
        if r.is_relevant(ci):
            (ox, oy, oz), (ex, ey, ez) = r.sample_origin, r.sample_extent
            covered[ox:ox + ex - 1, oy:oy + ey - 1, oz:oz + ez - 1] = True
    assert covered.ravel(order="F")[mixed].all()


def test_constant_field_prunes_and_out_of_range_refused():
    """test_chr.py:49-61"""
    vol = G.Volume(dims=(8, 8, 8), values=np.full(512, 3.0))
    with pytest.warns(UserWarning):
        arch = G.build_chr(vol, [7.0], block_size=4, out_of_range="warn")
    assert all(not r.relevance for r in arch.regions)
    assert np.array_equal(G.stitch(G.request(arch, 7.0, drop_pruned=False), vol.dims), vol.grid)
    with pytest.raises(X.ParameterError):
        G.build_chr(sphere((8, 8, 8), 2.0), [1e6], block_size=4)


def test_rebuild_and_roundtrip_byte_identical(tmp_path, sphere_archive):
    """test_chr.py:64-87"""
    vol = smooth((20, 20, 20), seed=8)
    k = float(np.median(vol.values))
    a, b = tmp_path / "a.chr", tmp_path / "b.chr"
    G.write_chr(G.build_chr(vol, [k], block_size=8, accuracy=0.95), a)
    G.write_chr(G.build_chr(vol, [k], block_size=8, accuracy=0.95), b)
    assert a.read_bytes() == b.read_bytes()
    assert G.build_chr(vol, [k], 8, workers=1) == G.build_chr(vol, [k], 8, workers=4)
    _, arch = sphere_archive
    p = tmp_path / "s.chr"
    G.write_chr(arch, p)
    assert G.read_chr(p) == arch


def test_damaged_files_are_refused(tmp_path, sphere_archive):
    """test_chr.py:90-137"""
    _, arch = sphere_archive
    p = tmp_path / "t.chr"
    G.write_chr(arch, p)
    blob = p.read_bytes()
    p.write_bytes(blob[:-10])
    with pytest.raises(X.ChecksumError):
        G.read_chr(p)
    p.write_bytes(b"NOPE" + blob[4:])
    with pytest.raises(X.BadMagicError):
        G.read_chr(p)
    bad = bytearray(blob)
    bad[4] = 99
    bad[-4:] = struct.pack("<I", zlib.crc32(bytes(bad[:-4])))
    p.write_bytes(bytes(bad))
    with pytest.raises(X.VersionError):
        G.read_chr(p)


def test_request_selection_report_and_errors(sphere_archive):
    """test_chr.py:140-182"""
    _, arch = sphere_archive
    rep = G.request(arch, 0.0, drop_pruned=True).report
    assert rep.regions_returned < rep.regions_total and rep.bytes_touched < rep.bytes_total
    assert rep.bytes_touched == arch.header_table_nbytes() + sum(
        r.payload_nbytes for r in arch.regions if r.is_relevant(rep.candidate_index))
    full = G.request(arch, 0.0, drop_pruned=False).report
    assert full.regions_returned == full.regions_total and full.bytes_touched == full.bytes_total - 4
    with pytest.raises(X.NoSuchIsovalueError):
        G.request(arch, 0.25)
    r = G.request(arch, 2.5, snap=True).report  # equidistant: the lower candidate
    assert r.isovalue == 0.0 and r.snapped
    assert G.request(arch, 4.9, snap=True).report.isovalue == 5.0
    low = G.build_chr(sphere((12, 12, 12), 4.0), [0.0], block_size=6, accuracy=0.9)
    with pytest.raises(X.InsufficientAccuracyError) as exc:
        G.request(low, 0.0, accuracy=0.95)
    assert exc.value.requested == 0.95 and exc.value.stored == 0.9
    G.request(low, 0.0, accuracy=0.5)


def test_reconstruction_within_region_bounds_and_stitch(sphere_archive):
    """test_chr.py:185-213"""
    vol, arch = sphere_archive
    recon = G.request(arch, 0.0, drop_pruned=False)
    g = vol.grid
    for region, samples in recon.regions:
        (ox, oy, oz), (ex, ey, ez) = region.sample_origin, region.sample_extent
        assert np.abs(samples - g[ox:ox + ex, oy:oy + ey, oz:oz + ez]).max() <= region.error_bound
    st = G.stitch(recon, vol.dims)
    assert np.isfinite(st).all()
    assert np.abs(st - g).max() <= max(r.error_bound for r in arch.regions)
    exact = G.Volume(dims=(3, 3, 3), values=np.arange(27.0))
    a = G.build_chr(exact, [13.0], block_size=4)
    assert a.regions[0].error_bound == 0.0
    assert np.array_equal(G.stitch(G.request(a, 13.0, drop_pruned=False), exact.dims), exact.grid)


def test_ghost_plane_owner_wins():
    """test_chr.py:226-240"""
    x = np.arange(9, dtype=np.float64)
    vol = G.Volume(dims=(9, 4, 4), values=np.tile(x, 16))
    arch = G.build_chr(vol, [1.0], block_size=4)
    assert len(arch.regions) == 2
    recon = G.request(arch, 1.0, drop_pruned=False)
    st = G.stitch(recon, vol.dims)
    arrays = {r.sample_origin: s for r, s in recon.regions}
    low = min(arrays)
    ex = {r.sample_origin: r for r in arch.regions}[low].sample_extent[0]
    assert np.array_equal(st[low[0] + ex - 1], arrays[low][ex - 1])


def test_plugin_codec_flows_through(tmp_path):
    """test_chr.py:243-276: a registered codec id survives build / write /
    read / request (decoded by its plugin)"""
    def comp(samples, error_bound, source_dtype="f64"):
        grid = np.asfortranarray(np.asarray(samples, dtype=np.float64))
        payload = bytes(b ^ 0x33 for b in grid.ravel(order="F").astype("<f8").tobytes())
        return CompressedBlock(201, grid.shape, float(error_bound), source_dtype, payload, zlib.crc32(payload))

    def decomp(block):
        n = block.dims[0] * block.dims[1] * block.dims[2]
        raw = bytes(b ^ 0x33 for b in block.payload)
        return np.frombuffer(raw, dtype="<f8", count=n).astype(np.float64).reshape(block.dims, order="F")

    try:
        G.register_codec(201, "xor-behaviour", decomp)
    except X.ParameterError:
        pass  # registered by an earlier run in this process
    vol = sphere((12, 12, 12), 4.0)
    arch = G.build_chr(vol, [0.0], block_size=6, codec=comp)
    assert all(r.block.codec_id == 201 for r in arch.regions)
    p = tmp_path / "x.chr"
    G.write_chr(arch, p)
    assert np.array_equal(G.stitch(G.request(G.read_chr(p), 0.0, drop_pruned=False), vol.dims), vol.grid)


def test_accuracy_changes_only_bound_fields():
    """test_chr.py:279-294"""
    vol = smooth((16, 16, 16), seed=6)
    k = float(np.median(vol.values))
    a = G.build_chr(vol, [k], block_size=8, accuracy=1.0)
    b = G.build_chr(vol, [k], block_size=8, accuracy=0.8)
    assert len(a.regions) == len(b.regions)
    for ra, rb in zip(a.regions, b.regions):
        assert (ra.region_id, ra.block_span, ra.sample_origin, ra.sample_extent, ra.relevance) == \
               (rb.region_id, rb.block_span, rb.sample_origin, rb.sample_extent, rb.relevance)
        if ra.relevance:
            assert ra.error_bound <= rb.error_bound
        assert ra.accuracy == 1.0 and rb.accuracy == 0.8


# ------------------------------------------------------------------ isosurface (test_isosurf.py)
def test_cell_cases_and_empty_mesh():
    """test_isosurf.py:20-40, 69-72"""
    assert G.cell_case([0.0] * 8, 0.5) == 0 and G.cell_case([1.0] * 8, 0.5) == 255
    for i in range(8):
        c = [0.0] * 8
        c[i] = 1.0
        assert G.cell_case(c, 0.5) == 1 << i
    assert (G.case_field(np.full((4, 4, 4), 2.0), 2.0).codes == 255).all()
    m = G.marching_cubes(np.zeros((4, 4, 4)), k=0.5)
    assert m.num_triangles == 0 and m.num_vertices == 0


def test_linear_ramp_vertices_exact_and_on_edges():
    """test_isosurf.py:75-81, 139-155"""
    x = np.arange(5, dtype=np.float64)
    g = np.broadcast_to(x[:, None, None], (5, 3, 3)).copy()
    m = G.marching_cubes(g, k=1.5)
    assert m.num_triangles > 0 and np.all(m.vertices[:, 0] == 1.5)
    rng = np.random.default_rng(7)
    g = rng.normal(size=(7, 6, 5))
    m = G.marching_cubes(g, k=0.0)
    v = m.vertices
    frac = v - np.floor(v)
    assert np.all((frac != 0).sum(axis=1) <= 1)  # each vertex on one axis-aligned edge


def test_spacing_origin_and_shared_vertices():
    """test_isosurf.py:83-88, 158-162"""
    g = sphere((10, 10, 10), 3.0).grid
    a = G.marching_cubes(g, k=0.0)
    b = G.marching_cubes(g, spacing=(2.0, 3.0, 0.5), origin=(1.0, -1.0, 4.0), k=0.0)
    assert np.array_equal(b.triangles, a.triangles)
    assert np.allclose(b.vertices, a.vertices * [2.0, 3.0, 0.5] + [1.0, -1.0, 4.0], rtol=0, atol=1e-12)
    assert len(np.unique(a.vertices, axis=0)) == a.num_vertices  # no duplicated vertex


def test_verify_topology_and_merge():
    """test_isosurf.py:165-186, 218-224"""
    g = sphere((10, 10, 10), 3.0).grid
    rep = G.verify_topology(g, g.copy(), 0.0)
    assert rep.preserved_fraction == 1.0 and rep.differing_cells == 0 and rep.first_diff is None
    h = g.copy()
    h[5, 5, 5] = -h[5, 5, 5] if h[5, 5, 5] != 0 else 1.0
    rep = G.verify_topology(g, h, 0.0)
    assert rep.differing_cells > 0 and rep.preserved_fraction < 1.0
    with pytest.raises(X.ParameterError):
        G.verify_topology(g, g[:-1], 0.0)
    m1 = G.marching_cubes(g, k=0.0)
    merged = G.merge_meshes([m1, m1])
    assert merged.num_triangles == 2 * m1.num_triangles
    assert np.array_equal(merged.triangles[m1.num_triangles:], m1.triangles + m1.num_vertices)


# ------------------------------------------------------------------ acceptance criteria (test_acceptance.py)
def _fields():
    from paper_2408_05462_b200 import synth

    out = [("sphere", sphere((40, 40, 40), 12.0), 0.0)]
    for name, n in (("c2", 64), ("c3", 64), ("c5", 48)):
        vals, dims, bs, cands, r = synth.make_config(name, device="cuda", n=n)
        out.append((name, G.Volume(dims, (1.0, 1.0, 1.0), vals.cpu().numpy().astype(np.float64), "f32"), cands[0]))
    return out


def test_acceptance_strict_topology_and_relaxation_monotone():
    """test_acceptance.py:61-75 (criterion 1) and 130-158 (criterion 4):
    strict accuracy 1 preserves every cell case; relaxing the accuracy
    never shrinks the bounds and never grows the bytes a request touches"""
    for name, vol, k in _fields():
        bounds, touched, kept = [], [], {}
        for acc in (0.80, 0.95, 0.99, 1.0):
            arch = G.build_chr(vol, [k], block_size=16, accuracy=acc)
            bounds.append(max(r.error_bound for r in arch.regions if r.relevance))
            touched.append(G.request(arch, k, accuracy=acc, drop_pruned=True).report.bytes_touched)
            full = G.stitch_device(G.request(arch, k, accuracy=acc, drop_pruned=False), vol.dims)
            kept[acc] = G.verify_topology(vol.grid, full, k).preserved_fraction
        assert all(a >= b for a, b in zip(bounds, bounds[1:])), (name, bounds)
        assert all(a <= b for a, b in zip(touched, touched[1:])), (name, touched)
        assert kept[1.0] == 1.0, (name, kept)
        paper = G.build_chr(vol, [k], block_size=16, bound_mode="paper_edges")
        full = G.stitch(G.request(paper, k, drop_pruned=False), vol.dims)
        assert 0.0 <= G.verify_topology(vol.grid, full, k).preserved_fraction <= 1.0


def test_acceptance_codec_bound_exhaustive():
    """test_acceptance.py:106-127 (criterion 3): no sample ever outside the
    bound, 20 random 32^3 fields x 3 bounds"""
    violations = 0
    for seed in range(20):
        g = np.random.default_rng(seed).normal(size=(32, 32, 32))
        for frac in (1e-1, 1e-2, 1e-3):
            e = frac * (g.max() - g.min())
            violations += int((np.abs(G.decompress(G.compress(g, e)) - g) > e).sum())
    assert violations == 0
