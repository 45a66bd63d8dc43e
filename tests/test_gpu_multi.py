"""z-slab multi-GPU protocol on one GPU: two processes share
cuda:0 and exchange only the small records over gloo (no kernel of one rank
waits on the other).  The slices they write must OR into exactly the file
the single-GPU path writes."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _field(case):
    rng = np.random.default_rng(7)
    if case == "grf":
        dims, bs = (48, 40, 70), 8
        g = rng.normal(size=dims[::-1]).cumsum(0).cumsum(1).cumsum(2)
    elif case == "outliers":
        dims, bs = (33, 30, 61), 8
        g = rng.normal(size=dims[::-1]).cumsum(2)
        idx = rng.choice(g.size, size=25, replace=False)
        g.reshape(-1)[idx] = rng.uniform(1e11, 1e12, size=25)
    else:  # "exact": a candidate equal to a sample value (lossless regions)
        dims, bs = (40, 36, 50), 8
        g = rng.normal(size=dims[::-1]).cumsum(0)
    return dims, bs, np.ascontiguousarray(g, dtype=np.float32).reshape(-1)  # [z][y][x] -> x fastest


def _worker(rank, world, port, case, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2408_05462_b200 import device as D, multi

    dims, bs, flat = _field(case)
    nx, ny, nz = dims
    vals = torch.from_numpy(flat)
    k = float(np.percentile(flat.astype(np.float64), 60))
    if case == "exact":
        k = float(flat[1234])
    cands = [k]
    slab = multi.slab_of(nz, bs, world, rank)
    local = vals[slab.z_base * nx * ny: (slab.z_base + slab.nz_local) * nx * ny].cuda()
    res = multi.build_archive_slab(local, dims, slab, cands, bs, loose_fraction=1e-3)
    full = multi.assemble(res)
    if rank == 0:
        ref = D.build_archive(vals.cuda(), dims, cands, bs, loose_fraction=1e-3)
        got = full.cpu().numpy().tobytes()
        want = ref.blob[: ref.nbytes].cpu().numpy().tobytes()
        with open(out_path, "w") as f:
            codecs = "".join(str(int(c)) for c in sorted(set(ref.regions["codec_id"].tolist())))
            f.write(f"{len(got)} {len(want)} {int(got == want)} {len(ref.regions)} {codecs}\n")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["grf", "outliers", "exact"])
def test_slab_archive_matches_single_gpu(tmp_path, world, case):
    out = str(tmp_path / "res.txt")
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    ng, nw, same, nreg, codecs = open(out).read().split()
    assert int(nreg) >= 1
    if case == "outliers":
        assert "2" in codecs  # escapes across slab boundaries
    assert ng == nw and same == "1", (ng, nw)


def _mesh_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2408_05462_b200 import device as D, multi

    dims, bs, flat = _field("grf")
    nx, ny, nz = dims
    vals = torch.from_numpy(flat)
    k = float(np.percentile(flat.astype(np.float64), 60))
    slab = multi.slab_of(nz, bs, world, rank)
    local = vals[slab.z_base * nx * ny: (slab.z_base + slab.nz_local) * nx * ny].cuda()
    res = multi.build_archive_slab(local, dims, slab, [k], bs, loose_fraction=1e-3)
    full = multi.assemble(res)
    m = multi.request_extract_slab(full, res.regions, 0, k)
    # the same request from the slices alone (owned payloads by one all-to-all, no file assembly)
    m2 = multi.request_extract_slab(res, res.regions, 0, k, dims=dims, bs=bs)
    same_local = (m2.regions == m.regions and m2.tri_base == m.tri_base and m2.vert_base == m.vert_base
                  and torch.equal(m2.tris, m.tris) and torch.equal(m2.verts, m.verts))
    flags = [None] * world
    dist.all_gather_object(flags, bool(same_local))
    # gather every rank's rows into the merged mesh on rank 0
    parts = [None] * world
    dist.all_gather_object(parts, (m.tri_base, m.vert_base, m.regions, m.tris.cpu().numpy(), m.verts.cpu().numpy()))
    if rank == 0:
        T = np.zeros((m.ntri_total, 3), np.int32)
        V = np.zeros((m.nvert_total, 3), np.float64)
        bases = {}  # selected-region index -> (tri base, vert base) in the merged mesh
        for tb, vb, regs, _, _ in parts:
            bases.update({i: (x, y) for i, x, y in zip(regs, tb, vb)})
        order = sorted(bases)
        ends = {i: (bases[j][0], bases[j][1]) for i, j in zip(order, order[1:])}
        ends[order[-1]] = (m.ntri_total, m.nvert_total)
        for tb, vb, regs, t, v in parts:
            to = vo = 0
            for i in regs:  # a rank's rows are its regions in selection order
                nt_i, nv_i = ends[i][0] - bases[i][0], ends[i][1] - bases[i][1]
                T[bases[i][0]: bases[i][0] + nt_i] = t[to: to + nt_i]
                V[bases[i][1]: bases[i][1] + nv_i] = v[vo: vo + nv_i]
                to += nt_i
                vo += nv_i
        ref = D.build_archive(vals.cuda(), dims, [k], bs, loose_fraction=1e-3)
        sel = ref.regions[(ref.regions["mask"] & np.uint64(1)) != 0]
        dec = D.dec_table(sel["block_offset"] + D.BLOCK_HEADER, sel["block_nbytes"] - D.BLOCK_HEADER, sel["codec_id"],
                          sel["extent"], sel["error_bound"], sel["payload_crc"])
        wins, _, _ = D.decode(ref.blob, dec)
        mct = D.mc_table(dec["out_offset"], sel["extent"], sel["origin"] * 1.0, (1.0, 1.0, 1.0))
        rv, rt, _, _ = D.marching(wins, mct, k)
        ok = np.array_equal(rt.cpu().numpy(), T) and np.array_equal(rv.cpu().numpy(), V) and all(flags)
        with open(out_path, "w") as f:
            f.write(f"{int(ok)} {len(T)} {len(V)} {len(sel)}\n")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_request_extract_matches_single_gpu(tmp_path, world):
    out = str(tmp_path / "mesh.txt")
    mp.spawn(_mesh_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    ok, nt, nv, nsel = open(out).read().split()
    assert int(nsel) >= world and int(nt) > 0
    assert ok == "1"


def _c4_field():
    """BASELINE c4 recipe (GRF k^-11/3 in [0,1], bs32, r=1e-4, k=0.5) at 96^3,
    generated ONCE by the test process and handed to every rank (torch's CPU
    FFT under three competing processes is not bit-reproducible, so ranks
    generating it themselves could disagree about the input)."""
    from paper_2408_05462_b200 import synth

    v, dims, bs, cands, r = synth.make_config("c4", device="cpu", n=96)
    return v.numpy().copy(), dims, bs, float(cands[0]), r


def _portion_worker(rank, world, port, case, out_path, c4=None):
    """z-slab compress, then the per-portion request + marching cubes
    (request_extract_portions: no payload bytes leave their rank); rank 0
    reassembles the merged mesh from every rank's rows and compares it with
    the ORACLE's (oracle/, pinned to the reference) on the same field."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys

    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2408_05462_b200 import multi

    if case == "c4":
        flat, dims, bs, k, r = c4
    else:
        dims, bs, flat = _field(case)
        r = 1e-3
        k = float(np.percentile(flat.astype(np.float64), 60))
    nx, ny, nz = dims
    vals = torch.from_numpy(flat)
    slab = multi.slab_of(nz, bs, world, rank)
    local = vals[slab.z_base * nx * ny: (slab.z_base + slab.nz_local) * nx * ny].cuda()
    res = multi.build_archive_slab(local, dims, slab, [k], bs, loose_fraction=r)
    m = multi.request_extract_portions(res, 0, k)
    parts = [None] * world
    dist.all_gather_object(parts, (m.tri_base, m.vert_base, m.ntri, m.nvert, m.tris.cpu().numpy(),
                                   m.verts.cpu().numpy()))
    if rank == 0:
        T = np.full((m.ntri_total, 3), -1, np.int32)
        V = np.full((m.nvert_total, 3), np.nan, np.float64)
        for tb, vb, nts, nvs, t, vv in parts:
            to = vo = 0
            for b0, b1, a, c in zip(tb, vb, nts, nvs):
                T[b0: b0 + a] = t[to: to + a]
                V[b1: b1 + c] = vv[vo: vo + c]
                to += a
                vo += c
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O

        ref = O.build_chr(flat.astype(np.float64), dims, [k], bs, source_dtype="f32", loose_fraction=r)
        sel = O.request(ref, k)
        rv, rt = O.extract_regions(sel, (1.0, 1.0, 1.0), k)
        ok = np.array_equal(rt, T) and np.array_equal(rv, V)
        codecs = "".join(str(int(c)) for c in sorted(set(res.regions["codec_id"].tolist())))
        with open(out_path, "w") as f:
            f.write(f"{int(ok)} {len(T)} {len(rt)} {len(V)} {len(rv)} {codecs}\n")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["grf", "outliers", "c4"])
def test_slab_portion_request_matches_oracle(tmp_path, world, case):
    out = str(tmp_path / "mesh.txt")
    c4 = _c4_field() if case == "c4" else None
    mp.spawn(_portion_worker, args=(world, _free_port(), case, out, c4), nprocs=world, join=True)
    ok, nt, ntr, nv, nvr, codecs = open(out).read().split()
    assert int(ntr) > 0 and (nt, nv) == (ntr, nvr)
    if case == "outliers":
        assert "2" in codecs
    assert ok == "1"
