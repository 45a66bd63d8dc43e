"""The z-slab path under NCCL (world = 1 on one B200): the branches that move
CUDA tensors through NCCL (all-gathers of block stats, stream summaries, CRC
shares, z-carry and boundary planes, mesh counts; the assemble all-reduce)
run for real, and the result equals the single-GPU path's file and the
oracle's mesh."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, port, out_path):
    import sys

    import torch.distributed as dist

    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    torch.cuda.set_device(0)
    from paper_2408_05462_b200 import device as D, multi, synth

    v, dims, bs, cands, r = synth.make_config("c4", device="cpu", n=96)
    k = cands[0]
    vals = v.cuda()
    slab = multi.slab_of(dims[2], bs, 1, 0)
    res = multi.build_archive_slab(vals, dims, slab, [k], bs, loose_fraction=r)
    full = multi.assemble(res)
    ref = D.build_archive(vals, dims, [k], bs, loose_fraction=r)
    same_file = full.cpu().numpy().tobytes() == ref.blob[: ref.nbytes].cpu().numpy().tobytes()
    m = multi.request_extract_portions(res, 0, k)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O

    oref = O.build_chr(v.numpy().astype(np.float64), dims, [k], bs, source_dtype="f32", loose_fraction=r)
    rv, rt = O.extract_regions(O.request(oref, k), (1.0, 1.0, 1.0), k)
    ok = same_file and np.array_equal(m.tris.cpu().numpy(), rt) and np.array_equal(m.verts.cpu().numpy(), rv)
    with open(out_path, "w") as f:
        f.write(f"{int(ok)} {int(same_file)} {dist.get_backend()}\n")
    dist.destroy_process_group()


def test_slab_path_under_nccl(tmp_path):
    if not torch.cuda.is_available() or not torch.distributed.is_nccl_available():
        pytest.skip("needs CUDA + NCCL")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "r.txt")
    mp.spawn(_worker, args=(port, out), nprocs=1, join=True)
    ok, same_file, backend = open(out).read().split()
    assert backend == "nccl" and same_file == "1" and ok == "1"
