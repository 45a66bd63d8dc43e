"""Stress of the z-slab per-portion request: world ranks sharing one GPU
(gloo), the c4 recipe at 96^3, `reps` repetitions inside the same
processes; prints per-rank stage checksums (multi.DEBUG_SUMS) whenever they
differ from the first repetition.   python tools/stress_portion.py [world] [reps]"""
import os
import socket
import sys

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, reps, data):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CHR_SLAB_DEBUG="1")
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2408_05462_b200 import multi

    flat, dims, bs, k, r = data  # generated once by the parent (torch CPU FFT is not reproducible across processes)
    v = torch.from_numpy(flat)
    nx, ny, nz = dims
    slab = multi.slab_of(nz, bs, world, rank)
    host = v[slab.z_base * nx * ny: (slab.z_base + slab.nz_local) * nx * ny]
    local = host.cuda()
    hs = int(host.view(torch.int32).to(torch.int64).sum())

    def chk(tag):
        torch.cuda.synchronize()
        ds = int(local.view(torch.int32).to(torch.int64).sum())
        if ds != hs:
            print(f"rank {rank} CORRUPT at {tag}: host {hs} device {ds}", flush=True)

    chk("upload")
    import hashlib
    print(f"rank {rank} flat {hashlib.sha1(flat.tobytes()).hexdigest()[:12]} k {k}", flush=True)
    first = None
    bad = 0
    for it in range(reps):
        res = multi.build_archive_slab(local, dims, slab, [k], bs, loose_fraction=r)
        chk("compress")
        m = multi.request_extract_portions(res, 0, k)
        chk("request")
        sums = dict(multi.DEBUG_SUMS)
        sums["archive"] = int(res.blob.to(torch.int64).sum())
        sums["ntri"] = m.ntri_total
        dump = os.environ.get("STRESS_DUMP")
        if dump:
            import numpy as np
            np.savez_compressed(f"{dump}_r{rank}.npz", b=res.blob.cpu().numpy())
            if rank == 0:
                np.save(f"{dump}_regions.npy", res.regions)
        if first is None:
            first = sums
        elif sums != first:
            bad += 1
            diff = {kk: (first.get(kk), sums.get(kk)) for kk in sums if first.get(kk) != sums.get(kk)}
            print(f"rank {rank} rep {it}: {diff}", flush=True)
    print(f"rank {rank}: {bad} of {reps} repetitions differ; first {sorted(first.items())}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    from paper_2408_05462_b200 import synth

    v, dims, bs, cands, r = synth.make_config("c4", device="cpu", n=96)
    mp.spawn(worker, args=(world, port, reps, (v.numpy().copy(), dims, bs, float(cands[0]), r)), nprocs=world,
             join=True)
