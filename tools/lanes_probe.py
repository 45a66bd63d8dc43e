"""Throughput of the c3 device-resident step run serially vs on L host
threads (one stream + workspaces each, steps interleaved): how much of the
step is idle GPU time (host syncs, launch gaps, kernel tails) that another
step's kernels can fill."""
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2408_05462_b200 import device as D  # noqa: E402

torch.cuda.set_device(0)
vals, dims, bs, cands, r = bench.make_input("c3", 512, 0, "cuda")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def lane(nsteps, ws, stream, out):
    torch.cuda.set_device(0)
    with torch.cuda.stream(stream):
        for _ in range(nsteps):
            out.append(bench.run_step(vals, dims, bs, cands, r, ws, light=True)["ntri"])
        stream.synchronize()


for L in (1, 2, 3):
    wss = [D.Workspaces() for _ in range(L)]
    sts = [torch.cuda.Stream() for _ in range(L)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        outs = [[] for _ in range(L)]
        th = [threading.Thread(target=lane, args=(K // L, wss[i], sts[i], outs[i])) for i in range(L)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        n = sum(len(o) for o in outs)
        print(f"lanes {L} rep {rep}: {n} steps {dt:.1f} ms -> {dt / n:.3f} ms/step  (tris {set(sum(outs, []))})")
