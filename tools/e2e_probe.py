"""Timeline of bench.py's pipelined e2e loop: per step, when the H2D, the
compute and the D2H start and end (ms from the first H2D)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2408_05462_b200 import device as D  # noqa: E402

torch.cuda.set_device(0)
vals, dims, bs, cands, r = bench.make_input("c3", 512, 0, "cuda")
N = vals.numel()
ws0 = D.Workspaces()
info = bench.run_step(vals, dims, bs, cands, r, ws0)
host_in = torch.empty(N, dtype=torch.float32, pin_memory=True)
host_in.copy_(vals)
s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
wss = [ws0, D.Workspaces()]
dvols = [torch.empty_like(vals), torch.empty_like(vals)]
hout = [(torch.empty(info["archive"] + 1024, dtype=torch.uint8, pin_memory=True),
         torch.empty(info["nvert"] * 3 + 16, dtype=torch.float64, pin_memory=True),
         torch.empty(info["ntri"] * 3 + 16, dtype=torch.int32, pin_memory=True)) for _ in range(2)]
ev_in = [torch.cuda.Event() for _ in range(2)]
ev_used = [torch.cuda.Event() for _ in range(2)]
ev_out = [torch.cuda.Event() for _ in range(2)]
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
marks = {}


def mark(key, stream):
    e = E()
    e.record(stream)
    marks[key] = e


torch.cuda.synchronize()
with torch.cuda.stream(s_in):
    mark(("h2d", 0, "a"), s_in)
    dvols[0].copy_(host_in, non_blocking=True)
    mark(("h2d", 0, "b"), s_in)
    ev_in[0].record()
for i in range(nsteps):
    bi = i % 2
    if i + 1 < nsteps:
        nb = (i + 1) % 2
        with torch.cuda.stream(s_in):
            if i >= 1:
                s_in.wait_event(ev_used[nb])
            mark(("h2d", i + 1, "a"), s_in)
            dvols[nb].copy_(host_in, non_blocking=True)
            mark(("h2d", i + 1, "b"), s_in)
            ev_in[nb].record()
    with torch.cuda.stream(s_cmp):
        s_cmp.wait_event(ev_in[bi])
        if i >= 2:
            s_cmp.wait_event(ev_out[bi])
        mark(("cmp", i, "a"), s_cmp)
        inf = bench.run_step(dvols[bi], dims, bs, cands, r, wss[bi])
        mark(("cmp", i, "b"), s_cmp)
        ev_used[bi].record()
    with torch.cuda.stream(s_out):
        s_out.wait_event(ev_used[bi])
        mark(("d2h", i, "a"), s_out)
        nbytes = inf["archive"]
        ha, hv, ht = hout[bi]
        ha[:nbytes].copy_(inf["res"].blob[:nbytes], non_blocking=True)
        hv[: inf["nvert"] * 3].copy_(inf["verts"].reshape(-1), non_blocking=True)
        ht[: inf["ntri"] * 3].copy_(inf["tris"].reshape(-1), non_blocking=True)
        mark(("d2h", i, "b"), s_out)
        ev_out[bi].record()
torch.cuda.synchronize()
t0 = marks[("h2d", 0, "a")]
for i in range(nsteps):
    row = []
    for k in ("h2d", "cmp", "d2h"):
        if (k, i, "a") in marks:
            a = t0.elapsed_time(marks[(k, i, "a")])
            b = t0.elapsed_time(marks[(k, i, "b")])
            row.append(f"{k} {a:7.2f}-{b:7.2f} ({b - a:5.2f})")
    print(f"step {i}: " + "  ".join(row))
