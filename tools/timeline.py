"""Device timeline of one bench step (library launches only): kernels in
launch order with start/end, and the idle gaps between them.
    python tools/timeline.py [n] [min_gap_us]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2408_05462_b200 import _abi  # noqa: E402
from paper_2408_05462_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
min_gap = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
torch.cuda.set_device(0)
vals, dims, bs, cands, r = bench.make_input("c3", n, 0, "cuda")
ws = D.Workspaces()
L = _abi.lib()
for _ in range(3):
    bench.run_step(vals, dims, bs, cands, r, ws)
# host phase marks: every library entry point records "@>name" when called
# and "@<name" when it returns (zero-length records on the stream)
for nm in list(_abi.EXPORTS):
    if nm.startswith("chr_prof") or nm in ("chr_launch_count",):
        continue
    f = getattr(L, nm)

    def wrap(*a, _f=f, _n=nm):
        L.chr_prof_mark((">" + _n).encode(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        rc = _f(*a)
        L.chr_prof_mark(("<" + _n).encode(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        return rc
    setattr(L, nm, wrap)
torch.cuda.synchronize()
L.chr_prof_enable(1)
bench.run_step(vals, dims, bs, cands, r, ws)
torch.cuda.synchronize()
L.chr_prof_enable(0)
buf = ctypes.create_string_buffer(1 << 20)
L.chr_prof_timeline(buf, len(buf))
rows = [ln.split() for ln in buf.value.decode().splitlines()]
prev_end = 0.0
busy = 0.0
gaps = []
for name, a, b in rows:
    a, b = float(a), float(b)
    gap = (a - prev_end) * 1e3
    if gap > min_gap:
        gaps.append((gap, name))
    print(f"{a:8.3f} {b:8.3f} {1e3 * (b - a):8.1f}us gap {gap:7.1f}us  {name}")
    busy += b - a
    prev_end = max(prev_end, b)
print(f"span {prev_end:.3f} ms, kernels {busy:.3f} ms, idle {prev_end - busy:.3f} ms")
for g, nm in sorted(gaps, reverse=True)[:15]:
    print(f"  gap {g:7.1f}us before {nm}")
