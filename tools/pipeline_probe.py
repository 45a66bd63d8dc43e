"""Timeline of the bench's pipelined e2e loop (per-stream events)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2408_05462_b200 import device as D  # noqa: E402

torch.cuda.set_device(0)
vals, dims, bs, cands, r = bench.make_input("c3", 512, 0, "cuda")
N = vals.numel()
host_in = torch.empty(N, dtype=torch.float32, pin_memory=True)
host_in.copy_(vals)
wss = [D.Workspaces(), D.Workspaces()]
for w in wss:
    info = bench.run_step(vals, dims, bs, cands, r, w)
s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
dv = [torch.empty_like(vals), torch.empty_like(vals)]
hout = [(torch.empty(info["archive"] + 1024, dtype=torch.uint8, pin_memory=True),
         torch.empty(info["nvert"] * 3 + 16, dtype=torch.float64, pin_memory=True),
         torch.empty(info["ntri"] * 3 + 16, dtype=torch.int32, pin_memory=True)) for _ in range(2)]
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
from paper_2408_05462_b200 import _abi  # noqa: E402

L = _abi.lib()
CTAS = int(os.environ.get("SM_COPY_CTAS", "32"))


def chunked(dst, src):
    assert L.chr_sm_copy(dst.data_ptr(), src.data_ptr(), dst.numel() * dst.element_size(), CTAS,
                         torch.cuda.current_stream().cuda_stream) == 0


torch.cuda.synchronize()
# kernel times of a few isolated steps vs the overlapped ones
L.chr_prof_enable(1)
_abi.prof_report()
for _ in range(3):
    bench.run_step(vals, dims, bs, cands, r, wss[0])
torch.cuda.synchronize()
iso = _abi.prof_report()
base = E()
base.record()
marks = []
ev_in = [E(), E()]
ev_used = [E(), E()]
ev_out = [E(), E()]
with torch.cuda.stream(s_in):
    a = E(); a.record(); chunked(dv[0], host_in); ev_in[0].record(); marks.append(("h2d0", a, ev_in[0]))
t0 = time.perf_counter()
for i in range(6):
    b = i % 2
    if i + 1 < 6:
        nb = (i + 1) % 2
        with torch.cuda.stream(s_in):
            if i >= 1:
                s_in.wait_event(ev_used[nb])
            a = E(); a.record(); chunked(dv[nb], host_in); e = E(); e.record(); ev_in[nb] = e
            marks.append((f"h2d{i+1}", a, e))
    with torch.cuda.stream(s_cmp):
        s_cmp.wait_event(ev_in[b])
        a = E(); a.record()
        h0 = time.perf_counter()
        inf = bench.run_step(dv[b], dims, bs, cands, r, wss[b])
        h1 = time.perf_counter()
        e = E(); e.record(); ev_used[b] = e
        marks.append((f"cmp{i} host {1e3*(h1-h0):.1f}ms", a, e))
    with torch.cuda.stream(s_out):
        s_out.wait_event(ev_used[b])
        a = E(); a.record()
        nbytes = inf["archive"]
        chunked(hout[b][0][:nbytes], inf["res"].blob[:nbytes])
        chunked(hout[b][1][: inf["nvert"] * 3], inf["verts"].reshape(-1))
        chunked(hout[b][2][: inf["ntri"] * 3], inf["tris"].reshape(-1))
        e = E(); e.record(); ev_out[b] = e
        marks.append((f"d2h{i}", a, e))
torch.cuda.synchronize()
ovl = _abi.prof_report()
L.chr_prof_enable(0)
print("wall ms per step", (time.perf_counter() - t0) * 1e3 / 6)
ti = sum(t for k, (c, t) in iso.items() if k != "k_sm_copy") / 3
to = sum(t for k, (c, t) in ovl.items() if k != "k_sm_copy") / 6
print(f"chr kernel ms/step isolated {ti:.2f} overlapped {to:.2f}")
for k in sorted(iso, key=lambda k: -iso[k][1])[:6]:
    print(f"  {k:24s} iso {iso[k][1]/3:.3f} ovl {ovl.get(k, (0, 0))[1]/6:.3f}")
for name, a, e in marks:
    print(f"{name:28s} start {base.elapsed_time(a):8.2f}  end {base.elapsed_time(e):8.2f}")
