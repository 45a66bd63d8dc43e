"""One warm c3 pipeline step between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (every kernel of exactly one step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_05462_b200 import device as D, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
vals, dims, bs, cands, r = synth.make_config(cfg, device="cuda")
ws = D.Workspaces()
for _ in range(2):
    D.pipeline(vals, dims, cands, bs, loose_fraction=r, ws=ws)
torch.cuda.synchronize()
torch.cuda.profiler.start()
D.pipeline(vals, dims, cands, bs, loose_fraction=r, ws=ws)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("one step done")
