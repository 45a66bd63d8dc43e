"""Run the bench step (compress -> request -> MC) a few times on one config,
for ncu / compute-sanitizer captures.  Usage: python tools/profile_step.py [n] [steps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2408_05462_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = sys.argv[3] if len(sys.argv) > 3 else "c3"
torch.cuda.set_device(0)
vals, dims, bs, cands, r = bench.make_input(cfg, n, 0, "cuda")
ws = D.Workspaces()
for _ in range(steps):
    info = bench.run_step(vals, dims, bs, cands, r, ws)
torch.cuda.synchronize()
print("ok", info["archive"], info["ntri"], info["nvert"])
