"""cProfile of the host side of bench.run_step (device work included as waits).
    python tools/host_profile.py [n] [steps]"""
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2408_05462_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
torch.cuda.set_device(0)
vals, dims, bs, cands, r = bench.make_input("c3", n, 0, "cuda")
ws = D.Workspaces()
for _ in range(3):
    bench.run_step(vals, dims, bs, cands, r, ws)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    bench.run_step(vals, dims, bs, cands, r, ws)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
