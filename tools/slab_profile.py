"""cProfile of one warm z-slab step (world 1, NCCL) at c3."""
import cProfile
import os
import pstats
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2408_05462_b200 import device as D, multi, synth  # noqa: E402

with socket.socket() as so:
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
torch.cuda.set_device(0)
vals, dims, bs, cands, r = synth.make_config("c3", device="cuda")
slab = multi.slab_of(dims[2], bs, 1, 0)
ws = D.Workspaces()


def step():
    res = multi.build_archive_slab(vals, dims, slab, cands, bs, loose_fraction=r, ws=ws)
    m = multi.request_extract_portions(res, 0, cands[0], ws=ws)
    torch.cuda.synchronize()
    return m


step()
step()
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(25)
dist.destroy_process_group()
