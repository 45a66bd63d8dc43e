"""cProfile of the drop-in API path (bench.api_e2e's run) at c3 on the GPU box."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_05462_b200 as G  # noqa: E402
from paper_2408_05462_b200 import synth  # noqa: E402

vals, dims, bs, cands, r = synth.make_config("c3", device="cuda")
host = vals.cpu().numpy()
k = cands[0]


def run():
    vol = G.Volume(dims, values=host, source_dtype="f32")
    arch = G.build_chr(vol, [k], bs, loose_fraction=r)
    rs = G.request(arch, k)
    meshes = [G.marching_cubes(win, vol.spacing, tuple(o * sp for o, sp in zip(reg.sample_origin, vol.spacing)), k)
              for reg, win in rs.regions]
    m = G.merge_meshes(meshes)
    torch.cuda.synchronize()
    return m


run()
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(30)
st.sort_stats("tottime").print_stats(20)
