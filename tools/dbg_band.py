import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2408_05462_b200 as G
from oracle import oracle as O
for shape in [(4,4,4), (33,33,33), (64,8,8), (33,33,300), (300,40,9)]:
    g = np.random.default_rng(1).normal(size=shape).cumsum(axis=0)
    blk = G.compress(g, 1e-3)
    print("compressed", shape, blk.codec_id, flush=True)
    t = time.time()
    out = G.decompress(blk)
    print("decoded", shape, time.time() - t, flush=True)
    ref = O.decompress_block(blk.to_bytes())[1]
    print("match", np.array_equal(out.ravel(order="F"), ref), flush=True)
