"""A small end-to-end workload for compute-sanitizer (tools/sanitize.sh):
c1 / c2 / c3 recipes at reduced size through every device stage --
stats, plan, compress (piece and segment encoders), read_table, decode
(band tiles: face flag waits, shared mask-word atomics; int64 re-pass; the
generic path), fused masks, marching cubes (batch queues), stitch, topology
compare, the kernel-seam shims."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_05462_b200 import device as D, synth  # noqa: E402


def run(name, n, **kw):
    vals, dims, bs, cands, r = synth.make_config(name, device="cuda", n=n, **kw)
    res = D.build_archive(vals, dims, cands, bs, loose_fraction=r)
    ft = D.read_table(res.blob, res.nbytes)
    assert int(ft.info["error"][0]) == 0
    regs = res.regions
    sel = regs[(regs["mask"] & np.uint64(1)) != 0]
    dec = D.dec_table(sel["block_offset"] + D.BLOCK_HEADER, sel["block_nbytes"] - D.BLOCK_HEADER, sel["codec_id"],
                      sel["extent"], sel["error_bound"], sel["payload_crc"])
    wins, offs, st = D.decode(res.blob, dec, iso=cands[0])
    assert not any(st)
    mct = D.mc_table(dec["out_offset"], sel["extent"], sel["origin"] * 1.0, (1.0, 1.0, 1.0))
    v, t, _, _ = D.marching(wins, mct, cands[0], masks=D._DEFAULT_WS.get("decode_mask", 4, torch.int32))
    v2, t2, _, _ = D.marching(wins, mct, cands[0])
    assert torch.equal(t, t2) and torch.equal(v, v2)
    p = D.pipeline(vals, dims, cands, bs, loose_fraction=r)
    assert torch.equal(p.tris, t)
    tab = np.zeros(len(sel), dtype=D._abi.STITCH_DT)
    for i in range(len(sel)):
        tab[i] = (offs[i], sel["origin"][i], sel["extent"][i], sel["lo"][i], sel["hi"][i])
    vol = D.stitch(wins, tab, dims, bs)
    D.topology_compare(vals, vol, dims, cands[0])
    print(name, n, len(regs), "regions", int(t.shape[0]), "triangles", flush=True)


run("c1", 48)
run("c2", 64)
run("c3", 64)
g = np.random.default_rng(5).uniform(-1e7, 1e7, size=(20, 20, 20))  # int64 band re-pass
import paper_2408_05462_b200 as G  # noqa: E402

blk = G.compress(g, 0.5)
G.decompress(blk)
q = torch.from_numpy(np.random.default_rng(1).integers(-300, 300, 5000)).cuda()
D.rle_varint_decode(D.rle_varint_encode(q), 5000)
os.environ["CHR_ENC_SEG"] = "1"  # the segment encoder (new plan cache key)
run("c2", 48)
print("sanitize case done")
