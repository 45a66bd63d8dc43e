"""Parity at BASELINE.json's full sizes (c3 512^3 single GPU,
c4 1024^3, c5 1536^3 with 16 candidates).

* c3 512^3 (always; c4 / c5 with CHR_FULLSIZE=1): archive bytes, request
  windows and the merged mesh are bit-identical to the oracle's on the same
  input (the oracle runs the whole volume on all host threads).
* every config (c4 / c5 only with CHR_FULLSIZE=1 -- 4 GiB / 13.5 GiB inputs):
  size-independent properties -- the file validates on the device (trailer
  CRC, table, block headers), every region decodes within its error bound
  (escapes and verbatim regions exactly), and with the strict accuracy-1
  bound every cell's marching-cubes case is preserved for every candidate
  (verify_topology over the stitched full request == 1.0).
"""

import hashlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_05462_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2408_05462_b200 import device, synth  # noqa: E402

FULL = os.environ.get("CHR_FULLSIZE", "") == "1"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _properties(vals, dims, bs, cands, r):
    assert vals.numel() == dims[0] * dims[1] * dims[2]
    res = device.build_archive(vals, dims, cands, bs, loose_fraction=r)
    # f1: trailer CRC, header, every record and block header, on the device
    ft = device.read_table(res.blob, res.nbytes)
    info = ft.info[0]
    assert int(info["error"]) == 0 and int(info["stored_crc"]) == int(info["actual_crc"])
    assert not ft.entries["status"].any()
    regs = res.regions
    assert np.array_equal(ft.regions["block_offset"], regs["block_offset"])
    # every region within its bound
    dec = device.dec_table(regs["block_offset"] + device.BLOCK_HEADER, regs["block_nbytes"] - device.BLOCK_HEADER,
                           regs["codec_id"], regs["extent"], regs["error_bound"], regs["payload_crc"])
    wins, offs, st = device.decode(res.blob, dec)
    assert not any(st)
    nx, ny, nz = dims
    vol3 = vals.view(nz, ny, nx)
    worst = 0.0
    for i in range(len(regs)):
        ox, oy, oz = (int(v) for v in regs["origin"][i])
        ex, ey, ez = (int(v) for v in regs["extent"][i])
        ref = vol3[oz:oz + ez, oy:oy + ey, ox:ox + ex].double()
        got = wins[offs[i]: offs[i] + ex * ey * ez].view(ez, ey, ex)
        err = float((got - ref).abs().max())
        e = float(regs["error_bound"][i])
        assert err <= e, (i, err, e, int(regs["codec_id"][i]))
        if int(regs["codec_id"][i]) in (0, 3):
            assert err == 0.0
        worst = max(worst, err / e if e > 0 else 0.0)
    # strict accuracy 1: every cell case preserved, for every candidate
    tab = np.zeros(len(regs), dtype=device._abi.STITCH_DT)
    for i in range(len(regs)):
        tab[i] = (offs[i], regs["origin"][i], regs["extent"][i], regs["lo"][i], regs["hi"][i])
    stitched = device.stitch(wins, tab, dims, bs)
    assert not bool(torch.isnan(stitched).any())
    for k in cands:
        nd, first = device.topology_compare(vals, stitched, dims, float(k))
        assert nd == 0, (k, nd, first)
    return res, worst


@pytest.mark.parametrize("name", ["c3"] + (["c4", "c5"] if FULL else []))
def test_fullsize_bit_exact_vs_oracle(name):
    vals, dims, bs, cands, r = synth.make_config(name, device="cuda")
    assert dims == {"c3": (512,) * 3, "c4": (1024,) * 3, "c5": (1536,) * 3}[name]
    res, _ = _properties(vals, dims, bs, cands, r)
    host = vals.cpu().numpy().astype(np.float64)
    ref = O.build_chr(host, dims, cands, bs, source_dtype="f32", loose_fraction=r,
                      workers=len(os.sched_getaffinity(0)))
    assert res.blob[: res.nbytes].cpu().numpy().tobytes() == ref.to_bytes()
    k = cands[0]
    sel = O.request(ref, k, workers=len(os.sched_getaffinity(0)))
    regs = res.regions
    mine = regs[(regs["mask"] & np.uint64(1)) != 0]
    assert [int(x) for x in np.nonzero((regs["mask"] & np.uint64(1)) != 0)[0]] == [s["id"] for s, _ in sel]
    dec = device.dec_table(mine["block_offset"] + device.BLOCK_HEADER, mine["block_nbytes"] - device.BLOCK_HEADER,
                           mine["codec_id"], mine["extent"], mine["error_bound"], mine["payload_crc"])
    wins, offs, st = device.decode(res.blob, dec, iso=k)
    assert not any(st)
    host_w = wins.cpu().numpy()
    for (s, w), o in zip(sel, offs):
        assert np.array_equal(host_w[o:o + w.size], w), s["id"]
    mct = device.mc_table(dec["out_offset"], mine["extent"], mine["origin"].astype(np.float64), (1.0, 1.0, 1.0))
    ws = device.Workspaces()
    v, t, _, _ = device.marching(wins, mct, k, ws=ws)
    rv, rt = O.extract_regions(sel, (1.0, 1.0, 1.0), k)
    assert np.array_equal(v.cpu().numpy(), rv) and np.array_equal(t.cpu().numpy(), rt)


@pytest.mark.skipif(not FULL, reason="CHR_FULLSIZE=1 runs the 1024^3 / 1536^3 configs")
@pytest.mark.parametrize("name", ["c4", "c5"])
def test_fullsize_properties(name):
    vals, dims, bs, cands, r = synth.make_config(name, device="cuda")
    assert dims == {"c4": (1024,) * 3, "c5": (1536,) * 3}[name]
    res, worst = _properties(vals, dims, bs, cands, r)
    print(f"{name}: {dims}, {len(cands)} candidates, {len(res.regions)} regions, archive {res.nbytes} bytes, "
          f"worst |recon - v| / e = {worst:.3f}")
