"""Race / initialisation checks without compute-sanitizer (it is closed on
this GPU pool: profiles/r02_compute_sanitizer_refused.log).  The reference's
own stand-in is determinism across worker counts (test_chr.py:64-71); here:

* the whole path run repeatedly gives bit-identical archives, windows and
  meshes (the decoder's tile hand-offs spin on flags published with release
  fences; its mask words are shared by two bands through atomics; the
  marching-cubes passes take work from atomic queues -- any race would show
  as run-to-run differences over many repetitions and tile orders);
* every workspace poisoned with random bytes between runs changes nothing
  (no kernel reads scratch it did not write: the initcheck stand-in);
* two streams running the path concurrently on different inputs give the
  results each gives alone (no shared mutable state in the library)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2408_05462_b200 import device as D, synth  # noqa: E402


def _run(vals, dims, bs, cands, r, ws):
    p = D.pipeline(vals, dims, cands, bs, loose_fraction=r, ws=ws)
    torch.cuda.current_stream().synchronize()
    return (p.archive.cpu().numpy().tobytes(), p.windows.cpu().numpy().tobytes(), p.verts.cpu().numpy().tobytes(),
            p.tris.cpu().numpy().tobytes())


def _poison(ws, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    for name, t in ws._bufs.items():
        if isinstance(t, torch.Tensor) and t.is_cuda:
            b = t.view(torch.uint8) if t.dtype != torch.uint8 else t
            b.copy_(torch.randint(0, 256, b.shape, dtype=torch.uint8, device="cuda", generator=g))


@pytest.mark.parametrize("name,n", [("c3", 128), ("c2", 96), ("c1", 64)])
def test_repeated_runs_bit_identical_with_poisoned_workspaces(name, n):
    vals, dims, bs, cands, r = synth.make_config(name, device="cuda", n=n)
    ws = D.Workspaces()
    ref = _run(vals, dims, bs, cands, r, ws)
    for it in range(8):
        _poison(ws, it)
        assert _run(vals, dims, bs, cands, r, ws) == ref, it


def test_two_streams_concurrently():
    a = synth.make_config("c3", device="cuda", n=96)
    b = synth.make_config("c2", device="cuda", n=96)
    ra = _run(*a, D.Workspaces())
    rb = _run(*b, D.Workspaces())
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    wa, wb = D.Workspaces(), D.Workspaces()
    for _ in range(3):
        with torch.cuda.stream(sa):
            pa = D.pipeline(a[0], a[1], a[3], a[2], loose_fraction=a[4], ws=wa)
        with torch.cuda.stream(sb):
            pb = D.pipeline(b[0], b[1], b[3], b[2], loose_fraction=b[4], ws=wb)
        torch.cuda.synchronize()
        assert pa.archive.cpu().numpy().tobytes() == ra[0] and pb.archive.cpu().numpy().tobytes() == rb[0]
        assert pa.tris.cpu().numpy().tobytes() == ra[3] and pb.tris.cpu().numpy().tobytes() == rb[3]
