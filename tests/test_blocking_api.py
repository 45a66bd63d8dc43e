"""The blocking API (decompose / build_index / merge_regions,
blocking.py:77-193) against fixtures the reference produced
(tests/golden/golden_large.json, make_golden_large.py).

merge_regions is host C++ (chr_merge_keys) and runs here without a GPU;
decompose reads the block extrema from the chr_stats kernel (``-m gpu``)."""

import json
import os
import sys

import numpy as np
import pytest

import paper_2408_05462_b200 as G
from paper_2408_05462_b200 import exceptions as E
from paper_2408_05462_b200.index import BlockMeta, IsoIndex

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from recipes import sha  # noqa: E402


@pytest.fixture(scope="module")
def large():
    with open(os.path.join(HERE, "golden", "golden_large.json")) as fh:
        return json.load(fh)


def _blocks(case):
    return [BlockMeta(b[0], tuple(b[1]), tuple(b[2]), tuple(b[3]), b[4], b[5]) for b in case["blocks"]]


def _regions(regs):
    return [[r.region_id, [list(r.block_span[0]), list(r.block_span[1])], list(r.sample_origin),
             list(r.sample_extent), sorted(r.relevance_key)] for r in regs]


@pytest.mark.parametrize("name", ["sphere", "smooth", "odd_dims", "custom_keys"])
def test_merge_regions_matches_reference(large, name):
    case = large["blocking"][name]
    idx = IsoIndex(tuple(case["cands"]), tuple(frozenset(s) for s in case["relevant"]))
    regs = G.merge_regions(_blocks(case), idx)
    assert _regions(regs) == case["regions"]


@pytest.mark.parametrize("name", ["sphere", "smooth", "odd_dims"])
def test_build_index_matches_reference(large, name):
    case = large["blocking"][name]
    idx = G.build_index(_blocks(case), case["cands"])
    assert [sorted(s) for s in idx.relevant] == case["relevant"]
    assert list(idx.candidates) == case["cands"]


def test_build_index_rejects_bad_candidates(large):
    blocks = _blocks(large["blocking"]["sphere"])
    for bad in ([], [1.0, float("nan")], [1.0, 1.0], [2.0, 1.0]):
        with pytest.raises(E.ParameterError):
            G.build_index(blocks, bad)


def test_merge_regions_empty():
    assert G.merge_regions([], IsoIndex((0.0,), (frozenset(),))) == []


def _volume(name, golden):
    if name == "odd_dims":
        vals = np.random.default_rng(5).normal(size=23 * 17 * 30)
        return G.Volume((23, 17, 30), values=vals)
    dims = {"sphere": (24, 24, 24), "smooth": (20, 21, 19)}[name]
    return G.Volume(dims, values=golden[name + "_in"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sphere", "smooth", "odd_dims"])
def test_decompose_matches_reference(large, golden, name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    case = large["blocking"][name]
    vol = _volume(name, golden)
    assert sha(vol.values) == case["values_sha"]
    blocks = G.decompose(vol, case["bs"])
    got = [[b.block_id, list(b.block_coords), list(b.sample_origin), list(b.sample_extent), b.vmin, b.vmax]
           for b in blocks]
    assert got == case["blocks"]
    # the whole chain on the device-derived blocks
    regs = G.merge_regions(blocks, G.build_index(blocks, case["cands"]))
    assert _regions(regs) == case["regions"]


@pytest.mark.gpu
def test_value_range_from_device_kernel():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rng = np.random.default_rng(3)
    for dt in (torch.float32, torch.float64):
        a = torch.from_numpy(rng.normal(size=(7, 9, 11))).to(dt)
        vol = G.Volume((11, 9, 7), values=a.cuda())
        lo, hi = vol.value_range
        assert (lo, hi) == (float(a.min()), float(a.max()))
        b = a.clone().reshape(-1)
        b[123] = float("inf")
        b[456] = float("nan")
        with pytest.raises(E.NonFiniteSampleError) as ei:
            _ = G.Volume((11, 9, 7), values=b.cuda()).value_range
        assert ei.value.index == 123
