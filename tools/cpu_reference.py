"""CPU baseline of the hot path: the REFERENCE package itself (isochr, numba)
when it is installed under baseline/_ref (tools/install_ref.sh; it travels to
the GPU box with the repo), else the oracle port (oracle/).  Used only by
bench.py's ``cpu_baseline`` leg and its ``--impl reference`` arm -- never by
the product path.

Timing follows BASELINE.md §2 / the reference harness: warmed with
``isochr.pipeline._warmup`` (pipeline.py:106-118), median of ``repeats``
runs per stage (pipeline._median_time, pipeline.py:82-90) of
  build_chr(volume, [k], bs, loose_fraction=r, workers=w)
  request(archive, k, drop_pruned=True, workers=w)
  per-region marching_cubes + merge_meshes (pipeline._extract_regions)
at a stated worker count.  The sample is a bounded z-slab of the workload
(the first ``planes`` planes of the same field, same bs / r / k).
"""

from __future__ import annotations

import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_module():
    """The installed reference package, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "isochr")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/chr_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import isochr  # noqa: PLC0415
    except Exception:  # pragma: no cover - broken install
        return None
    return isochr


def _sample(vals_host, dims, planes):
    nx, ny, nz = dims
    pz = min(planes, nz) if planes > 0 else nz
    return np.ascontiguousarray(vals_host[: nx * ny * pz]), (nx, ny, pz)


def time_stages(vals_host, dims, bs, k, r, planes, workers, repeats=3):
    """Per-stage median seconds on the sample; returns dict with kind."""
    sample, sdims = _sample(vals_host, dims, planes)
    lo, hi = float(sample.min()), float(sample.max())
    k = float(min(max(k, lo), hi))
    iso = reference_module()
    if iso is not None:
        from isochr import pipeline  # noqa: PLC0415

        pipeline._warmup()
        vol = iso.Volume(dims=sdims, values=sample.astype(np.float32), source_dtype="f32")
        tb, arch = pipeline._median_time(
            lambda: iso.build_chr(vol, [k], block_size=bs, loose_fraction=r, workers=workers), repeats)
        tr, rs = pipeline._median_time(lambda: iso.request(arch, k, drop_pruned=True, workers=workers), repeats)
        tm, mesh = pipeline._median_time(lambda: pipeline._extract_regions(rs, vol.spacing, k), repeats)
        kind = "reference"
        what = "isochr (the reference package, numba) from baseline/_ref"
    else:
        sys.path.insert(0, ROOT)
        from oracle import oracle as O  # noqa: PLC0415

        f64 = sample.astype(np.float64)

        def med(fn):
            ts, out = [], None
            for _ in range(max(1, repeats)):
                t0 = time.perf_counter()
                out = fn()
                ts.append(time.perf_counter() - t0)
            return statistics.median(ts), out

        tb, arch = med(lambda: O.build_chr(f64, sdims, [k], bs, source_dtype="f32", loose_fraction=r,
                                           workers=workers, out_of_range="warn"))
        tr, sel = med(lambda: O.request(arch, k, workers=workers))
        tm, _ = med(lambda: O.extract_regions(sel, (1.0, 1.0, 1.0), k))
        kind = "port"
        what = "the oracle port of the reference (oracle/, C), baseline/_ref absent"
    n = sdims[0] * sdims[1] * sdims[2]
    t = tb + tr + tm
    return {
        "value": 4 * n / t / 1e9, "unit": "GB/s", "cores": workers, "kind": kind,
        "stages_s": {"build_chr": tb, "request": tr, "marching_cubes": tm},
        "sample": (f"{sdims[0]}x{sdims[1]}x{sdims[2]} z-slab of the same field (first {sdims[2]} of {dims[2]} planes), "
                   f"same bs/r/k; {what}; median of {repeats} per stage, workers={workers}"),
    }
