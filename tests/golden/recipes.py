"""Bit-reproducible CPU generators for the BASELINE.json config recipes
 -- TEST INFRASTRUCTURE.

``make_golden_large.py`` runs these here, feeds the result to the reference
(``isochr``) and commits SHA-256s of the reference's outputs keyed by the
SHA-256 of the input; the ``-m gpu`` tests regenerate the same input on the
GPU box, check its SHA first, then compare the CUDA path's outputs with the
reference's.  So every operation here must give identical bits on any x86-64
host running this image:

* white noise: ``numpy.random.default_rng(seed).standard_normal`` (integer
  ziggurat; libm only in the tails);
* FFTs: ``numpy.fft`` (pocketfft, no runtime SIMD dispatch);
* the spectrum amplitude ``|k|^(slope/2)`` from a table over the integer
  ``|k|^2`` filled with ``math.pow`` (glibc), not ``np.power`` (SIMD-dispatched);
* ``exp`` for the lognormal field as range reduction + a Horner polynomial
  of separately rounded numpy multiplies/adds (``np.exp`` is SIMD-dispatched);
* standardisation from exact ``math.fsum`` sums over a fixed subsample;
* min/max, percentiles (selection + one lerp) and f32 rounding are exact.

Inputs are float32, x fastest (what ``load_raw`` reads).
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

LN2_HI = 6.93147180369123816490e-01  # trailing zero bits: k * LN2_HI is exact
LN2_LO = 1.90821492927058770002e-10
INV_LN2 = 1.44269504088896338700e00


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def det_exp(x: np.ndarray) -> np.ndarray:
    """exp(x) to ~1 ulp with IEEE +,-,*,ldexp only (deterministic)."""
    k = np.rint(x * INV_LN2)
    r = (x - k * LN2_HI) - k * LN2_LO
    p = np.full_like(r, 1.0 / math.factorial(13))
    for n in range(12, -1, -1):
        p = p * r + 1.0 / math.factorial(n)
    return np.ldexp(p, k.astype(np.int32))


def grf(n: int, slope: float, seed: int = 0, kmax: float | None = None, nz: int | None = None) -> np.ndarray:
    """Gaussian random field, amplitude |k|^(slope/2) (power |k|^slope),
    zero at k = 0 and beyond kmax; f64 array indexed [z, y, x]."""
    nz = n if nz is None else nz
    white = np.random.default_rng(seed).standard_normal((nz, n, n))
    spec = np.fft.rfftn(white)
    del white
    iz = np.fft.fftfreq(nz, d=1.0 / nz).astype(np.int64).reshape(nz, 1, 1)
    iy = np.fft.fftfreq(n, d=1.0 / n).astype(np.int64).reshape(1, n, 1)
    ix = np.fft.rfftfreq(n, d=1.0 / n).astype(np.int64).reshape(1, 1, n // 2 + 1)
    k2 = iz * iz + iy * iy + ix * ix  # integer |k|^2
    table = np.array([0.0] + [math.pow(float(v), slope / 4.0) for v in range(1, int(k2.max()) + 1)])
    if kmax is not None:
        table[np.arange(table.size) > kmax * kmax] = 0.0
    spec *= table[k2]
    del k2
    return np.fft.irfftn(spec, s=(nz, n, n), axes=(0, 1, 2))


def _minmax01(f: np.ndarray) -> np.ndarray:
    lo, hi = f.min(), f.max()
    return (f - lo) / (hi - lo)


def _standardise(g: np.ndarray) -> np.ndarray:
    s = g.reshape(-1)[::97]
    mu = math.fsum(s.tolist()) / s.size
    var = math.fsum(np.square(s - mu).tolist()) / s.size
    return (g - mu) / math.sqrt(var)


def percentile(values_f32: np.ndarray, q: float) -> float:
    """np.percentile(values.astype(np.float64), q)."""
    return float(np.percentile(values_f32.astype(np.float64), q))


def c2_field(n: int = 256, seed: int = 0) -> np.ndarray:
    """c2: GRF P(k) ~ k^-11/3 truncated at |k| = 32, min-max to [0, 1]."""
    return _minmax01(grf(n, -11.0 / 3.0, seed, kmax=32)).astype("<f4").reshape(-1)


def c3_field(n: int = 512, seed: int = 0) -> np.ndarray:
    """c3: lognormal exp(1.5 g), g a unit-variance GRF with P(k) ~ k^-3."""
    g = _standardise(grf(n, -3.0, seed))
    return det_exp(1.5 * g).astype("<f4").reshape(-1)


C2_R = (1e-2, 1e-3, 1e-4)
C2_Q = (25.0, 50.0, 75.0)
