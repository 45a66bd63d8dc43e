"""Seeded synthetic scalar fields for the BASELINE.json configs.

There is no public dataset for this path; these
generators produce inputs with the configs' shapes, spectra and value
distributions.  They run in torch on any device: on the GPU for the large
configs (fast FFT), on the CPU for tests.  Parity never depends on
reproducing a generator bit-for-bit across machines: every parity check
hands the *same* array to the oracle and to the CUDA path.

  c1  64^3  8 Gaussian blobs + U(+-1e-3) noise, bs16, r=1e-3, k=0.5*max
  c2  256^3 GRF P(k)~k^-11/3 truncated |k|<=32, [0,1], bs16, r in {1e-2,1e-3,1e-4},
            k = 25/50/75th percentile
  c3  512^3 lognormal exp(1.5 g), g unit-variance GRF P(k)~k^-3, bs32, r=1e-3, k=p99
  c4  1024^3 GRF P(k)~k^-11/3, [0,1], bs32, r=1e-4, k=0.5
  c5  1536^3 GRF + 64 blobs (sigma 8..48) -> [0,1], bs32, r=1e-4, 16 candidates
"""

from __future__ import annotations

import math

import numpy as np
import torch


def _gen(seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def grf(n, slope, seed=0, kmax=None, device="cpu", nz=None):
    """Gaussian random field with amplitude |k|^(slope/2) (power |k|^slope).

    Returned as float32 (n, n, nz) tensor indexed [x, y, z]; memory order
    is x fastest when flattened with ``.permute(2, 1, 0).reshape(-1)``.
    Internally the array is built z-major ([z][y][x]) so ``reshape(-1)``
    of the internal tensor already is x-fastest raster order.
    """
    nz = n if nz is None else nz
    gen = _gen(seed, device)
    white = torch.randn((nz, n, n), generator=gen, device=device, dtype=torch.float32)
    spec = torch.fft.rfftn(white)
    del white
    kz = torch.fft.fftfreq(nz, d=1.0 / nz, device=device).view(nz, 1, 1)
    ky = torch.fft.fftfreq(n, d=1.0 / n, device=device).view(1, n, 1)
    kx = torch.fft.rfftfreq(n, d=1.0 / n, device=device).view(1, 1, n // 2 + 1)
    kk = torch.sqrt(kx * kx + ky * ky + kz * kz)
    amp = torch.where(kk > 0, kk.clamp_min(1e-12) ** (slope / 2.0), torch.zeros_like(kk))
    if kmax is not None:
        amp = torch.where(kk > kmax, torch.zeros_like(amp), amp)
    spec *= amp
    del amp, kk
    field = torch.fft.irfftn(spec, s=(nz, n, n))
    del spec
    return field  # [z][y][x]


def _minmax01(f):
    lo = f.min()
    hi = f.max()
    return (f - lo) / (hi - lo)


def _blobs(shape_zyx, count, sig_lo, sig_hi, amp_lo, amp_hi, seed, device):
    nz, ny, nx = shape_zyx
    rng = np.random.default_rng(seed)
    out = torch.zeros(shape_zyx, dtype=torch.float32, device=device)
    z = torch.arange(nz, device=device, dtype=torch.float32).view(nz, 1, 1)
    y = torch.arange(ny, device=device, dtype=torch.float32).view(1, ny, 1)
    x = torch.arange(nx, device=device, dtype=torch.float32).view(1, 1, nx)
    for _ in range(count):
        cx, cy, cz = rng.uniform(0, nx), rng.uniform(0, ny), rng.uniform(0, nz)
        sig = rng.uniform(sig_lo, sig_hi)
        a = rng.uniform(amp_lo, amp_hi)
        out += a * torch.exp(-(((x - cx) ** 2) + ((y - cy) ** 2) + ((z - cz) ** 2)) / (2.0 * sig * sig))
    return out


def percentile(flat: torch.Tensor, q: float) -> float:
    """Linear-interpolation percentile (numpy's default method) in f64."""
    n = flat.numel()
    s = torch.sort(flat.reshape(-1).to(torch.float64)).values
    pos = (q / 100.0) * (n - 1)
    lo = int(math.floor(pos))
    hi = min(lo + 1, n - 1)
    t = pos - lo
    a = float(s[lo])
    b = float(s[hi])
    d = b - a
    return b - d * (1.0 - t) if t >= 0.5 else a + d * t


CONFIGS = {
    "c1": dict(n=64, bs=16, r=1e-3),
    "c2": dict(n=256, bs=16, r=1e-3),
    "c3": dict(n=512, bs=32, r=1e-3),
    "c4": dict(n=1024, bs=32, r=1e-4),
    "c5": dict(n=1536, bs=32, r=1e-4),
}


def make_config(name: str, device="cpu", seed=0, n=None, quantile=None, r=None, nz=None):
    """Returns (values float32 flat x-fastest tensor, dims, bs, candidates, loose_fraction).

    ``n`` overrides the edge length (tests run the configs' recipes at small n);
    ``nz`` gives slab volumes (n, n, nz) for weak scaling.
    """
    cfg = dict(CONFIGS[name])
    n = cfg["n"] if n is None else n
    nz = n if nz is None else nz
    bs, rr = cfg["bs"], cfg["r"] if r is None else r
    if name == "c1":
        f = _blobs((nz, n, n), 8, 4.0, 12.0, 0.5, 1.0, seed, device)
        gen = _gen(seed + 1, device)
        f += (torch.rand(f.shape, generator=gen, device=device) * 2.0 - 1.0) * 1e-3
        f = f.to(torch.float32)
        cands = [0.5 * float(f.max())]
    elif name == "c2":
        f = _minmax01(grf(n, -11.0 / 3.0, seed, kmax=32, device=device, nz=nz)).to(torch.float32)
        cands = [percentile(f, 50.0 if quantile is None else quantile)]
    elif name == "c3":
        g = grf(n, -3.0, seed, device=device, nz=nz)
        g = (g - g.mean()) / g.std()
        f = torch.exp(1.5 * g).to(torch.float32)
        del g
        cands = [percentile(f, 99.0 if quantile is None else quantile)]
    elif name == "c4":
        f = _minmax01(grf(n, -11.0 / 3.0, seed, device=device, nz=nz)).to(torch.float32)
        cands = [0.5]
    elif name == "c5":
        f = grf(n, -11.0 / 3.0, seed, device=device, nz=nz)
        f = (f - f.mean()) / f.std()
        f += _blobs((nz, n, n), 64, 8.0, 48.0, 0.5, 1.0, seed, device) * 3.0
        f = _minmax01(f).to(torch.float32)
        cands = [float(v) for v in np.linspace(0.05, 0.95, 16)]
    else:
        raise KeyError(name)
    return f.reshape(-1).contiguous(), (n, n, nz), bs, cands, rr
