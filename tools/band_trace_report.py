"""Summary of a k_band phase trace (tools/band_trace.sh): mean per-tile phase
durations, their share of tile time, concurrency and wait percentiles.
    python tools/band_trace_report.py gpurun_out/band_trace.bin"""
import sys

import numpy as np

a = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/band_trace.bin", dtype=np.uint64)
a = a.reshape(-1, 8).astype(np.int64)
a = a[a[:, 1] > 0]
t0 = a[:, 1].min()
st, sc, xy, fa, fc, pub, end = [a[:, i] for i in range(1, 8)]


def us(x, y):
    return (y - x) / 1e3


tot = us(st, end).sum()
print(f"tiles {len(a)}  kernel span {us(t0, end.max()):.1f} us  mean tile {us(st, end).mean():.2f} us")
for name, x, y in (("scatter", st, sc), ("x/y prefix", sc, xy), ("face waits + dF", xy, fc), ("publish", fc, pub),
                   ("recon + mask", pub, end)):
    print(f"  {name:16s} mean {us(x, y).mean():6.2f} us  share {us(x, y).sum() / tot:.2f}")
ev = np.concatenate([np.stack([st, np.ones_like(st)], 1), np.stack([end, -np.ones_like(end)], 1)])
ev = ev[np.argsort(ev[:, 0], kind="stable")]
c = np.cumsum(ev[:, 1])
dt = np.diff(ev[:, 0])
print(f"  concurrent tiles: mean {(c[:-1] * dt).sum() / dt.sum():.1f}  max {c.max()}")
print("  wait percentiles (50/90/99/max us):", np.percentile(us(xy, fc), [50, 90, 99, 100]).round(1).tolist())
