"""Instruction / stall shares of one kernel by source-line ranges (phases).
    python tools/ncu_phases.py report.ncu-rep kernel_regex name:lo-hi [name:lo-hi ...]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
phases = []
for a in sys.argv[3:]:
    name, rng = a.split(":")
    lo, hi = rng.split("-")
    phases.append((name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern,
                      "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[h]
ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cur, agg = None, {}
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0] and not r[0].startswith("0x"):
        try:
            cur = int(r[0])
        except ValueError:
            cur = None
        continue
    if cur is None:
        continue
    ph = next((n for n, lo, hi in phases if lo <= cur <= hi), "other")
    a = agg.setdefault(ph, [0, 0])
    try:
        a[0] += int(r[ii] or 0)
        a[1] += int(r[si] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:12s} {v[0] / tot * 100:5.1f}% inst {v[1] / ts * 100:5.1f}% stall")
