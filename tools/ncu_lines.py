"""Instruction / stall totals of a kernel grouped by CUDA source line ranges.
    python tools/ncu_lines.py report.ncu-rep kernel_regex a-b:name c-d:name ..."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    r, name = spec.split(":")
    a, b = r.split("-")
    ranges.append((int(a), int(b), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[h]
ii, si, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
line = None
agg = {}
tot = [0, 0]
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0] and not r[0].startswith("0x"):
        try:
            line = int(r[0])
        except ValueError:
            line = None
        continue
    try:
        n, s = int(r[ii] or 0), int(r[si] or 0)
    except ValueError:
        continue
    tot[0] += n
    tot[1] += s
    name = "other"
    for a, b, nm in ranges:
        if line is not None and a <= line <= b:
            name = nm
            break
    x = agg.setdefault(name, [0, 0])
    x[0] += n
    x[1] += s
for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:12s} {n / 1e6:8.1f}M inst {100 * n / tot[0]:5.1f}%  stall {100 * s / tot[1]:5.1f}%")
