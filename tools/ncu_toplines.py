"""Top CUDA source lines of one kernel by instructions executed and stall samples.
    python tools/ncu_toplines.py report.ncu-rep kernel_regex [N]"""
import csv
import io
import os
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern,
                      "-c", "1"], capture_output=True, text=True).stdout
fname, hdr, agg, tot = "?", None, [], [0, 0]
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r[0].isdigit() or len(r) <= ii:
        continue
    try:
        n, s = int(r[ii] or 0), int(r[si] or 0)
    except ValueError:
        continue
    tot[0] += n
    tot[1] += s
    agg.append((n, s, f"{fname}:{r[0]}", r[1].strip()[:90]))
print(f"total {tot[0] / 1e6:.1f}M inst, {tot[1]} stall samples")
for n, s, l, t in sorted(agg, key=lambda x: -x[0])[:topn]:
    print(f"{l:>22} {n / 1e6:7.1f}M {100 * n / tot[0]:5.1f}%  st {100 * s / max(tot[1], 1):5.1f}%  {t}")
