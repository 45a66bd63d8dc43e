"""Per-source-line instruction / stall totals of one kernel from an ncu report
(run here, no GPU):  python tools/ncu_srclines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
agg = {}
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        n, s = int(r[ii]), int(r[si])
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0, 0, r[1].strip()[:90]])
    a[0] += n
    a[1] += s
tot = sum(v[0] for v in agg.values()) or 1
stot = sum(v[1] for v in agg.values()) or 1
print(f"total {tot / 1e6:.1f}M inst, {stot} stall samples")
for (f, ln), (n, s, t) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f:>16s}:{ln:<5d} {n / 1e6:8.1f}M {100 * n / tot:5.1f}%  st {100 * s / stot:5.1f}%  {t}")
