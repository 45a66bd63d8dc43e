"""Per-CUDA-source-line instruction and stall shares of one kernel in an ncu report.
    python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[h]
ii, si, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
cur, agg = None, {}
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0] and not r[0].startswith("0x"):
        cur = (r[0], r[src][:100])
        continue
    try:
        a = agg.setdefault(cur, [0, 0])
        a[0] += int(r[ii] or 0)
        a[1] += int(r[si] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-inst {tot/1e6:.0f}M, stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] / tot + kv[1][1] / ts))[:top]:
    print(f"{v[0]/tot*100:5.1f}% inst {v[1]/ts*100:5.1f}% stall  L{k[0]}: {k[1]}")
