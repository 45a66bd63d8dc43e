"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list.
    python tools/ncu_launches.py launches.csv [out.md] [steps]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
agg = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) < len(hdr) or r[mn] != "gpu__time_duration.sum":
        continue
    name = r[kn].split("(")[0].replace("void ", "")
    if not (name.startswith("chr::") or "::k_" in name or name.startswith("k_")):
        continue  # synthetic-input generation, torch kernels
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[mv].replace(",", "")) / 1e6
tot = sum(v[1] for v in agg.values())
lines = ["| kernel | launches | total ms | ms / step | share |", "|---|---|---|---|---|"]
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| `{k}` | {c} | {t:.3f} | {t / steps:.3f} | {100 * t / tot:.1f} % |")
lines.append(f"| **all chr kernels** | {sum(v[0] for v in agg.values())} | {tot:.3f} | {tot / steps:.3f} | 100 % |")
txt = "\n".join(lines)
print(txt)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(
        f"# ncu launch list (`gpu__time_duration.sum`, --clock-control none, serialised, cold caches)\n\n"
        f"Source: `{sys.argv[1]}`; {steps} pipeline step(s) captured (`tools/prof_r02.sh`: one warm c3 step of `tools/one_step.py` between cudaProfilerStart/Stop).\n"
        f"Per-launch times are cold-cache and serialised, so compare SHARES with the bench's CUDA-event table.\n\n"
        + txt + "\n")
