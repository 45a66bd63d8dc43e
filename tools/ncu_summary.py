"""Summarise an ncu report (run here, no GPU): per kernel duration, DRAM bytes,
achieved DRAM GB/s, SM/memory throughput, instructions, registers.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [out.md] [traffic.json]"""
import csv
import io
import json
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
     "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics", ",".join(M)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def main():
    rep = sys.argv[1]
    rows = load(rep)
    lines = ["| kernel | ms | DRAM rd MB | DRAM wr MB | DRAM GB/s | DRAM % | SM % | warp-inst (M) | regs | grid |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d in rows:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        t = float(d["gpu__time_duration.sum"]) * 1e-9  # ns
        rd = float(d["dram__bytes_read.sum"])
        wr = float(d["dram__bytes_write.sum"])
        lines.append(f"| {name} | {t*1e3:.3f} | {rd/1e6:.1f} | {wr/1e6:.1f} | {(rd+wr)/t/1e9:.0f} | "
                     f"{float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                     f"{float(d['sm__throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                     f"{float(d['smsp__inst_executed.sum'])/1e6:.0f} | {d['launch__registers_per_thread']} | "
                     f"{d['launch__grid_size']} |")
        traffic[name.replace("<float, 0>", "<float, false>").replace("<float, 1>", "<float, true>")] = rd + wr
    txt = "\n".join(lines)
    print(txt)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(f"# ncu summary of `{rep}`\n\n{txt}\n")
    if len(sys.argv) > 3:
        json.dump(traffic, open(sys.argv[3], "w"), indent=1)


if __name__ == "__main__":
    main()
