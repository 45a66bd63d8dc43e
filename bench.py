#!/usr/bin/env python
"""Benchmark of the CHR hot path on B200 (BASELINE.json metric).

One STEP = the whole north_star path over one synthetic volume:
    compress  (stats -> plan -> quantise/Lorenzo/tokens -> .chr file, on device)
 -> request   (selective decode of the regions relevant to k)
 -> extract   (marching cubes of the selected windows, merged mesh)
Workload at N=1: BASELINE config c3 (512^3 f32 lognormal exp(1.5 g),
P(k)~k^-3, bs32, r=1e-3, k = 99th percentile), the config the north_star
target is stated on.  value = 4*N / t_step (GB/s of f32 input through the
whole path), inputs resident in HBM; `e2e` is the same metric with the
input host->device copy and the archive + mesh device->host copies inside
the timed region (chr_pipeline, pipelined); `e2e_api` times the drop-in API
a reference user calls (Volume from host numpy -> build_chr -> request ->
marching_cubes per region -> merge_meshes, pipeline.py:121-202).  Stage
throughputs and per-stage rooflines follow SURVEY §8(d).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: ``python bench.py --gpus N`` launches N ranks itself (torchrun,
127.0.0.1) unless WORLD_SIZE is already set.  Default N>1 workload: one
c3-recipe volume of 512 x 512 x 512N in z-slabs, one 512^3 slab per GPU
(weak scaling: per-GPU work = the N=1 workload) through the distributed
path of SURVEY §8(e): z-slab compress (all-gathers of block stats, stream
summaries, CRC shares) and per-portion request + marching cubes (all-gathers
of region z-carries, boundary planes and mesh counts; no payload bytes move).
``--scaling strong --config c4``: one 1024^3 volume split over the N GPUs.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CHR compress/decompress GB/s + isosurface cells/s, % of HBM roofline, 1–8 GPU"
FALLBACK_HBM = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class Clocks:
    """SM clock and throttle-reason sampling during the timed region
    (B200_PROFILING.md): NVML polled every 5 ms from a thread (a c3 timed
    region is ~70 ms, shorter than nvidia-smi's start-up), nvidia-smi -lms as
    the fallback when NVML is absent."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (N, h)
            self.mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self._sample_nvml()  # one sample before the region starts
            self.rows.clear()
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _sample_nvml(self):
        N, h = self.nvml
        sm = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
        rs = int(N.nvmlDeviceGetCurrentClocksEventReasons(h))
        self.rows.append([str(sm), str(self.mx), hex(rs)] +
                         ["Active" if rs & self.BITS[n] else "Not Active" for n in
                          ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")])

    def _poll_nvml(self):
        while True:
            try:
                self._sample_nvml()
            except Exception:
                return
            if self.stop.wait(0.005):
                return

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=1)
            try:
                self._sample_nvml()  # the region's last moment
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": "nvml" if self.nvml else "nvidia-smi"}


def make_input(cfg, n, rank, device):
    from paper_2408_05462_b200 import synth

    vals, dims, bs, cands, r = synth.make_config(cfg, device=device, n=n, seed=rank)
    return vals, dims, bs, cands, r


def run_step(vol, dims, bs, cands, r, ws, spacing=(1.0, 1.0, 1.0), stage_events=None, after_compress=None,
             light=False):
    """compress -> request(k) -> marching cubes, all device resident, in one
    library call (device.pipeline -> chr_pipeline: the same bytes, windows
    and mesh as build_archive + decode + marching, without host round trips
    between the phases); returns sizes.  ``after_compress(archive)`` runs as
    soon as the archive exists (the e2e loop starts its device->host copy
    there, overlapping request + extract).  stage_events: 4 CUDA events
    recorded at the start, after compress, after decode, after the mesh."""
    from paper_2408_05462_b200 import device as D

    p = D.pipeline(vol, dims, cands, bs, loose_fraction=r, k_index=0, spacing=spacing, ws=ws,
                   stage_events=stage_events, after_compress=after_compress)
    if light:  # timed loops: outputs only (the region statistics below are bench bookkeeping)
        return dict(archive_view=p.archive, verts=p.verts, tris=p.tris, archive=int(p.archive.numel()),
                    ntri=int(p.tris.shape[0]), nvert=int(p.verts.shape[0]))
    regs = p.regions
    sel = regs[(regs["mask"] & np.uint64(1)) != 0]  # regions relevant to candidate 0
    ext = sel["extent"].astype(np.int64)
    return dict(archive_view=p.archive, wins=p.windows, verts=p.verts, tris=p.tris,
                n_sel=int(np.prod(ext, axis=1).sum()), cells=int(np.prod(ext - 1, axis=1).sum()),
                c_sel=int(sel["block_nbytes"].sum()), archive=int(p.archive.numel()), nreg=len(regs),
                n_all=int(np.prod(regs["extent"].astype(np.int64), axis=1).sum()), nsel=len(sel),
                ntri=int(p.tris.shape[0]), nvert=int(p.verts.shape[0]), payload=int(regs["block_nbytes"].sum()))


def timed_lanes(args, lanes, local, vals, dims, bs, cands, r, ws, info):
    """The same K steps as the serial timed loop, dealt to `lanes` host
    threads, each with its own stream and workspaces (a serving process
    keeps several volumes in flight): one step's host syncs (the block
    statistics read-back before the plan, the mesh-size read-back) and
    launch gaps are filled by another step's kernels.  Timed on the device:
    a start event on the launching thread's stream that every lane waits on,
    and a stop event after every lane's last kernel.  Every step's triangle
    count is checked against the serial run's."""
    from paper_2408_05462_b200 import device as D

    wss = [ws] + [D.Workspaces() for _ in range(lanes - 1)]
    sts = [torch.cuda.Stream() for _ in range(lanes)]
    share = [args.steps // lanes + (1 if i < args.steps % lanes else 0) for i in range(lanes)]
    go = torch.cuda.Event()
    ends = [torch.cuda.Event() for _ in range(lanes)]
    bad = []

    def lane(i, nsteps, timed):
        torch.cuda.set_device(local)
        with torch.cuda.stream(sts[i]):
            if timed:
                sts[i].wait_event(go)
            for _ in range(nsteps):
                out = run_step(vals, dims, bs, cands, r, wss[i], light=True)
                if out["ntri"] != info["ntri"] or out["archive"] != info["archive"]:
                    bad.append((i, out["ntri"], out["archive"]))
            ends[i].record()

    def run(counts, timed):
        th = [threading.Thread(target=lane, args=(i, counts[i], timed)) for i in range(lanes)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    run([1] * lanes, False)  # each lane's workspaces sized once, untimed
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        start.record()
        go.record()
        run(share, True)
        cur = torch.cuda.current_stream()
        for e in ends:
            cur.wait_event(e)
        stop.record()
        torch.cuda.synchronize()
    if bad:
        raise RuntimeError(f"lane steps differ from the serial step: {bad[:4]}")
    return start.elapsed_time(stop) / args.steps, clk


def kernel_bytes(name, info, N):
    """Algorithmic bytes per launch of the main kernels: each
    kernel's share of its stage's algorithmic bytes -- input reads, archive /
    window / mesh writes -- never the design's own intermediates (token
    values, piece records, faces), so a kernel that only moves an
    intermediate has none (None)."""
    c_all = info["archive"]
    table = {
        "k_stats<float>": 4 * N,                # stats read (compress: 8N + C)
        "k_stats_rows": 4 * N,
        "k_quant<float>": 4 * N,                # encode read
        "k_qseg<float>": 4 * N,
        "k_emit_q<float>": c_all,               # archive write
        "k_qemit<float>": c_all,
        "k_tok_fast": info["c_sel"],            # selected payload read (decompress: C_sel + 8 N_sel)
        "k_band": info["c_sel"] + 8 * info["n_sel"],
        "k_lorenzo": info["c_sel"] + 8 * info["n_sel"],
        "k_mc_emit4": 24 * info["nvert"] + 12 * info["ntri"],  # mesh write (MC: 8 N_sel + 24 nv + 12 nt)
    }
    return table.get(name)


def stage_roofline(t_ms, alg_bytes, peak):
    gbs = alg_bytes / (t_ms * 1e-3) / 1e9
    return {"ms": t_ms, "algorithmic_bytes": int(alg_bytes), "achieved_gbs": gbs, "frac": gbs / peak}


def workload_name(config, n, bs, r, cands):
    return (f"{config}: {n}^3 f32 " + {
        "c3": "lognormal exp(1.5 g), g unit-variance GRF P(k)~k^-3", "c4": "GRF P(k)~k^-11/3 [0,1]",
        "c2": "GRF P(k)~k^-11/3 |k|<=32 [0,1]", "c1": "8 Gaussian blobs + noise",
        "c5": "GRF + 64 blobs"}.get(config, "") +
        f", bs{bs}, r={r}, k={cands[0]:.6g}; step = compress -> request(k) -> marching cubes")


def cpu_baseline(vals_host, dims, bs, cands, r, planes, workers, repeats=3):
    """The reference's CPU path (isochr from baseline/_ref when installed,
    else the oracle port) on host cores, on a bounded z-slab sample."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import cpu_reference  # noqa: PLC0415

    return cpu_reference.time_stages(vals_host, dims, bs, cands[0], r, planes, workers, repeats)


def api_e2e(vals, dims, bs, cands, r, steps):
    """The drop-in path timed end to end (pipeline.py:121-202 calls): a host
    numpy field -> Volume -> build_chr -> request(k) -> marching_cubes per
    selected region -> merge_meshes, every result back on the host as the
    reference's dataclasses.  One warm-up call, then the median of `steps`."""
    import paper_2408_05462_b200 as G  # noqa: PLC0415

    host = vals.cpu().numpy()
    k = cands[0]

    def run():
        vol = G.Volume(dims, values=host, source_dtype="f32")
        arch = G.build_chr(vol, [k], bs, loose_fraction=r)
        rs = G.request(arch, k)
        meshes = [G.marching_cubes(win, vol.spacing, tuple(o * sp for o, sp in zip(reg.sample_origin, vol.spacing)), k)
                  for reg, win in rs.regions]
        return G.merge_meshes(meshes)

    run()
    ts = []
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = run()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    n = dims[0] * dims[1] * dims[2]
    return {"value": 4 * n / t / 1e9, "unit": "GB/s", "ms_per_step": t * 1e3, "steps": steps,
            "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": None, "triangles": int(m.num_triangles),
            "path": "Volume(host f32) -> build_chr -> request -> marching_cubes per region -> merge_meshes "
                    "(host numpy results, reference dataclasses); wall clock, median"}


def launch_ranks(args) -> int:
    """``--gpus N`` without torchrun: start N ranks on this node (127.0.0.1)."""
    if torch.cuda.device_count() < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus}: only {torch.cuda.device_count()} "
                                                      "CUDA device(s) visible"}), flush=True)
        return 1
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--edge", "--size", dest="n", type=int, default=None, help="edge length override (tests)")
    ap.add_argument("--cpu-planes", type=int, default=128,
                    help="CPU baseline sample: first P z-planes of the volume (0 = the whole volume)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-copy", default="dma", choices=["dma", "sm"],
                    help="bulk H2D/D2H of the e2e loop: DMA engines or the UVA copy kernel")
    ap.add_argument("--mode", default="slab", choices=["replica", "slab"],
                    help="N>1: one volume in z-slabs (SURVEY 8e, default) or independent volumes per rank")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="slab mode: n x n x nN volume (weak) or one n^3 volume split over the ranks (strong)")
    ap.add_argument("--no-api-e2e", action="store_true", help="skip the drop-in API e2e timing")
    ap.add_argument("--lanes", type=int, default=1,
                    help="host threads (own stream + workspaces each) sharing the K device-resident steps")
    ap.add_argument("--dist1", action="store_true",
                    help="run the distributed (slab) path even at N=1 (one NCCL rank)")
    ap.add_argument("--backend", default=None, help="torch.distributed backend (default nccl; gloo for 1-GPU tests)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1 or args.dist1:
        import torch.distributed as dist

        torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
        if world == 1:  # --dist1: the distributed path on one rank (NCCL branches exercised)
            import socket

            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            dist.init_process_group(args.backend or "nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                    world_size=1)
        else:
            dist.init_process_group(args.backend or "nccl")
    else:
        torch.cuda.set_device(0)

    from paper_2408_05462_b200 import _abi, synth
    from paper_2408_05462_b200 import device as D

    n = args.n or synth.CONFIGS[args.config]["n"]
    workers = len(os.sched_getaffinity(0))

    if args.impl == "reference":
        # the reference's CPU path on host cores: the reference package itself
        # (isochr + numba, installed under baseline/_ref) or, absent, the oracle port
        if rank != 0:
            if dist:
                dist.barrier()
            return
        vals, dims, bs, cands, r = make_input(args.config, n, rank, "cuda")
        host = vals.cpu().numpy()
        del vals
        times = []
        for i in range(args.warmup + args.steps):  # a step = one run of the sample, every stage once
            cb = cpu_baseline(host, dims, bs, cands, r, args.cpu_planes, workers, repeats=1)
            if i >= args.warmup:
                times.append(cb)
        v = statistics.median([t["value"] for t in times])
        pz = min(args.cpu_planes, dims[2]) if args.cpu_planes > 0 else dims[2]
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 4 * dims[0] * dims[1] * pz / v / 1e6,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded torch GRF; no public dataset)",
                "config": {"workload": workload_name(args.config, n, bs, r, cands), "dims": list(dims),
                           "block_size": bs, "cpu_sample_planes": pz},
                "cpu_baseline": dict(times[-1], value=v),
                "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        if dist:
            dist.barrier()
        return

    if dist and args.mode == "slab":
        return slab_main(args, dist, rank, world, local, n, workers)

    vals, dims, bs, cands, r = make_input(args.config, n, rank, "cuda")
    N = dims[0] * dims[1] * dims[2]
    ws = D.Workspaces()
    host_in = torch.empty(N, dtype=torch.float32, pin_memory=True)
    host_in.copy_(vals)
    L = _abi.lib()

    # warm-up (also validates the path once)
    for _ in range(args.warmup):
        info = run_step(vals, dims, bs, cands, r, ws)
    torch.cuda.synchronize()

    # ---- timed, device resident
    stage = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = L.chr_launch_count()
    from paper_2408_05462_b200 import multi
    with Clocks(local) as clk:
        start.record()
        for i in range(args.steps):
            out = run_step(vals, dims, bs, cands, r, ws, stage_events=stage[i], light=True)
            if dist:  # the exchange step: global offsets of every rank's outputs
                multi.place(out["archive"], out["ntri"], out["nvert"], device="cuda")
        stop.record()
        torch.cuda.synchronize()
    launches = L.chr_launch_count() - l0
    ms = start.elapsed_time(stop) / args.steps
    ms_1lane = ms
    lanes = 1 if dist else max(1, args.lanes)
    if lanes > 1:
        ms, clk = timed_lanes(args, lanes, local, vals, dims, bs, cands, r, ws, info)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # per-kernel CUDA-event times: the same K steps again with the library's
    # profiler on (its event records cost ~0.3 ms of host time per step, so
    # the step time above is taken without it)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    L.chr_prof_enable(1)
    _abi.prof_report()  # clear
    pstart = torch.cuda.Event(enable_timing=True)
    pstop = torch.cuda.Event(enable_timing=True)
    pstart.record()
    for i in range(args.steps):
        run_step(vals, dims, bs, cands, r, ws, light=True)
    pstop.record()
    torch.cuda.synchronize()
    L.chr_prof_enable(0)
    kern = _abi.prof_report()
    ms_prof = pstart.elapsed_time(pstop) / args.steps
    st = [(s[0].elapsed_time(s[1]), s[1].elapsed_time(s[2]), s[2].elapsed_time(s[3])) for s in stage]
    t_c = statistics.median(x[0] for x in st)
    t_d = statistics.median(x[1] for x in st)
    t_m = statistics.median(x[2] for x in st)

    # ---- e2e through host buffers: every step copies its input in (pinned host
    #      -> device) and its archive + mesh out (device -> pinned host).  Steps
    #      are pipelined on three streams (the H2D of step i+1 and the D2H of
    #      step i overlap step i's compute; inputs, workspaces and host outputs
    #      double-buffered), and the K timed steps run from an empty pipeline:
    #      e2e = (first H2D start .. last D2H end) / K.
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    wss = [ws, D.Workspaces()]
    dvols = [torch.empty_like(vals), torch.empty_like(vals)]
    hout = [(torch.empty(info["archive"] + 1024, dtype=torch.uint8, pin_memory=True),
             torch.empty(info["nvert"] * 3 + 16, dtype=torch.float64, pin_memory=True),
             torch.empty(info["ntri"] * 3 + 16, dtype=torch.int32, pin_memory=True)) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    h2d = d2h = 0

    def chunked(dst, src):
        """bulk copy on the DMA engines (full duplex over PCIe); the library's own small
        transfers bypass the engines (xfer.cu), so they never queue behind these.
        --e2e-copy sm: a 16-CTA UVA copy kernel (chr_sm_copy) instead"""
        if args.e2e_copy == "dma":
            dst.copy_(src, non_blocking=True)
            return
        nbytes = dst.numel() * dst.element_size()
        rc = L.chr_sm_copy(dst.data_ptr(), src.data_ptr(), nbytes, 16, torch.cuda.current_stream().cuda_stream)
        if rc:
            raise RuntimeError(f"chr_sm_copy failed ({rc})")

    def pipeline(nsteps, timed):
        nonlocal h2d, d2h
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s_in):
            t0.record()
            chunked(dvols[0], host_in)
            ev_in[0].record()
        for i in range(nsteps):
            bi = i % 2
            if i + 1 < nsteps:  # prefetch the next step's input
                nb = (i + 1) % 2
                with torch.cuda.stream(s_in):
                    if i >= 1:
                        s_in.wait_event(ev_used[nb])
                    chunked(dvols[nb], host_in)
                    ev_in[nb].record()
            ha, hv, ht = hout[bi]

            def archive_out(archive, bi=bi, ha=ha):
                # the archive leaves while request + extract run
                ev_arch = torch.cuda.Event()
                ev_arch.record(s_cmp)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_arch)
                    chunked(ha[: archive.numel()], archive)

            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[bi])
                if i >= 2:
                    s_cmp.wait_event(ev_out[bi])  # step i-2's outputs have left workspace bi
                inf = run_step(dvols[bi], dims, bs, cands, r, wss[bi], after_compress=archive_out, light=True)
                ev_used[bi].record()
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_used[bi])
                nbytes = inf["archive"]
                chunked(hv[: inf["nvert"] * 3], inf["verts"].reshape(-1))
                chunked(ht[: inf["ntri"] * 3], inf["tris"].reshape(-1))
                ev_out[bi].record()
            h2d = 4 * N
            d2h = nbytes + 24 * inf["nvert"] + 12 * inf["ntri"]
        with torch.cuda.stream(s_out):
            t1.record()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / nsteps

    pipeline(args.warmup, False)
    e2e_ms = [pipeline(args.steps, True)]
    e2e = statistics.median(e2e_ms)
    if dist:
        t = torch.tensor([e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())

    # ---- roofline of the dominant kernel
    peak, peak_src = _peaks()
    dom = max(kern.items(), key=lambda kv: kv[1][1]) if kern else None
    roof = None
    if dom:
        name, (cnt, tot) = dom
        alg = kernel_bytes(name, info, N)
        avg = tot / cnt
        achieved = alg / (avg * 1e-3) / 1e9 if alg else None
        traffic = None  # dram bytes of the same kernel on the same config (one ncu --set full capture)
        tp = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
        if os.path.exists(tp) and args.n is None:
            try:
                traffic = json.load(open(tp)).get(name)
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "algorithmic_bytes": alg, "avg_ms": avg, "launches_per_step": cnt / args.steps,
                "share_of_step": tot / args.steps / ms_prof, "peak_source": peak_src,
                "timed": "K profiled steps after the K timed steps (CUDA events around each launch)"}
    kern_tab = {k: {"launches": c, "avg_ms": t / c, "share": t / args.steps / ms_prof,
                    "gbs": (kernel_bytes(k, info, N) / (t / c * 1e-3) / 1e9) if kernel_bytes(k, info, N) else None}
                for k, (c, t) in sorted(kern.items(), key=lambda kv: -kv[1][1])}

    # per-stage rooflines on SURVEY §8(d)'s algorithmic bytes
    stage_roof = {
        "compress": stage_roofline(t_c, 8 * N + info["archive"], peak),
        "decompress": stage_roofline(t_d, info["c_sel"] + 8 * info["n_sel"], peak),
        "marching_cubes": stage_roofline(t_m, 8 * info["n_sel"] + 24 * info["nvert"] + 12 * info["ntri"], peak),
        "step": stage_roofline(ms, 8 * N + info["archive"] + info["c_sel"] + 16 * info["n_sel"] +
                               24 * info["nvert"] + 12 * info["ntri"], peak),
        "peak_gbs": peak, "peak_source": peak_src,
    }

    # drop-in API e2e: what a reference user calls, host numpy in and out
    api = None
    if not args.no_api_e2e:
        api = api_e2e(vals, dims, bs, cands, r, max(1, min(args.steps, 3)))

    cpu = cpu1 = None
    if rank == 0 and not args.no_cpu_baseline:
        host_vals = vals.cpu().numpy()
        cpu = cpu_baseline(host_vals, dims, bs, cands, r, args.cpu_planes, workers)
        cpu1 = cpu_baseline(host_vals, dims, bs, cands, r, args.cpu_planes, 1)

    value = world * 4 * N / (ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded torch GRF; no public dataset)",
        "ms_per_step_1lane": ms_1lane,
        "config": {
            "workload": workload_name(args.config, n, bs, r, cands),
            "lanes": lanes,
            "dims": list(dims), "block_size": bs, "regions": info["nreg"], "regions_selected": info["nsel"],
            "archive_bytes": info["archive"], "selected_samples": info["n_sel"], "cells": info["cells"],
            "triangles": info["ntri"], "vertices": info["nvert"],
            "l2": "no flush: input (4N bytes) and decoded windows (8 N_sel bytes) are each larger than the 126 MB L2",
        },
        "stages": {
            "compress_ms": t_c, "compress_gbs": 4 * N / (t_c * 1e-3) / 1e9,
            "request_ms": t_d, "decompress_gbs": 4 * info["n_sel"] / (t_d * 1e-3) / 1e9,
            "mc_ms": t_m, "mc_cells_per_s": info["cells"] / (t_m * 1e-3),
            "roofline": stage_roof,
        },
        "kernels": kern_tab,
        "roofline": roof,
        "cpu_baseline": cpu,
        "cpu_baseline_1core": cpu1,
        "e2e_api": api,
        "e2e": {"value": world * 4 * N / (e2e * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "ms_per_step_profiled": ms_prof,  # the kernel table's K steps (library profiler on)
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def slab_main(args, dist, rank, world, local, n, workers):
    """N>1, one volume in z-slabs: weak scaling n x n x (n N)
    (default: per-GPU work = the N=1 workload) or strong scaling n^3 split
    over the ranks.  Step = distributed compress (block-stats / stream-summary
    / CRC-share all-gathers; every rank writes its slice of the file) ->
    per-portion request + marching cubes (every rank decodes and meshes its
    own planes; all-gathers of z-carry planes, boundary planes, CRC shares
    and mesh counts; no payload bytes move).  Times are the max over ranks."""
    from paper_2408_05462_b200 import _abi, multi, synth
    from paper_2408_05462_b200 import device as D

    nz_total = n * world if args.scaling == "weak" else n
    full, dims, bs, cands, r = synth.make_config(args.config, device="cuda", n=n, nz=nz_total, seed=0)
    nx, ny, nz = dims
    slab = multi.slab_of(nz, bs, world, rank)
    vol = full[slab.z_base * nx * ny: (slab.z_base + slab.nz_local) * nx * ny].clone()
    del full
    torch.cuda.empty_cache()
    ws = D.Workspaces()
    L = _abi.lib()
    k = cands[0]

    def step(ev=None, v=None):
        if ev:
            ev[0].record()
        res = multi.build_archive_slab(vol if v is None else v, dims, slab, cands, bs, loose_fraction=r, ws=ws)
        if ev:
            ev[1].record()
        m = multi.request_extract_portions(res, 0, k, ws=ws)
        if ev:
            ev[2].record()
        return res, m

    for _ in range(args.warmup):
        res, m = step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = L.chr_launch_count()
    with Clocks(local % max(1, torch.cuda.device_count())) as clk:
        a.record()
        for i in range(args.steps):
            res, m = step(evs[i])
        b.record()
        torch.cuda.synchronize()
    launches = L.chr_launch_count() - l0

    def maxr(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = maxr(a.elapsed_time(b) / args.steps)
    st = [(e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])) for e in evs]
    t_c = maxr(statistics.median(x[0] for x in st))
    t_rm = maxr(statistics.median(x[1] for x in st))
    # per-kernel table: the same K steps again with the library's profiler on
    dist.barrier()
    torch.cuda.synchronize()
    L.chr_prof_enable(1)
    _abi.prof_report()
    for i in range(args.steps):
        step()
    torch.cuda.synchronize()
    L.chr_prof_enable(0)
    kern = _abi.prof_report()
    # e2e: H2D of this rank's slab, D2H of its mesh rows and its share of the file
    host_in = torch.empty(vol.numel(), dtype=torch.float32, pin_memory=True)
    host_in.copy_(vol)
    dvol = torch.empty_like(vol)
    e2e = []
    h2d = d2h = 0
    for i in range(args.warmup + args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        dvol.copy_(host_in, non_blocking=True)
        res, m = step(v=dvol)
        hv = m.verts.cpu()
        ht = m.tris.cpu()
        contrib = multi.contributors(res.regions, dims, bs, world)[:, rank]
        rs = res.regions[contrib]
        parts = [res.blob[int(o): int(o) + int(c)] for o, c in zip(rs["block_offset"], rs["block_nbytes"])]
        if rank == 0:
            parts.append(res.blob[: D.header_table_nbytes(len(cands), len(res.regions))])
        hf = torch.cat(parts).cpu() if parts else None
        eb.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e.append(ea.elapsed_time(eb))
        h2d = 4 * vol.numel()
        d2h = int(hv.numel() * 8 + ht.numel() * 4 + (hf.numel() if hf is not None else 0))
    e2e_ms = maxr(statistics.median(e2e))
    Ntot = nx * ny * nz
    sel = res.regions[(res.regions["mask"] & np.uint64(1)) != 0]
    ncell = int(np.prod(sel["extent"].astype(np.int64) - 1, axis=1).sum())
    peak, peak_src = _peaks()
    kern_tab = {kk: {"launches": c, "avg_ms": t / c, "share": t / args.steps / ms}
                for kk, (c, t) in sorted(kern.items(), key=lambda kv: -kv[1][1])}
    dom = next(iter(kern_tab.items()), None)
    line = {
        "metric": METRIC, "value": 4 * Ntot / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded torch GRF; no public dataset)",
        "config": {"workload": f"{args.config} recipe on {nx}x{ny}x{nz} f32 in z-slabs over {world} GPUs "
                               f"({args.scaling} scaling); step = slab compress -> per-portion request(k) + "
                               "marching cubes (no payload bytes move between ranks)",
                   "dims": list(dims), "block_size": bs, "k": k, "regions": int(len(res.regions)),
                   "regions_selected": int(len(sel)), "archive_bytes": int(res.nbytes),
                   "triangles": m.ntri_total, "vertices": m.nvert_total, "parallelism": f"zslab{world}",
                   "l2": "no flush: per-rank input and outputs exceed the 126 MB L2"},
        "stages": {"compress_ms": t_c, "request_mc_ms": t_rm,
                   "compress_gbs": 4 * Ntot / (t_c * 1e-3) / 1e9, "cells": ncell},
        "kernels": kern_tab,
        "roofline": {"bound": "hbm", "kernel": dom[0] if dom else None, "achieved": None, "peak": peak,
                     "unit": "GB/s", "frac": None, "traffic": None, "peak_source": peak_src,
                     "note": "per-kernel roofline is reported by the N=1 run"},
        "cpu_baseline": None,
        "e2e": {"value": 4 * Ntot / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
