#!/usr/bin/env python
"""Benchmark: NU points/sec (exec, device-timed) for the BASELINE configs.

Default workload = BASELINE.json configs[3] ("C4"), the largest single-GPU
configuration (BASELINE's metric is not quoted on one config, so the
headline is the largest): 3D double precision, N = 256^3 (fine 512^3,
w = 13), M = 1e8 uniform points, eps = 1e-12.  A step = one type-1 execute
(spread -> cuFFT forward -> deconvolution) plus one type-2 execute (pad ->
cuFFT inverse -> interp) on the same points, both with the points already
set (the paper's "exec"); value = 2 M / step time.

  python bench.py [--gpus N --steps K --warmup W] [--config c4] [--method sm]
  python bench.py --impl reference ...   # the reference algorithm on host cores

Multi-GPU (torchrun, one process per GPU, NCCL).  --scaling strong (the C4
default) splits the config's M points across ranks (contiguous slices of
the input order); --scaling weak (the default for the other configs) gives
every rank its own M points.  Type-1 transforms spread each rank's points
into its own fine grid and sum the grids with an NCCL reduce before the
root's FFT + deconvolution; type-2 transforms broadcast the root's modes
and interpolate each rank's points on the replicated grid.  c5 runs
independent replicas (no collective).  Times are CUDA-event device times,
max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(type=1, modes=(256, 256), M=1_000_000, dist="rand", eps=1e-5, prec="single",
               desc="C1 2D type-1 f32 N=256^2 M=1e6 uniform eps=1e-5"),
    "c2": dict(type=2, modes=(1024, 1024), M=10_000_000, dist="rand", eps=1e-5, prec="single",
               desc="C2 2D type-2 f32 N=1024^2 M=1e7 uniform eps=1e-5"),
    "c3a": dict(type=1, modes=(128, 128, 128), M=10_000_000, dist="cluster", eps=1e-6,
                prec="single", desc="C3a 3D type-1 f32 N=128^3 M=1e7 box-cluster eps=1e-6"),
    "c3b": dict(type=1, modes=(128, 128, 128), M=10_000_000, dist="gauss", eps=1e-6,
                prec="single",
                desc="C3b 3D type-1 f32 N=128^3 M=1e7 Gaussian(0,(pi/8)^2) eps=1e-6"),
    "c3t2": dict(type=2, modes=(128, 128, 128), M=10_000_000, dist="gauss", eps=1e-6,
                 prec="single",
                 desc="C3t2 3D type-2 f32 N=128^3 M=1e7 Gaussian(0,(pi/8)^2) eps=1e-6 "
                      "(north_star 3D single type-2 target)"),
    "c3t2u": dict(type=2, modes=(128, 128, 128), M=10_000_000, dist="rand", eps=1e-5,
                  prec="single",
                  desc="C3t2u 3D type-2 f32 N=128^3 M=1e7 uniform eps=1e-5 "
                       "(north_star 3D single type-2 target)"),
    "c3t1u": dict(type=1, modes=(128, 128, 128), M=10_000_000, dist="rand", eps=1e-5,
                  prec="single",
                  desc="C3t1u 3D type-1 f32 N=128^3 M=1e7 uniform eps=1e-5 "
                       "(north_star 3D single type-1 target)"),
    "c5t1": dict(type=1, modes=(128, 128, 128), M=10_000_000, dist="rand", eps=1e-12,
                 prec="double", desc="C5t1 3D type-1 f64 N=128^3 M=1e7 uniform eps=1e-12 "
                                     "(the type-1 half of C5)"),
    "c5t2": dict(type=2, modes=(128, 128, 128), M=10_000_000, dist="rand", eps=1e-12,
                 prec="double", desc="C5t2 3D type-2 f64 N=128^3 M=1e7 uniform eps=1e-12 "
                                     "(the type-2 half of C5)"),
    "c4t1": dict(type=1, modes=(256, 256, 256), M=100_000_000, dist="rand", eps=1e-12,
                 prec="double", desc="C4 3D type-1 f64 N=256^3 M=1e8 uniform eps=1e-12"),
    "c4t2": dict(type=2, modes=(256, 256, 256), M=100_000_000, dist="rand", eps=1e-12,
                 prec="double", desc="C4 3D type-2 f64 N=256^3 M=1e8 uniform eps=1e-12"),
    "c4": dict(type=21, modes=(256, 256, 256), M=100_000_000, dist="rand", eps=1e-12,
               prec="double", scaling="strong", cpu_sample=300_000,
               desc="C4 3D type-1 + type-2 f64 N=256^3 M=1e8 uniform eps=1e-12"),
    "c5": dict(type=12, modes=(128, 128, 128), M=10_000_000, dist="rand", eps=1e-12,
               prec="double", cpu_sample=300_000,
               desc="C5 3D type-2 then type-1 f64 N=128^3 M=1e7 per rank, eps=1e-12"),
}
for _k in ("c4t1", "c4t2"):
    CONFIGS[_k]["scaling"] = "strong"
    CONFIGS[_k]["cpu_sample"] = 300_000
for _k in ("c5t1", "c5t2"):
    CONFIGS[_k]["cpu_sample"] = 300_000


def config_types(cfg):
    """Transforms per step, in execution order (c5: type 2 then type 1,
    the M-TIP slicing/merging pair; c4: type 1 then type 2)."""
    return {12: [2, 1], 21: [1, 2]}.get(cfg["type"], [cfg["type"]])
METRIC = "NU points/sec (exec, device-timed) at tol eps, 2D/3D type 1/2, at 1/2/4/8 B200"
L2_FLUSH_BYTES = 256 << 20


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def algorithmic_bytes(cfg, fine, M=None):
    """SURVEY.md §8(d) per-kernel bytes of the dominant kernel
    (spread for type 1, interp for type 2): M (d+2) s + 2 n_tot s."""
    d = len(cfg["modes"])
    s = 4 if cfg["prec"] == "single" else 8
    M = cfg["M"] if M is None else M
    return M * (d + 2) * s + 2 * int(np.prod(fine)) * s


def fp64_peak():
    """Measured FP64 FMA throughput (TFLOP/s) from profiles/fp64_peak.json
    (scripts/fp64_peak.cu on a B200 of this pool), else the architectural
    148 SMs x 64 DFMA/clk x 2 flops x 1.965 GHz."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
            j = json.load(fh)
        return float(j["fp64_fma_tflops"]), "measured (profiles/fp64_peak.json, scripts/fp64_peak.cu)"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "architectural: 148 SMs x 64 DFMA/clk x 2 x 1965 MHz"


def dmma_peak():
    """Measured FP64 tensor-core (DMMA m8n8k4) throughput in TFLOP/s, the
    best of profiles/r2/dmma_peak.json (scripts/dmma_peak.cu), else the
    FP64 FMA peak (B200 runs both at the same rate)."""
    try:
        best = 0.0
        with open(os.path.join(ROOT, "profiles", "r2", "dmma_peak.json")) as fh:
            for ln in fh:
                j = json.loads(ln)
                best = max(best, float(j.get("dmma_tflops", 0.0)))
        if best > 0:
            return best, "measured (profiles/r2/dmma_peak.json, scripts/dmma_peak.cu)"
    except Exception:
        pass
    return fp64_peak()


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x.strip() for x in cvd.split(",") if x.strip()]
        self.index = ids[index] if index < len(ids) and ids[index].isdigit() else index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
                 "utilization.gpu", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, util = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                util.append(float(parts[8]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        busy = [s for s, u in zip(sm, util) if u > 0] or sm
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(cfg, seed, rank=0):
    from oracle import oracle as orc   # generators only (seeded synthetic data)
    grid = orc.make_grid(cfg["modes"], cfg["eps"], cfg["prec"])
    rdt = np.float32 if cfg["prec"] == "single" else np.float64
    cdt = np.complex64 if cfg["prec"] == "single" else np.complex128
    pts = orc.gen_points(cfg["dist"], cfg["M"], grid, seed + rank, rdt)
    rng = np.random.default_rng(seed + 17)
    nmodes = int(np.prod(cfg["modes"]))
    f = (rng.uniform(0, 1, nmodes) + 1j * rng.uniform(0, 1, nmodes)).astype(cdt)
    c = (rng.uniform(0, 1, cfg["M"]) + 1j * rng.uniform(0, 1, cfg["M"])).astype(cdt)
    return grid, pts, f.reshape(cfg["modes"][::-1]), c


# ---------------------------------------------------------------- reference

def cpu_reference(cfg, steps, warmup, sample_cap):
    """The reference algorithm (oracle C port of nufftkit, all host threads)
    on a bounded sample: fixed-size stages (pad/deconv, FFT) at full size,
    the M-proportional stage (interp / spread) on `sample` points and scaled
    linearly to M.  Returns (pts_per_sec, cores, sample description)."""
    from oracle import oracle as orc
    # every host core the process may use (torchrun exports OMP_NUM_THREADS=1,
    # which omp_get_max_threads would report); the oracle takes the count
    # explicitly
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:
        threads = os.cpu_count() or orc.host_threads()
    sub = dict(cfg)
    if sample_cap is None:
        sample_cap = cfg.get("cpu_sample", cfg["M"])
    sample = min(cfg["M"], sample_cap)
    sub["M"] = sample
    grid, pts, f, c = make_inputs(sub, 0)
    box = None
    if sample < cfg["M"] and cfg["dist"] == "rand":
        # keep the full-M point density: the sample fills a sub-box of the
        # domain (side (sample / M)^(1/d) of 2 pi) instead of thinning the
        # whole grid, so the SM spread's per-bin setup / merge is amortised
        # over as many points per bin as at full size
        box = (sample / cfg["M"]) ** (1.0 / len(cfg["modes"]))
        pts = (-np.pi + (pts + np.pi) * box).astype(pts.dtype)
    types = config_types(cfg)
    plans = {}
    for t in types:
        p = orc.OraclePlan(t, cfg["modes"], cfg["eps"], "sm" if t == 1 else "gmsort",
                           cfg["prec"], workers=threads)
        p.set_points(pts)
        plans[t] = p
    times = []
    for it in range(warmup + steps):
        tot = 0.0
        for t in types:
            p = plans[t]
            g, prm = p.grid, p.params
            if t == 2:
                t0 = time.perf_counter()
                bh = orc.deconvolve_type2(f, g, prm, p.corr)
                b = orc.fft_fine(bh, "inverse", threads).astype(prm.complex_dtype, copy=False)
                t1 = time.perf_counter()
                orc.interpolate(p.points, b, prm, g, p.layout, threads)
                t2 = time.perf_counter()
                fixed, prop = t1 - t0, t2 - t1
            else:
                t0 = time.perf_counter()
                b = p.spread(c)
                t1 = time.perf_counter()
                bh = orc.fft_fine(b, "forward", threads).astype(prm.complex_dtype, copy=False)
                orc.deconvolve_type1(bh, g, prm, p.corr)
                t2 = time.perf_counter()
                fixed, prop = t2 - t1, t1 - t0
            tot += fixed + prop * (cfg["M"] / sample)
        if it >= warmup:
            times.append(tot)
    t_step = float(np.median(times))
    npts = cfg["M"] * len(types)
    what = " + ".join({2: "GM-sort interp", 1: "SM spread"}[t] for t in types)
    if sample == cfg["M"]:
        size = f"every stage at full size (M = {cfg['M']})"
    else:
        size = (f"SUBSAMPLED: the M-proportional stage timed on {sample} of {cfg['M']} "
                f"points and scaled linearly"
                + (f" (the sample fills a {box:.3f}^{len(cfg['modes'])} fraction of the "
                   f"domain at the full-M density)" if box else "")
                + "; pad/FFT/deconv at full size")
    desc = (f"oracle C port (nufftkit algorithm: {what}, scipy.fft) on {threads} host "
            f"threads; {size}; median of {steps}")
    return npts / t_step, threads, desc, t_step


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    v, cores, desc, t_step = cpu_reference(cfg, args.steps, args.warmup, args.cpu_sample)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "NU pts/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": cfg.get("scaling", "weak"),
            "vs_baseline": None, "dtype": "f32" if cfg["prec"] == "single" else "f64",
            "data": "synthetic (seeded numpy: uniform / cluster / gauss points, U[0,1)^2 "
                    "complex strengths)",
            "config": {"workload": cfg["desc"]},
            "cpu_baseline": {"value": v, "unit": "NU pts/s", "cores": cores, "kind": "port",
                             "sample": desc},
            "e2e": {"value": v, "unit": "NU pts/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- ours

def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test knobs for exercising the N > 1 path on a one-GPU box: every rank
    # on cuda:0 over gloo (type-1 grids then all-reduced: gloo has no CUDA
    # reduce).  Production runs use NCCL, one GPU per rank.
    backend = os.environ.get("NK_DIST_BACKEND", "nccl")
    if os.environ.get("NK_BENCH_SAME_DEVICE"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    import paper_2102_08463_b200 as nk
    from paper_2102_08463_b200.dist import CudaStageOps, ReplicaPlan, ShardedPlan, shard_bounds

    types = config_types(cfg)
    scaling = args.scaling or cfg.get("scaling", "weak")
    replicas = cfg["type"] == 12               # C5: independent M-TIP replicas
    sharded = world > 1 and not replicas
    if scaling == "strong" and world > 1:
        # the config's M points split across ranks: same inputs as N = 1
        grid, pts, f_host, c_host = make_inputs(cfg, args.seed, 0)
        lo, hi = shard_bounds(cfg["M"], world, rank)
        pts = np.ascontiguousarray(pts[lo:hi])
        c_host = np.ascontiguousarray(c_host[lo:hi])
        total_pts = cfg["M"]
    else:
        grid, pts, f_host, c_host = make_inputs(cfg, args.seed, rank)
        total_pts = world * cfg["M"]
    M = pts.shape[0]
    plans = {}
    pts_dev = torch.from_numpy(pts).to(dev)
    setpts_ms = {}
    for t in types:
        method = args.method or "default"
        kw = {"max_subproblem": args.msub} if args.msub else {}
        if args.bins:
            kw["bin_dims"] = tuple(int(v) for v in args.bins.split(","))
        plans[t] = nk.make_plan(t, cfg["modes"], cfg["eps"], method, cfg["prec"], **kw)
        plans[t].set_points(pts_dev)          # first call allocates
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        plans[t].set_points(pts_dev)          # setpts on resident coordinates
        e1.record()
        torch.cuda.synchronize()
        setpts_ms[f"type{t}"] = e0.elapsed_time(e1)
    torch.cuda.synchronize()
    f_dev = torch.from_numpy(f_host).to(dev)
    c_dev = torch.from_numpy(c_host).to(dev)
    out_dev = {2: torch.empty(M, dtype=c_dev.dtype, device=dev),
               1: torch.empty(cfg["modes"][::-1], dtype=c_dev.dtype, device=dev)}
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    runners = {}
    for t in types:
        runners[t] = (ShardedPlan(CudaStageOps(plans[t]), t, root=0) if sharded
                      else ReplicaPlan(plans[t]))
    spread_ev = []

    def step():
        """One exec per transform in the config; returns this library's
        kernel launches.  Sharded type 1: spread -> NCCL reduce -> root FFT +
        deconv; sharded type 2: NCCL broadcast of the modes -> this rank's
        execute (pad + FFT + interp)."""
        launches = 0
        for t in types:
            r = runners[t]
            if isinstance(r, ReplicaPlan):
                r.execute(f_dev if t == 2 else c_dev, out_dev[t])
                launches += plans[t].last_launch_count()
            elif t == 1:
                ev_a = torch.cuda.Event(enable_timing=True)
                ev_b = torch.cuda.Event(enable_timing=True)
                ev_a.record()
                fine = r.ops.spread(c_dev)
                ev_b.record()
                spread_ev.append((ev_a, ev_b))
                if backend == "nccl":
                    dist.reduce(fine, dst=0)
                else:
                    dist.all_reduce(fine)
                launches += 1
                if rank == 0:
                    r.ops.fft_deconvolve(fine, out_dev[1])
                    launches += 1
            else:
                r.execute(f_dev, out_dev[2])
                launches += plans[t].last_launch_count()
        return launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = 0
    kern_ms = {t: [] for t in types}
    stage = {}
    with Clocks(local) as clk:
        # the timed region can be milliseconds long; keep the same load
        # running (untimed) until the sampler has readings on both sides
        t_pre = time.time()
        soak = 0.0 if os.environ.get("NK_BENCH_NO_CLOCKS") else 5.0

        def soak_while(cond):
            # rank 0 decides: with a collective inside step() every rank
            # must run the same number of soak steps
            while True:
                go = torch.tensor([1 if cond() else 0], device=dev, dtype=torch.int32)
                if world > 1:
                    dist.broadcast(go, src=0)
                if not int(go.item()):
                    return
                step()
                torch.cuda.synchronize()

        soak_while(lambda: len(clk.lines) < 3 and time.time() - t_pre < soak)
        n_pre = len(clk.lines)
        # K steps back to back, bracketed by barrier + synchronize; before
        # each step a 256 MiB write flushes L2 (asynchronous, same stream:
        # it also covers the host's enqueue of the next step, so the step
        # events see device time only)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        spread_ev.clear()
        evs = []
        for _ in range(args.steps):
            flush.fill_(1.0)                       # L2 flush between timed steps
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            launches += step()
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        step_ms = [a.elapsed_time(b) for a, b in evs]
        if sharded and 1 in types:
            kern_ms[1] = [a.elapsed_time(b) for a, b in spread_ev]
        spread_ev.clear()
        # per-kernel times for the rooflines: the same steps again with the
        # plans' per-stage CUDA events on (direct launches, no graph replay;
        # every rank runs the same steps, collectives included)
        timed = [t for t in types if not (sharded and t == 1)]
        for t in timed:
            plans[t].set_timing(True)
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            step()
            torch.cuda.synchronize()
            for t in timed:
                st = plans[t].stage_times()
                kern_ms[t].append(st["interp" if t == 2 else "spread"])
                stage[f"type{t}"] = st
        for t in timed:
            plans[t].set_timing(False)
        spread_ev.clear()
        t_post = time.time()
        soak_while(lambda: len(clk.lines) < n_pre + 3 and time.time() - t_post < soak)
    tot_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())

    # ---- e2e (headline): the public API with pinned host buffers, copies
    # inside the timing.  Unsharded: plan.execute(host in, host out) through
    # the C-ABI (H2D + exec + D2H, synchronous) for every transform of the
    # step.  Sharded: each rank copies its inputs H2D, runs the sharded step
    # (collectives included) and reads its result back D2H.
    pin_in, pin_out = {}, {}
    for t in types:
        src = f_host if t == 2 else c_host
        pin_in[t] = torch.empty(src.shape, dtype=c_dev.dtype, pin_memory=True)
        pin_in[t].numpy()[...] = src
        pin_out[t] = torch.empty(out_dev[t].shape, dtype=c_dev.dtype, pin_memory=True)

    def e2e_step():
        if not sharded:
            for t in types:
                plans[t].execute(pin_in[t].numpy(), pin_out[t].numpy())
            return
        for t in types:
            (f_dev if t == 2 else c_dev).copy_(pin_in[t], non_blocking=True)
        step()
        for t in types:
            if t == 2 or rank == 0:
                pin_out[t].copy_(out_dev[t], non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(max(1, args.warmup)):
        e2e_step()
    spread_ev.clear()
    e2e_s = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_step()
        e2e_s.append(time.perf_counter() - t0)
    spread_ev.clear()
    e2e_t = float(np.sum(e2e_s))
    if world > 1:
        t = torch.tensor([e2e_t], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    csz = c_dev.element_size()
    nmodes = int(np.prod(cfg["modes"]))
    h2d = sum((nmodes if t == 2 else M) * csz for t in types)
    d2h = sum((M if t == 2 else nmodes) * csz for t in types)
    e2e = {"value": total_pts * len(types) * args.steps / e2e_t, "unit": "NU pts/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "mode": "one synchronous execute(host in, host out) per transform per step "
                   "through the C-ABI (pinned host buffers; H2D + exec + D2H timed)"}

    # ---- streamed variant (unsharded): the same public execute() on device
    # buffers, every step's H2D input copy and D2H result copy on their own
    # streams so step i's D2H overlaps step i+1's H2D and compute (PCIe is
    # full duplex).  Reported beside the synchronous headline.
    if not sharded:
        dins = {t: [torch.empty(pin_in[t].shape, dtype=c_dev.dtype, device=dev)
                    for _ in range(2)] for t in types}
        douts = {t: [torch.empty(out_dev[t].shape, dtype=c_dev.dtype, device=dev)
                     for _ in range(2)] for t in types}
        pouts = {t: [torch.empty(out_dev[t].shape, dtype=c_dev.dtype, pin_memory=True)
                     for _ in range(2)] for t in types}
        s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("in", "cmp", "out")}

        def streamed(n):
            for i in range(n):
                b = i & 1
                with torch.cuda.stream(s_in):
                    if i >= 2:
                        s_in.wait_event(ev["cmp"][b])      # step i-2 done reading dins
                    for t in types:
                        dins[t][b].copy_(pin_in[t], non_blocking=True)
                    ev["in"][b].record(s_in)
                with torch.cuda.stream(s_cmp):
                    s_cmp.wait_event(ev["in"][b])
                    if i >= 2:
                        s_cmp.wait_event(ev["out"][b])     # D2H of step i-2 done with douts
                    for t in types:
                        plans[t].execute(dins[t][b], douts[t][b])
                    ev["cmp"][b].record(s_cmp)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev["cmp"][b])
                    for t in types:
                        pouts[t][b].copy_(douts[t][b], non_blocking=True)
                    ev["out"][b].record(s_out)
            torch.cuda.synchronize()

        streamed(max(2, args.warmup))
        t0 = time.perf_counter()
        streamed(args.steps)
        st_t = time.perf_counter() - t0
        # same inputs as the synchronous e2e: results agree up to the float
        # reduction order of the spread's atomics
        ok = True
        for t in types:
            a_res = pouts[t][(args.steps - 1) & 1].numpy().reshape(-1)
            b_res = pin_out[t].numpy().reshape(-1)
            ok &= float(np.linalg.norm(a_res - b_res)) <= 1e-5 * float(np.linalg.norm(b_res))
        e2e["streamed"] = {
            "value": M * len(types) * args.steps / st_t, "unit": "NU pts/s",
            "mode": "per-step H2D / execute / D2H on three streams, double-buffered "
                    "(copies of step i+1 overlap step i)",
            "matches_sync_result": bool(ok)}
        for t in types:
            dins[t] = douts[t] = pouts[t] = None

    # per-kernel averages (max over ranks)
    kern_avg = {}
    for t in types:
        v = float(np.mean(kern_ms[t])) if kern_ms[t] else 0.0
        if world > 1:
            x = torch.tensor([v], device=dev)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            v = float(x.item())
        if v > 0:
            kern_avg[t] = v

    if rank == 0:
        dom_type = max(kern_avg, key=kern_avg.get) if kern_avg else types[0]
        fine = plans[dom_type].grid.fine
        w = plans[dom_type].params.w
        peak, peak_src = peaks()
        par = ("1 GPU" if world == 1 else
               f"{world} independent replicas" if replicas else
               f"{world} GPUs, {scaling} scaling: points sharded, type-1 fine grids "
               "NCCL-reduced to rank 0 / type-2 modes NCCL-broadcast")
        line = {
            "metric": METRIC,
            "value": total_pts * len(types) * args.steps / (tot_ms / 1e3),
            "unit": "NU pts/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": scaling if world > 1 else cfg.get("scaling", "weak"),
            "vs_baseline": None, "dtype": "f32" if cfg["prec"] == "single" else "f64",
            "data": "synthetic (seeded numpy: uniform / cluster / gauss points, U[0,1)^2 "
                    "complex strengths), inputs resident in HBM",
            "config": {"workload": cfg["desc"] + (f", per rank x {world}"
                                                  if world > 1 and scaling == "weak" else ""),
                       "transforms_per_step": [f"type{t}" for t in types],
                       "method": plans[dom_type].method,
                       "fine": list(fine), "w": w,
                       "bin_dims": {f"type{t}": list(plans[t].bin_dims) for t in types},
                       "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": par},
            "gpu_launches": launches,
            "setpts_ms": setpts_ms,
        }
        # setpts against its SURVEY §8(d) bytes: coords read + 3 M int32
        # (key write / re-read / perm write) + permuted coords written
        d = len(cfg["modes"])
        s = 4 if cfg["prec"] == "single" else 8
        sp_bytes = M * d * s * 2 + 3 * M * 4
        sp_ms = setpts_ms[f"type{types[0]}"]
        line["setpts_roofline"] = {"bound": "hbm", "algorithmic_bytes": sp_bytes,
                                   "achieved": sp_bytes / (sp_ms / 1e3) / 1e9, "peak": peak,
                                   "unit": "GB/s",
                                   "frac": sp_bytes / (sp_ms / 1e3) / 1e9 / peak}
        if kern_avg:
            dom_ms = kern_avg[dom_type]
            B = algorithmic_bytes(cfg, fine, M)
            ach = B / (dom_ms / 1e3) / 1e9
            line["roofline"] = {"bound": "hbm",
                                "kernel": "interp" if dom_type == 2 else "spread",
                                "achieved": ach, "peak": peak, "unit": "GB/s",
                                "frac": ach / peak, "traffic": traffic_for(args.config),
                                "algorithmic_bytes": B, "kernel_ms": dom_ms,
                                "kernel_ms_by_type": {f"type{t}": v for t, v in kern_avg.items()},
                                "peak_source": peak_src}
            if cfg["prec"] == "double" and d == 3 and w >= 9 and \
                    plans[dom_type].method == "sm":
                # the tiled f64 spread / interp (K6t / K7t) run on the FP64
                # tensor cores: algorithmic flops = 4 w^3 per point (w^3
                # complex x real FMAs) over the measured DMMA peak; the
                # issued DMMA flops cover the 16^3 tile window (4 * 16^3)
                tpk, tpk_src = dmma_peak()
                flops = 4.0 * M * w ** d
                ach_t = flops / (dom_ms / 1e3) / 1e12
                hbm = line["roofline"]
                line["roofline"] = {"bound": "tensor",
                                    "kernel": hbm["kernel"] + " (DMMA m8n8k4)",
                                    "achieved": ach_t, "peak": tpk, "unit": "TFLOP/s",
                                    "frac": ach_t / tpk, "traffic": hbm["traffic"],
                                    "algorithmic_flops": flops,
                                    "issued_flops": 4.0 * M * 16 ** 3,
                                    "kernel_ms": dom_ms,
                                    "kernel_ms_by_type": hbm["kernel_ms_by_type"],
                                    "peak_source": tpk_src}
                line["hbm_roofline"] = {k: hbm[k] for k in ("bound", "achieved", "peak", "unit",
                                                            "frac", "algorithmic_bytes",
                                                            "peak_source")}
            if cfg["prec"] == "double":
                # the f64 spread / interp are FP64-pipe bound: w^d cell updates
                # per point, each a complex x real FMA (2 DFMA = 4 flops)
                fpk, fpk_src = fp64_peak()
                flops = 4.0 * M * w ** d
                line["fp64_roofline"] = {
                    "bound": "fp64", "flops_per_point": 4 * w ** d, "peak": fpk,
                    "unit": "TFLOP/s", "peak_source": fpk_src,
                    "by_kernel": {("interp" if t == 2 else "spread"): {
                        "achieved": flops / (v / 1e3) / 1e12,
                        "frac": flops / (v / 1e3) / 1e12 / fpk, "kernel_ms": v}
                        for t, v in kern_avg.items()}}
            # The SM kernels are bound by the shared-memory pipe, not HBM
            # (DESIGN.md §5): the same launch against the shared-memory
            # roofline.  Bytes = the footprint cells each point touches in
            # the padded bin (w^d complex values; read for interp, read +
            # write for the spread's cell updates), peak = 128 B/clk/SM x
            # 148 SMs at the max SM clock (architectural, not measured).
            cells = M * w ** d
            sb = cells * 2 * s * (1 if dom_type == 2 else 2)
            sh_peak = 148 * 128 * 1965e6 / 1e9
            line["shared_roofline"] = {
                "bound": "shared", "achieved": sb / (dom_ms / 1e3) / 1e9, "peak": sh_peak,
                "unit": "GB/s", "frac": sb / (dom_ms / 1e3) / 1e9 / sh_peak,
                "bytes": sb, "peak_source": "architectural: 128 B/clk/SM x 148 SMs x 1965 MHz"}
            if dom_type == 1:
                line["shared_roofline"]["note"] = (
                    "bytes = the reference SM scheme's per-point cell read-modify-writes; "
                    "register accumulation skips most of them, so frac can exceed 1")
            if stage:
                line["stage_ms"] = stage
        line["e2e"] = e2e
        line["clocks"] = clk.summary()
        if world == 1 and not args.no_cpu_baseline:
            v, cores, desc, _ = cpu_reference(cfg, 2, 1, args.cpu_sample)
            line["cpu_baseline"] = {"value": v, "unit": "NU pts/s", "cores": cores,
                                    "kind": "port", "sample": desc}
        print(json.dumps(line), flush=True)
    for p in plans.values():
        p.destroy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def traffic_for(config):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(config)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--scaling", choices=["strong", "weak"], default=None,
                    help="multi-GPU: split the config's M across ranks (strong) or give "
                         "every rank its own M (weak); default per config (c4 strong)")
    ap.add_argument("--method", default=None)
    ap.add_argument("--msub", type=int, default=None, help="max subproblem size override")
    ap.add_argument("--bins", default=None, help="bin dims override, e.g. 16,16")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="points of the CPU baseline's M-proportional stage (default: the "
                         "full M for c1-c3, a flagged subsample for c4 / c5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
