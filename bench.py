#!/usr/bin/env python
"""Benchmark of the direct-method hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--engine auto|simt|tensor]
    python bench.py --impl reference ...       # the FP64 CPU oracle on a bounded sample (the reference arm)

A "step" = one pass of the whole hot path over one batch of synthetic input: frame staging, I(q,t) for every
pixel of every frame, g2 for all lags, ring-averaged S(q,t) and g2, XSVS contrast for every exposure window.
Default workload = BASELINE.json configs[2] ("c3": N = 262144 atoms of two species, 1000 Brownian frames, 512 x 512
lattice plane, g2 tau = 1..200), the largest configuration that fits one GPU (BASELINE.json quotes its metric on no
config; c3 is 6.9e13 pairs per step, c2 2.1e11).  Metric: atom.q pairs/s for I(q,t) (whole job, all ranks).
Multi-GPU (torchrun, N > 1): ONE trajectory with the detector split across the ranks and the ring / XSVS moments
all-reduced once per step (SURVEY 8(e), strong scaling); --replicas runs independent trajectories instead (weak
scaling, no data-path collective).
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

import xpcs_inputs as xi  # noqa: E402

METRIC = "atom·q pairs/s for I(q,t) at 1 B200; fraction of FP32/SFU or tensor roofline"
UNIT = "pairs/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 10 ms through NVML during the timed region
    (the B200_PROFILING.md clocks line; nvidia-smi's 100 ms period is too coarse for a ~100 ms region)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index=0, period=0.01):
        self.index, self.period = index, period
        self.sm, self.mx, self.reasons = [], None, set()
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join(timeout=1)

    def summary(self):
        if not self.ok or not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml, 10 ms"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist
        rank = int(os.environ["RANK"])
        local = int(os.environ.get("LOCAL_RANK", rank))
        return ws, rank, local, dist
    return 1, 0, 0, None


def _traffic(workload, engine, pairs_launch):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/traffic.json, written from the capture summary), scaled to this launch's pairs; None if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
        rec = t[workload][engine]
        return rec["dram_bytes"] * pairs_launch / rec["pairs"]
    except (OSError, KeyError, ValueError, ZeroDivisionError):
        return None


def _roofline(cfg, wl, engine, f_h, prof, pairs_step, steps, step_ms, peaks, peak_src, sm_count, clk, xp):
    """Roofline of the dominant kernel of the step.

    achieved = the method's ALGORITHMIC work per launch / that kernel's average launch time (CUDA events on its
    stream, the library's per-class profiling over the timed graph replays).  Algorithmic work: on a
    lattice plane one complex MAC = 8 ops per atom.q pair, whatever the engine issues; for generic q one complex
    exponential = 2 XU (MUFU) ops per pair.  peak = MEASURED_PEAKS for the kernel's own dtype: fp16 = the measured
    bf16 dense rate, int8 = 2 x that (the guide's nominal int8/fp16 ratio; tools/mma_rate.cu measured 8192 vs 4096
    MAC/clk/SM); the burst figure for a short step, the sustained one for a step >= 50 ms (a kernel inside a long,
    power-capped step).  "pipe" reports what the tensor pipe actually issues (12 ops per pair: 3 split-precision
    products x 2 real MACs per pixel of a conjugate pair) against the same peak and against the tcgen05 issue rate
    at the run's SM clock."""
    mhz_max = peaks.get("sm_max_mhz", 1965.0)
    mhz_run = clk.get("sm_mhz") or mhz_max
    long_step = step_ms >= 50.0
    bf16 = peaks["bf16_tflops_sustained"] if long_step else peaks["bf16_tflops"]
    which = "sustained" if long_step else "burst"
    ms_i8, n_i8 = prof.get("intensity_i8", (0.0, 0))
    ms_tc, n_tc = prof.get("intensity_tc", (0.0, 0))
    ms_main, n_main = prof["intensity_main"]
    share_i8 = None
    if ms_i8 > 0 and ms_tc > 0:
        counts = np.bincount(wl.kinds, minlength=len(wl.kind_f))
        share_i8 = float(sum(xp.species_engines(counts, wl.kind_f))) / float(counts.sum())
    elif ms_i8 > 0:
        share_i8 = 1.0
    elif ms_tc > 0:
        share_i8 = 0.0
    engines = {}
    spec = {"i8": ("k_lattice_i8", ms_i8, n_i8, "int8 (two Q16 limbs) -> exact int32", 2.0 * bf16, "TOPS (int8)", 8190.0,
                   f"{peak_src} {which} bf16 x 2 (int8)"),
            "tensor": ("k_lattice_tc", ms_tc, n_tc, "fp16 (hi/lo split) -> fp32", bf16, "TFLOP/s (fp16)", 4095.0,
                       f"{peak_src} {which} bf16 (= fp16 rate)")}
    for name, (kern, ms_e, n_e, dt, peak, unit, rate, src) in spec.items():
        if ms_e <= 0:
            continue
        pairs = pairs_step * (share_i8 if name == "i8" else 1.0 - share_i8)
        t = ms_e / steps / 1e3                              # seconds per step in this engine
        ach = 8.0 * pairs / t / 1e12
        issued = 12.0 * pairs / t / 1e12
        issue_peak = sm_count * rate * 2 * mhz_run * 1e6 / 1e12
        engines[name] = {"kernel": kern, "dtype": dt, "bound": "tensor", "unit": unit, "peak": peak, "peak_source": src,
                         "achieved": ach, "frac": ach / peak, "ops_per_pair": 8,
                         "pairs_per_step": pairs, "kernel_ms_per_step": ms_e / steps, "launches_per_step": n_e / steps,
                         "pairs_per_launch": pairs / max(n_e / steps, 1e-9),
                         "pipe": {"issued_ops_per_pair": 12, "achieved": issued, "frac_of_peak": issued / peak,
                                  "vs_issue_rate": issued / issue_peak, "issue_rate_peak": issue_peak,
                                  "clock_mhz": mhz_run, "source": "tools/mma_rate.cu"}}
    if engines:
        dom = max(engines, key=lambda k: engines[k]["kernel_ms_per_step"])
        roof = dict(engines[dom])
        roof["engine"] = dom
        if len(engines) > 1:
            roof["engines"] = engines
            roof["int8_pair_share"] = share_i8
        eng_name = "i8+tensor" if len(engines) > 1 else dom
        dtype = " + ".join(f"{e['dtype']} ({e['kernel']}{'' if len(engines) == 1 else f', {100 * e['pairs_per_step'] / pairs_step:.1f}% of pairs'})"
                           for e in engines.values()) + "; positions f32, I f32"
        return roof, eng_name, dtype
    t = ms_main / steps / 1e3
    launches = max(n_main / steps, 1e-9)
    if cfg.n_plane == 0:
        # generic q: 2 XU (MUFU) ops per pair; ceiling = 148 SM x 16 XU/clk x max clock / 2
        peak = sm_count * 16 * mhz_max * 1e6 / 2 / 1e12
        roof = {"kernel": "k_generic32", "bound": "alu", "unit": "Tpairs/s (XU: 2 MUFU per pair)", "peak": peak,
                "achieved": pairs_step / t / 1e12, "peak_source": "derived (DESIGN.md)"}
        eng_name, dtype = "generic", "f32 (exact integer phase turns, SFU sincos, FP64 chunk folds)"
    else:
        peak = sm_count * 128 * 2 * mhz_max * 1e6 / 1e12
        roof = {"kernel": "k_lattice_simt" if wl.in_dtype != xp.F64 else "k_lattice64", "bound": "alu",
                "unit": "TFLOP/s (FP32 FMA pipe)", "peak": peak, "achieved": 8.0 * pairs_step / t / 1e12,
                "peak_source": "derived (DESIGN.md)"}
        eng_name = "fp64" if wl.in_dtype == xp.F64 else "simt"
        dtype = "f64" if wl.in_dtype == xp.F64 else "f32"
        if wl.in_dtype == xp.F64:
            roof["note"] = "FP64 workload: latency-bound (SURVEY 8(d)), report ms_per_step; frac is context only"
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel_ms_per_step"] = ms_main / steps
    roof["launches_per_step"] = n_main / steps
    roof["pairs_per_launch"] = pairs_step / launches
    return roof, eng_name, dtype


def run_reference(args):
    """The reference arm: the FP64 CPU oracle (as it stands) on a bounded sample of the same workload."""
    ws, rank, _, dist = _dist()
    if rank != 0:
        return 0
    # the oracle runs on all the host's cores (torchrun exports OMP_NUM_THREADS=1 per rank, and torch.distributed
    # has already initialised the OpenMP runtime with it)
    import oracle
    oracle.set_threads(len(os.sched_getaffinity(0)))
    cfg = xi.CONFIGS[args.config]
    pos = xi.positions(cfg, frames=1)[0]
    f = xi.form_factors(cfg).astype(np.float64) if cfg.two_species else None
    if cfg.n_plane:
        q = oracle.lattice_q(cfg.L, **oracle.plane_grid(cfg.n_plane))
    else:
        q = oracle.ewald_q(xi.EWALD_WAVELENGTH_SIGMA, cfg.detector, cfg.detector, xi.EWALD_PITCH_RAD).astype(np.float32)
    n_pix = min(q.shape[0], args.ref_pixels)
    pix = xi.pixel_subset(q.shape[0], n_pix, 1234)
    qs = q[pix].astype(np.float64)
    oracle.intensity(pos, f, qs[:64], cfg.L)            # load + warm
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.intensity(pos, f, qs, cfg.L)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    pairs = cfg.N * n_pix
    ms = 1e3 * float(np.mean(times))
    val = pairs / (ms / 1e3)
    sample = f"{args.config} frame 0, {n_pix} seeded pixels x {cfg.N} atoms = {pairs:.3g} pairs per step"
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "N": cfg.N, "n_q": int(q.shape[0]), "frames": cfg.T},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.threads(), "cpu_model": _cpu_model(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(cfg, budget_s):
    """Oracle timed on the host cores on a bounded sample (rank 0, N = 1 only)."""
    import oracle
    oracle.set_threads(len(os.sched_getaffinity(0)))
    pos = xi.positions(cfg, frames=1)[0]
    f = xi.form_factors(cfg).astype(np.float64) if cfg.two_species else None
    if cfg.n_plane:
        q = oracle.lattice_q(cfg.L, **oracle.plane_grid(cfg.n_plane))
    else:
        q = oracle.ewald_q(xi.EWALD_WAVELENGTH_SIGMA, cfg.detector, cfg.detector, xi.EWALD_PITCH_RAD).astype(np.float32)
    qs = q.astype(np.float64)
    # calibrate on 256 pixels, then size the sample to ~budget_s
    t0 = time.perf_counter()
    oracle.intensity(pos, f, qs[:256], cfg.L)
    per_pix = (time.perf_counter() - t0) / 256
    n_pix = int(max(256, min(q.shape[0], budget_s / max(per_pix, 1e-9))))
    pix = xi.pixel_subset(q.shape[0], n_pix, 99)
    t0 = time.perf_counter()
    oracle.intensity(pos, f, qs[pix], cfg.L)
    dt = time.perf_counter() - t0
    pairs = cfg.N * len(pix)
    return {"value": pairs / dt, "unit": UNIT, "cores": oracle.threads(), "cpu_model": _cpu_model(), "kind": "oracle",
            "sample": f"{cfg.name} frame 0, {len(pix)} seeded pixels x {cfg.N} atoms ({pairs:.3g} pairs, {dt:.1f} s)"}


def run_qshard(args, cfg, ws, rank, dev, dist):
    """N > 1 (default): ONE trajectory, the detector split across the ranks (pipeline.QShardPipeline: tile-aligned 2-D
    q-blocks of a lattice plane, pixel ranges of an explicit q list); every rank computes I and g2 of its
    block and the ring / XSVS moments, one NCCL all-reduce of the moments per step (the path's only exchange), ring
    results from the sums.  Strong scaling: value = the whole detector's pairs / the max-over-ranks step time.
    e2e: per rank, the pinned positions copied in, the step, and the block's I plus the ring results copied out."""
    import torch
    import paper_2204_13241_b200 as xp
    from paper_2204_13241_b200 import pipeline
    from paper_2204_13241_b200 import dist as xd
    wl = pipeline.workload_from_config(cfg, device=dev)
    wl.engine = {"auto": xp.ENGINE_AUTO, "simt": xp.ENGINE_SIMT, "tensor": xp.ENGINE_TENSOR,
                 "i8": xp.ENGINE_TENSOR_I8}[args.engine]
    Q = pipeline.QShardPipeline(wl, rank, ws, device=dev)
    pos_h = xi.positions(cfg)
    f_h = xi.form_factors(cfg) if cfg.two_species else None
    pos_d = torch.from_numpy(pos_h).to(dev)
    f_d = torch.from_numpy(f_h).to(dev) if f_h is not None else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        Q.run(pos_d, f_d)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    t_ms = []
    xp.profile_reset()
    n0 = xp.launch_count()
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            flush.zero_()
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            Q.run(pos_d, f_d, profile=True)
            b.record(stream)
            torch.cuda.synchronize()
            t_ms.append(a.elapsed_time(b))
    n_launch = xp.launch_count() - n0
    prof = xp.profile_query()
    ms = xd.max_over_ranks(float(np.mean(t_ms)), dev)
    peaks, peak_src = _peaks()
    sm_count, _ = xp.device_info()
    roof, eng_name, dtype = _roofline(cfg, wl, wl.engine, f_h, prof, Q.pairs_per_step, args.steps, float(np.mean(t_ms)),
                                      peaks, peak_src, sm_count, clk.summary(), xp)
    roof["note"] = "rank 0's block: its own pairs and kernel time"
    pairs = int(cfg.N) * int(Q.wl.q.shape[0] if cfg.n_plane == 0 else cfg.n_plane ** 2) * int(cfg.T)
    # end to end: pinned positions in, the step, this rank's I block and the ring results out, every step
    e2e = None
    if not args.no_e2e:
        h_pos = torch.from_numpy(pos_h).pin_memory()
        h_f = torch.from_numpy(f_h).pin_memory() if f_h is not None else None
        h_I = torch.empty(Q.I.shape, dtype=Q.I.dtype).pin_memory()
        t_e = []
        for _ in range(max(2, args.steps)):
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            pos_d.copy_(h_pos, non_blocking=True)
            if h_f is not None:
                f_d.copy_(h_f, non_blocking=True)
            res = Q.run(pos_d, f_d)
            h_I.copy_(Q.I, non_blocking=True)
            small = {k: v.to("cpu", non_blocking=True) for k, v in res.items() if k in ("S_rings", "g2_rings", "beta")}
            b.record(stream)
            torch.cuda.synchronize()
            t_e.append(a.elapsed_time(b))
        e_ms = xd.max_over_ranks(float(np.mean(t_e)), dev)
        d2h = h_I.numel() * h_I.element_size() + sum(v.numel() * v.element_size() for v in small.values())
        e2e = {"value": pairs / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "mode": "per rank: pinned positions in, the q-shard step, its I block and the ring results out",
               "h2d_bytes_per_step": int(pos_h.nbytes + (f_h.nbytes if f_h is not None else 0)),
               "d2h_bytes_per_step": int(d2h)}
    if rank == 0:
        line = {"metric": METRIC, "value": pairs / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": dtype, "data": "synthetic", "mode": "qshard",
                "config": {"workload": cfg.name, "N": cfg.N, "frames": cfg.T,
                           "n_q": int(cfg.n_plane ** 2 if cfg.n_plane else Q.wl.q.shape[0]),
                           "parallelism": f"q-shard x{ws} (one trajectory; detector blocks per rank; ring / XSVS "
                                          f"moments all-reduced once per step)",
                           "block_rank0": list(Q.block), "allreduce_bytes": int(Q.mom.numel() * 8),
                           "l2": "flushed between timed steps (256 MB write, untimed)"},
                "roofline": roof, "e2e": e2e, "gpu_launches": int(n_launch), "clocks": clk.summary(),
                "step_ms_all": t_ms, "engine_used": eng_name,
                "kernel_ms_rank0": {k: v[0] / max(args.steps, 1) for k, v in prof.items()}}
        print(json.dumps(line), flush=True)
    Q.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _e2e_streamed(args, P, pipeline, wl, dev, pos_h, f_h, slots, stream, dist):
    import torch
    # streaming: `slots` pipelines (own device buffers, pinned host buffers and CUDA graph each) replayed
    # round-robin on their own streams, so step k+1's H2D and kernels overlap step k's result D2H; every
    # step still copies its inputs in and its results out.  Time = whole run / steps (CUDA events).
    pipes = [P] + [pipeline.Pipeline(wl, device=dev) for _ in range(slots - 1)]
    for Q in pipes[1:]:
        Q.alloc_host_io(pos_h, f_h, batches=args.e2e_batches)
        Q.run_host()
    graphs = [Q.capture_host()[0] for Q in pipes]
    streams = [torch.cuda.Stream() for _ in pipes]
    n_e = max(2 * slots, args.steps)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for st_ in streams:
        st_.wait_stream(stream)
    for k in range(n_e):
        with torch.cuda.stream(streams[k % slots]):
            graphs[k % slots].replay()
    for st_ in streams:
        stream.wait_stream(st_)
    b.record(stream)
    torch.cuda.synchronize()
    e_ms = a.elapsed_time(b) / n_e
    for Q in pipes[1:]:
        Q.close()
    return e_ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(xi.CONFIGS))
    ap.add_argument("--engine", default="auto", choices=["auto", "simt", "tensor", "i8"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--ref-pixels", type=int, default=4096)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-slots", type=int, default=0,
                    help="pipelines in flight for the end-to-end figure (0: 3 when a step's pinned inputs are < 512 MB, "
                         "else 2)")
    ap.add_argument("--e2e-batches", type=int, default=4, help="frame batches per step in the end-to-end figure")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of replaying its CUDA graph")
    ap.add_argument("--qslab", "--qshard", dest="qshard", action="store_true",
                    help="ONE trajectory, the detector split into blocks across the ranks, ring moments all-reduced "
                         "once per step (SURVEY 8(e)); the default when more than one process runs")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent trajectories per rank instead (weak scaling, no data-path collective)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2204_13241_b200 as xp
    from paper_2204_13241_b200 import pipeline

    ws, rank, local, dist = _dist()
    torch.cuda.set_device(local)
    if dist is not None:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg = xi.CONFIGS[args.config]
    if args.qshard or (ws > 1 and not args.replicas):
        return run_qshard(args, cfg, ws, rank, dev, dist)
    # weak scaling: each rank its own independent trajectory
    from paper_2204_13241_b200 import dist as xd
    cfg_r = xi.scaled(cfg, seed=xd.trajectory_seed(cfg.seed, rank)) if rank else cfg
    pos_h = xi.positions(cfg_r)
    f_h = xi.form_factors(cfg_r) if cfg.two_species else None
    engine = {"auto": xp.ENGINE_AUTO, "simt": xp.ENGINE_SIMT, "tensor": xp.ENGINE_TENSOR,
              "i8": xp.ENGINE_TENSOR_I8}[args.engine]
    wl = pipeline.workload_from_config(cfg, device=dev)
    wl.engine = engine
    P = pipeline.Pipeline(wl, device=dev)
    pos_d = torch.from_numpy(pos_h).to(dev)
    f_d = torch.from_numpy(f_h).to(dev) if f_h is not None else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)    # 256 MB > 126 MB L2

    for _ in range(args.warmup):
        P.run(pos_d, f_d)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    xp.profile_reset()
    graph = None
    launch_note = "eager" if args.no_graph else "cuda graph (one replay per step)"
    if not args.no_graph:
        # the step as one CUDA graph (kernels, side-stream fork/join, profiling events): no host launch gaps inside
        # the timed region; every replay recomputes everything from pos_d
        try:
            graph, _ = P.capture(pos_d, f_d, profile=True)
            launches_graph = P.capture_launches
            for _ in range(args.warmup):                    # the first replays upload the graph: untimed
                flush.zero_()
                graph.replay()
            torch.cuda.synchronize()
        except Exception as e:                              # capture failed: time the eager step instead
            graph = None
            launch_note = f"eager (graph capture failed: {type(e).__name__})"
            torch.cuda.synchronize()
            xp.profile_reset()
    n_launch0 = xp.launch_count()
    prof = {}
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()                                   # L2 flush between timed iterations (untimed)
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            ev[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                P.run(pos_d, f_d, profile=True)
            ev[i][1].record(stream)
            torch.cuda.synchronize()
            if graph is not None:
                for k, (t_ms, n_k) in xp.profile_query().items():   # this replay's kernel-class times
                    a0, n0 = prof.get(k, (0.0, 0))
                    prof[k] = (a0 + t_ms, n0 + n_k)
    if graph is not None:
        n_launch = launches_graph * args.steps
    else:
        n_launch = xp.launch_count() - n_launch0
        prof = xp.profile_query()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    ms = xd.max_over_ranks(ms, dev)
    pairs_step = P.pairs_per_step
    value = ws * pairs_step / (ms / 1e3)

    # ---- roofline of the dominant kernel, CUDA events on its stream (the library's per-class profiling)
    peaks, peak_src = _peaks()
    sm_count, _ = xp.device_info()
    clk_sum = clk.summary()
    roof, eng_name, dtype = _roofline(cfg, wl, engine, f_h, prof, pairs_step, args.steps, ms, peaks, peak_src, sm_count,
                                      clk_sum, xp)
    main_ms = prof["intensity_main"][0]
    roof["traffic"] = _traffic(cfg.name, roof.get("kernel", eng_name), roof.get("pairs_per_launch", 0.0))
    roof["kernel_share_of_step"] = (roof["kernel_ms_per_step"] / ms) if ms > 0 else None

    # ---- end to end through the public API from pinned host memory: every step copies its positions in and I, g2,
    # rings and beta out (xpcs_step_host, frame-batched H2D / compute / D2H overlap inside the step).  value = one
    # pipeline, steps back to back (synchronous); "pipelined" = 2-3 pipelines in flight, so that step k's copies
    # overlap step k+1's kernels (no L2 flush between steps)
    e2e = None
    if not args.no_e2e:
        P.alloc_host_io(pos_h, f_h, batches=args.e2e_batches)
        P.run_host()
        torch.cuda.synchronize()
        h2d, d2h = P.io_bytes()
        auto_slots = 3 if pos_h.nbytes < (512 << 20) else 2
        slots = args.e2e_slots if args.e2e_slots > 0 else auto_slots
        e_sync = e_pipe = None
        if not args.no_graph:
            try:
                e_sync = _e2e_streamed(args, P, pipeline, wl, dev, pos_h, f_h, 1, stream, dist)
                if slots > 1:
                    e_pipe = _e2e_streamed(args, P, pipeline, wl, dev, pos_h, f_h, slots, stream, dist)
            except Exception:                                  # capture failed: eager host steps instead
                torch.cuda.synchronize()
                e_sync = e_pipe = None
        if e_sync is None:
            t_e = []
            for _ in range(max(2, args.steps)):
                if dist is not None:
                    dist.barrier()
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                P.run_host()
                b.record(stream)
                torch.cuda.synchronize()
                t_e.append(a.elapsed_time(b))
            e_sync = float(np.mean(t_e))
        e_sync = xd.max_over_ranks(e_sync, dev)
        e2e = {"value": ws * pairs_step / (e_sync / 1e3), "unit": UNIT, "ms_per_step": e_sync, "streams": 1,
               "mode": "one pipeline, steps back to back", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}
        if e_pipe is not None:
            e_pipe = xd.max_over_ranks(e_pipe, dev)
            e2e["pipelined"] = {"value": ws * pairs_step / (e_pipe / 1e3), "ms_per_step": e_pipe, "streams": slots,
                                "mode": f"{slots} pipelines in flight (step k's copies overlap step k+1's kernels)"}

    # ---- secondary kernels against their own bounds (algorithmic work per step / measured class time per step).
    # In the timed step the reductions run concurrently, so their event times overlap; they are timed here in a few
    # extra eager steps with the reductions serialised on one stream (outside the timed region).
    n_iso = 5
    P.serial_reductions = True
    xp.profile_reset()
    for _ in range(n_iso):
        P.run(pos_d, f_d, profile=True)
    torch.cuda.synchronize()
    prof_iso = xp.profile_query()
    P.serial_reductions = False
    xp.profile_reset()
    mhz = peaks.get("sm_max_mhz", 1965.0)
    T, n_q, nl = cfg.T, P.n_q, len(cfg.lags)
    i_bytes = (8 if wl.in_dtype == xp.F64 else 4) * T * n_q
    secondary = {}

    def _sec(cls, bound, work, peak, unit):
        ms_c = prof_iso.get(cls, (0.0, 0))[0] / n_iso
        if ms_c > 0:
            ach = work / (ms_c / 1e3)
            secondary[cls] = {"ms": ms_c, "bound": bound, "achieved": ach / 1e9, "peak": peak / 1e9, "unit": unit,
                              "frac": ach / peak}

    hbm = peaks.get("hbm_gbs", 6550.0) * 1e9
    # g2: one FP64 FMA per (pixel, lag, frame pair); FP64 peak = 148 SMs x 59 DFMA/clk (tools/microbench.cu)
    if nl:
        _sec("g2", "fp64", float(sum(T - tau for tau in cfg.lags)) * n_q, sm_count * 58.95 * mhz * 1e6,
             "G DFMA/s")
    # XSVS: one read of the intensity series for all exposure windows (4 T bytes per pixel)
    if cfg.windows:
        _sec("xsvs", "hbm", float(i_bytes), hbm, "GB/s")
    # staging: positions read (12 B) + 16-B records written per atom and frame
    _sec("stage", "hbm", float(cfg.N) * T * (12 + 16), hbm, "GB/s")
    # (the fold of the atom-chunk partials reads C partial planes, C chosen inside the library: ncu shows it at
    # ~6 TB/s, profiles/r01_launches_c2_summary.txt; it is left out here rather than under-counted)
    # rings: one read of I (S rings) and of g2 (g2 rings)
    _sec("rings", "hbm", float(i_bytes + 4 * nl * n_q), hbm, "GB/s")

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_budget)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": {"workload": cfg.name, "N": cfg.N, "n_q": P.n_q, "frames": cfg.T,
                           "lags": len(cfg.lags), "windows": list(cfg.windows), "rings": cfg.n_bins,
                           "pairs_per_step_per_gpu": pairs_step, "engine": args.engine,
                           "engine_used": ("fp64" if wl.in_dtype == xp.F64 else eng_name),
                           "l2": "flushed between timed steps (256 MB write, untimed)",
                           "launch": launch_note,
                           "parallelism": f"weak x{ws} (independent trajectories)"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(n_launch),
                "clocks": clk.summary(), "step_ms_all": step_ms,
                "kernel_ms": {k: v[0] / max(args.steps, 1) for k, v in prof.items()},
                "secondary_rooflines": secondary,
                "secondary_note": f"reductions timed alone (serialised, {n_iso} eager steps after the timed region); "
                                  "kernel_ms are event intervals per kernel class from the timed graph replays, where "
                                  "classes run concurrently (consecutive frame batches on two streams: a batch's "
                                  "staging / reduction / fix-up interval includes time spent beside the neighbouring "
                                  "batch's tensor engine), so they overlap and do not add up to ms_per_step"}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
