#!/usr/bin/env python
"""Benchmark of the direct-method hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--engine auto|simt|tensor]
    python bench.py --impl reference ...       # the FP64 CPU oracle on a bounded sample (the reference arm)

A "step" = one pass of the whole hot path over one batch of synthetic input: frame staging, I(q,t) for every
pixel of every frame, g2 for all lags, ring-averaged S(q,t) and g2, XSVS contrast for every exposure window.
Default workload = BASELINE.json configs[1] ("c2": N = 32000, 100 Brownian frames, 256 x 256 lattice plane,
g2 tau = 1..50).  Metric: atom.q pairs/s for I(q,t) (whole job, all ranks).  Multi-GPU = weak scaling: every
rank processes its own independent trajectory (no data-path collective).
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


def run_qslab(args, cfg, ws, rank, dev, dist):
    """--qslab: every rank holds the same trajectory and computes its slab of detector rows; one NCCL all-reduce of
    the ring / XSVS moments per step; value = the whole detector's pairs / the max-over-ranks step time."""
    import torch
    import paper_2204_13241_b200 as xp
    from paper_2204_13241_b200 import pipeline
    from paper_2204_13241_b200 import dist as xd
    assert cfg.n_plane and not cfg.two_species, "--qslab: lattice configs with unit form factors (c2)"
    wl = pipeline.workload_from_config(cfg, device=dev)
    wl.engine = {"auto": xp.ENGINE_AUTO, "simt": xp.ENGINE_SIMT, "tensor": xp.ENGINE_TENSOR,
                 "i8": xp.ENGINE_TENSOR_I8}[args.engine]
    Q = pipeline.QSlabPipeline(wl, rank, ws, device=dev)
    pos_d = torch.from_numpy(xi.positions(cfg)).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        Q.run(pos_d, None)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    t_ms = []
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            flush.zero_()
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            Q.run(pos_d, None)
            b.record(stream)
            torch.cuda.synchronize()
            t_ms.append(a.elapsed_time(b))
    ms = xd.max_over_ranks(float(np.mean(t_ms)), dev)
    pairs = int(cfg.N) * int(cfg.n_plane) ** 2 * int(cfg.T)
    if rank == 0:
        line = {"metric": METRIC, "value": pairs / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "mode": "qslab",
                "config": {"workload": cfg.name, "N": cfg.N, "n_q": cfg.n_plane ** 2, "frames": cfg.T,
                           "parallelism": f"q-slab x{ws} (one trajectory, detector rows split, moments all-reduced)",
                           "rows_per_rank": [xd.qslab(cfg.n_plane, -cfg.n_plane // 2, r, ws)[1] for r in range(ws)],
                           "allreduce_bytes": int(Q.mom.numel() * 8),
                           "l2": "flushed between timed steps (256 MB write, untimed)"},
                "e2e": None, "clocks": clk.summary(), "step_ms_all": t_ms}
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
    ap.add_argument("--config", default="c2", choices=sorted(xi.CONFIGS))
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
    ap.add_argument("--qslab", action="store_true",
                    help="strong scaling: ONE trajectory, the detector split into row slabs across the ranks, ring "
                         "moments all-reduced once per step (SURVEY 8(e)); lattice configs without species")
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
    if args.qslab:
        return run_qslab(args, cfg, ws, rank, dev, dist)
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

    # ---- roofline of the dominant kernel (intensity main kernel), CUDA events on its stream
    main_ms, main_n = prof["intensity_main"]
    per_launch_ms = main_ms / max(main_n, 1)
    launches_per_step = max(main_n // args.steps, 1)
    pairs_launch = pairs_step / launches_per_step
    peaks, peak_src = _peaks()
    sm_count, _ = xp.device_info()
    tc_used = bool(cfg.n_plane) and wl.in_dtype == xp.F32 and engine != xp.ENGINE_SIMT and \
        xp.engine_available(xp.ENGINE_TENSOR)
    i8_used = tc_used and xp.engine_resolved(engine, f_h is None) == xp.ENGINE_TENSOR_I8
    hybrid_share = None          # fraction of the pairs on the integer engine when kinds are split between engines
    if tc_used and engine == xp.ENGINE_AUTO and wl.kinds is not None:
        counts = np.bincount(wl.kinds, minlength=len(wl.kind_f))
        share = float(sum(xp.species_engines(counts, wl.kind_f))) / float(counts.sum())
        if 0.0 < share < 1.0:
            hybrid_share = share
        i8_used = share == 1.0
    # the tensor peak: MEASURED_PEAKS' burst bf16 figure (cuBLAS at full clock) when the SM clock stayed at its max
    # through the timed region (no power capping: the kernel ran at the clock the burst figure was taken at), else
    # the sustained figure (cuBLAS back to back for 4 s, power-capped clocks)
    clk_sum = clk.summary()
    at_max = bool(clk_sum.get("sm_mhz") and clk_sum.get("sm_max_mhz") and clk_sum["sm_mhz"] >= 0.97 * clk_sum["sm_max_mhz"])
    tensor_peak = peaks["bf16_tflops"] if at_max else peaks["bf16_tflops_sustained"]
    if cfg.n_plane == 0:
        # generic q: 2 XU (MUFU) ops per pair; peak = 148 SM x 16 XU/clk x max clock
        peak = sm_count * 16 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 2 / 1e12
        roof = {"bound": "alu", "unit": "Tpairs/s (XU: 2 MUFU per pair)", "peak": peak,
                "achieved": pairs_launch / (per_launch_ms / 1e3) / 1e12}
    elif hybrid_share is not None:
        # kinds split between the integer (int8, 2x rate) and split-FP16 engines: 24 ops per pair on both; the
        # peak is the pair-weighted harmonic blend, over the whole intensity stage of a step (both kernels)
        peak = 1.0 / (hybrid_share / (2.0 * tensor_peak) + (1.0 - hybrid_share) / tensor_peak)
        stage_ms = main_ms / max(args.steps, 1)
        roof = {"bound": "tensor", "unit": "T ops/s (int8 + fp16 blend)", "peak": peak,
                "achieved": 24.0 * pairs_step / (stage_ms / 1e3) / 1e12, "int8_pair_share": hybrid_share}
        per_launch_ms = stage_ms
        pairs_launch = pairs_step
    elif i8_used:
        # tcgen05 kind::i8: 3 int8 limb products x 4 real MAC = 24 int8 ops per pair vs the int8 dense peak =
        # 2 x the measured bf16 (= fp16) peak (B200: 4.5 POPS int8 vs 2.25 PFLOP/s fp16 nominal; tools/mma_rate.cu
        # measured 8192 vs 4096 MAC/clk/SM)
        peak = 2.0 * tensor_peak
        roof = {"bound": "tensor", "unit": "TOPS (int8)", "peak": peak,
                "achieved": 24.0 * pairs_launch / (per_launch_ms / 1e3) / 1e12}
    elif tc_used:
        # tcgen05 split-FP16: 3 fp16 products x 4 real MAC = 24 flop per pair vs measured bf16 (= fp16) dense peak
        peak = tensor_peak
        roof = {"bound": "tensor", "unit": "TFLOP/s", "peak": peak,
                "achieved": 24.0 * pairs_launch / (per_launch_ms / 1e3) / 1e12}
    else:
        # FP32 CUDA cores: 1 complex MAC = 4 FMA = 8 flop per pair; peak = 148 x 128 FMA/clk x 2 x max clock
        peak = sm_count * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        roof = {"bound": "alu", "unit": "TFLOP/s (FP32 FMA pipe)", "peak": peak,
                "achieved": 8.0 * pairs_launch / (per_launch_ms / 1e3) / 1e12}
    roof["frac"] = roof["achieved"] / roof["peak"]
    if wl.in_dtype == xp.F64:
        # config 1 (4.1e6 pairs, FP64): launch/latency-bound; the FP32 figure above is context only
        roof["note"] = "FP64 workload: latency-bound, report ms_per_step; frac against the FP32 pipe is context only"
    eng_name = "i8+tensor" if hybrid_share is not None else \
        ("i8" if i8_used else ("tensor" if tc_used else ("simt" if cfg.n_plane else "generic")))
    roof["traffic"] = _traffic(cfg.name, eng_name, pairs_launch)
    tensor_src = (f"{peak_src}, {'burst' if at_max else 'sustained'} bf16"
                  + (" x 2 (int8)" if i8_used else (" blended int8/fp16" if hybrid_share else "")))
    roof["peak_source"] = tensor_src if roof["bound"] == "tensor" else "derived (DESIGN.md)"
    if roof["bound"] == "tensor":
        # context: the same achieved rate against the tcgen05 issue rate microbenchmarked at the run's SM clock
        # (tools/mma_rate.cu: 8190 int8 / 4095 fp16 MAC per clock per SM; 2 ops per MAC), which sits above the
        # cuBLAS-measured peak the roofline uses (cuBLAS runs power-capped, MEASURED_PEAKS clocks_under_load)
        mhz_run = clk_sum.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        if hybrid_share is not None:
            rate = 1.0 / (hybrid_share / 8190.0 + (1.0 - hybrid_share) / 4095.0)
        else:
            rate = 8190.0 if i8_used else 4095.0
        mma_peak = sm_count * rate * 2 * mhz_run * 1e6 / 1e12
        roof["vs_mma_issue_rate"] = {"peak": mma_peak, "frac": roof["achieved"] / mma_peak,
                                     "clock_mhz": mhz_run, "source": "tools/mma_rate.cu"}
    if roof["frac"] > 1.0:
        roof["note"] = ("frac > 1: the peak is the cuBLAS bf16 matmul figure of MEASURED_PEAKS (x 2 for int8), taken "
                        "while the matmul ran power-capped (clocks_under_load median "
                        f"{peaks.get('clocks_under_load', {}).get('sm_mhz_median', '?')} MHz), whereas this kernel ran "
                        f"at {clk_sum.get('sm_mhz')} MHz; vs_mma_issue_rate is the same rate against the tcgen05 "
                        "issue rate (tools/mma_rate.cu) at this run's clock")
    roof["kernel_ms"] = per_launch_ms
    roof["kernel_share_of_step"] = main_ms / args.steps / ms if ms > 0 else None

    # ---- end to end through the public API from pinned host memory
    e2e = None
    if not args.no_e2e:
        P.alloc_host_io(pos_h, f_h, batches=args.e2e_batches)
        P.run_host()
        torch.cuda.synchronize()
        auto_slots = 3 if pos_h.nbytes < (512 << 20) else 2
        slots = 1 if args.no_graph else (args.e2e_slots if args.e2e_slots > 0 else auto_slots)
        e_ms = None
        if not args.no_graph:
            try:
                e_ms = _e2e_streamed(args, P, pipeline, wl, dev, pos_h, f_h, slots, stream, dist)
            except Exception:                                  # capture failed: eager host steps instead
                torch.cuda.synchronize()
                slots = 1
        if e_ms is None:
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
            e_ms = float(np.mean(t_e))
        e_ms = xd.max_over_ranks(e_ms, dev)
        h2d, d2h = P.io_bytes()
        e2e = {"value": ws * pairs_step / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms, "streams": slots,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

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
    # XSVS: one read of the intensity series per exposure window (L2 / HBM streaming)
    if cfg.windows:
        _sec("xsvs", "hbm", float(len(cfg.windows)) * i_bytes, hbm, "GB/s")
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
                "vs_baseline": None, "dtype": "f64" if wl.in_dtype == xp.F64 else "f32", "data": "synthetic",
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
                                  "kernel_ms are from the timed graph replays, where they run concurrently"}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
