#!/usr/bin/env python
"""Table 1 of the paper on the B200 (context line, not the bench headline): Algorithm 1 on the 81 x 81 x 81
reciprocal-lattice grid of one N = 4000, L = 59.19 frame (paper: 416.8243 s per frame on
"32 CPUs", 4.1836 s for the 81 x 81 slice).  Device time per frame with CUDA events, L2 flushed between reps;
the FP64 oracle timed on the host cores on a bounded sample.

    python tools/bench_table1.py [--reps 20] [--engine auto|simt|tensor]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import xpcs_inputs as xi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_2204_13241_b200 as xp
    t1 = xi.TABLE1
    n, h = t1["n"], t1["n"] // 2
    pos = xi.uniform_frame(t1["seed"], t1["N"], t1["L"], "f32")[None]
    dev = torch.device("cuda", 0)
    pos_d = torch.from_numpy(pos).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {"what": "Table 1 (PAPER.md:459): Algorithm 1, 81^3 lattice grid, N = 4000, one frame",
           "paper_s_per_frame": {"81^3 grid": 416.8243, "81^2 slice": 4.1836, "single q": 0.0015}}
    for name, shape in (("81^3 grid", (-h, n, -h, n, -h, n)), ("81^2 slice", (-h, n, -h, n, 0, 1))):
        v = xp.qvolume(t1["L"], *shape)
        pairs = t1["N"] * v.n_q
        for eng_name, eng in (("i8", xp.ENGINE_TENSOR_I8), ("tensor", xp.ENGINE_TENSOR), ("simt", xp.ENGINE_SIMT)):
            I = xp.xpcs_intensity_volume(pos_d, None, v, engine=eng)
            for _ in range(args.warmup):
                xp.xpcs_intensity_volume(pos_d, None, v, out=I, engine=eng)
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                xp.xpcs_intensity_volume(pos_d, None, v, out=I, engine=eng)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = float(np.median(ts))
            out[f"{name} {eng_name}"] = {"ms_per_frame": ms, "pairs": pairs, "pairs_per_s": pairs / (ms / 1e3),
                                         "speedup_vs_paper": out["paper_s_per_frame"][name] / (ms / 1e3)}
    # oracle on the host cores: 2 l-planes of the grid (2 x 6561 q x 4000 atoms)
    import oracle
    q = oracle.lattice_volume_q(t1["L"], -h, n, -h, n, 0, 2)
    oracle.intensity(pos[0], None, q[:100], t1["L"])
    t0 = time.perf_counter()
    oracle.intensity(pos[0], None, q, t1["L"])
    dt = time.perf_counter() - t0
    out["oracle"] = {"pairs_per_s": t1["N"] * q.shape[0] / dt, "cores": oracle.threads(),
                     "sample": f"2 l-planes ({q.shape[0]} q) x {t1['N']} atoms, {dt:.2f} s",
                     "extrapolated_s_per_81^3_frame": dt * n / 2}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
