"""Run one hot-path case for profiling (ncu / compute-sanitizer) -- no timing, no oracle.

    python tools/profile_case.py c2            # one full pipeline pass of config 2 (bench launch config)
    python tools/profile_case.py c4 --frames 1 --pixels 65536
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402
from paper_2204_13241_b200 import pipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--pixels", type=int, default=0)
    ap.add_argument("--engine", default="auto", choices=["auto", "simt", "tensor", "i8"])
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    cfg = xi.CONFIGS[a.config]
    if a.frames:
        cfg = xi.scaled(cfg, T=a.frames, lags=tuple(l for l in cfg.lags if l < a.frames),
                        windows=tuple(w for w in cfg.windows if w <= a.frames))
    pos = torch.from_numpy(xi.positions(cfg)).cuda()
    f = torch.from_numpy(xi.form_factors(cfg)).cuda() if cfg.two_species else None
    wl = pipeline.workload_from_config(cfg)
    wl.engine = {"auto": xp.ENGINE_AUTO, "simt": xp.ENGINE_SIMT, "tensor": xp.ENGINE_TENSOR,
                 "i8": xp.ENGINE_TENSOR_I8}[a.engine]
    if a.pixels and wl.q is not None:
        wl.q = wl.q[: a.pixels].contiguous()
    P = pipeline.Pipeline(wl)
    for _ in range(a.repeat):
        P.run(pos, f)
    torch.cuda.synchronize()
    print("ok", a.config, P.pairs_per_step, xp.launch_count())


if __name__ == "__main__":
    main()
