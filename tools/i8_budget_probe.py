"""Precision probe for AUTO's integer-engine error budget on the two-species configs (c3, c5): the species path with
f_max hints [1, 2] at several budgets (XPCS_I8_BUDGET; the share of pairs on the integer engine grows with it), vs
the FP64 oracle on sampled pixels of full-size frames (one oracle pass reused for every budget).  Prints per config
and budget: integer-engine pair share, worst |dI| / (1e-3 N + 1e-5 I) (the per-pixel gate ratio), rms |dI| / N.
    PROBE_PIXELS=30000 python tools/i8_budget_probe.py"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402

budgets = [float(b) for b in os.environ.get("PROBE_BUDGETS", "1.0,1.5,1.75,2.0,2.5").split(",")]
out = {}
for name, frames in (("c3", [0, 500, 999]), ("c5", [0, 199])):
    cfg = xi.CONFIGS[name]
    pos = xi.positions(cfg)[frames]
    f = xi.form_factors(cfg)
    n = cfg.n_plane
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(n))
    pix = xi.pixel_subset(q.shape[0], int(os.environ.get("PROBE_PIXELS", "3000")), 5)
    ref = oracle.intensity(pos, f.astype(np.float64), q[pix], cfg.L)
    sp = (f > 1.5).astype(np.int32)
    fq = torch.ones((2, n * n), dtype=torch.float32, device="cuda")
    fq[1] = 2.0
    d = torch.from_numpy(pos).cuda()
    v = xp.qvolume(cfg.L, -n // 2, n, -n // 2, n, 0, 1)
    counts = np.bincount(sp, minlength=2)
    res = {}
    for b in budgets:
        os.environ["XPCS_I8_BUDGET"] = str(b)
        I = xp.xpcs_intensity_volume(d, None, v, species=sp, f_q=fq, f_max=[1.0, 2.0]).cpu().numpy()
        err = np.abs(I[:, pix] - ref)
        ratio = err / (1e-3 * cfg.N + 1e-5 * ref)
        share = sum(xp.species_engines(counts, [1.0, 2.0], budget=b)) / counts.sum()
        res[str(b)] = {"i8_pair_share": float(share), "worst_ratio": float(ratio.max()),
                       "rms_dI_over_N": float(np.sqrt(np.mean((err / cfg.N) ** 2))), "samples": int(err.size)}
        print(name, b, res[str(b)], flush=True)
    out[name] = res
print(json.dumps(out))
