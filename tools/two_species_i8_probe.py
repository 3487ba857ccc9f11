"""Precision probe: two-species configs (f = 1, 2) through the species path (kinds with constant f_s(q) rows) vs the
FP64 oracle, on sampled pixels of full-size c3 / c5 frames: both kinds on the integer engine, the AUTO hybrid
(f = 1 kind on the integer engine, f = 2 kind on split-FP16, from the f_max hints), and split-FP16 with per-atom f.
Prints the worst |dI| / (1e-3 N + 1e-5 I) and the rms |dI|/N."""
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

out = {}
for name, frames in (("c3", [0, 500, 999]), ("c5", [0, 199])):
    cfg = xi.CONFIGS[name]
    pos_all = xi.positions(cfg)
    pos = pos_all[frames]
    f = xi.form_factors(cfg)
    n = cfg.n_plane
    g = xp.lattice_plane(cfg.L, n)
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(n))
    pix = xi.pixel_subset(q.shape[0], int(os.environ.get("PROBE_PIXELS", "3000")), 5)
    ref = oracle.intensity(pos, f.astype(np.float64), q[pix], cfg.L)
    sp = (f > 1.5).astype(np.int32)
    fq = torch.ones((2, n * n), dtype=torch.float32, device="cuda")
    fq[1] = 2.0
    d = torch.from_numpy(pos).cuda()
    res = {}
    for eng_name, eng in (("i8_species", xp.ENGINE_TENSOR_I8), ("hybrid_auto", xp.ENGINE_AUTO),
                          ("fp16_peratom", xp.ENGINE_TENSOR)):
        if eng_name != "fp16_peratom":
            v = xp.qvolume(cfg.L, -n // 2, n, -n // 2, n, 0, 1)
            I = xp.xpcs_intensity_volume(d, None, v, species=sp, f_q=fq, engine=eng,
                                         f_max=[1.0, 2.0] if eng_name == "hybrid_auto" else None).cpu().numpy()
        else:
            I = xp.xpcs_intensity_grid(d, torch.from_numpy(f).cuda(), g, engine=eng).cpu().numpy()
        err = np.abs(I[:, pix] - ref)
        ratio = err / (1e-3 * cfg.N + 1e-5 * ref)
        res[eng_name] = {"worst_ratio": float(ratio.max()), "rms_dI_over_N": float(np.sqrt(np.mean((err / cfg.N) ** 2))),
                         "samples": int(err.size)}
    out[name] = res
print(json.dumps(out))
