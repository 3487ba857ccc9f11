"""Quick tcgen05-engine check against the oracle (prints error statistics)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402

print("tensor available:", xp.engine_available(xp.ENGINE_TENSOR), "chunk", os.environ.get("XPCS_CHUNK_ATOMS"), "dbg", os.environ.get("XPCS_TC_DEBUG"))
for (N, nh, nk, T) in [(16, 128, 128, 1), (256, 128, 128, 1), (1024, 128, 128, 1), (4096, 128, 128, 1), (16384, 128, 128, 1)]:
    cfg = xi.scaled(xi.CONFIGS["c3"], N=N, T=T)
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg)
    g = xp.qgrid(cfg.L, -nh // 2, nh, -nk // 2, nk)
    t0 = time.time()
    I = xp.xpcs_intensity_grid(torch.from_numpy(pos).cuda(), torch.from_numpy(f).cuda(), g, engine=xp.ENGINE_TENSOR)
    torch.cuda.synchronize()
    I = I.cpu().numpy()
    q = oracle.lattice_q(g.L, g.h0, g.n_h, g.k0, g.n_k)
    ref = oracle.intensity(pos, f.astype(np.float64), q, cfg.L)
    err = np.abs(I - ref)
    print(f"N={N} {nh}x{nk} T={T}: max|dI|/N={err.max()/N:.3e} rms/N={np.sqrt((err**2).mean())/N:.3e} "
          f"gate={np.max(err/(1e-3*N+1e-5*ref)):.3e} mean I/N={I.mean()/N:.3f} ref {ref.mean()/N:.3f} ({time.time()-t0:.1f}s)",
          flush=True)
