"""Run one lattice-plane call (c2 or c3 shape) so ncu can capture the bright-pixel recompute kernels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import xpcs_inputs as xi
import paper_2204_13241_b200 as xp
cfg = xi.scaled(xi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"], T=int(sys.argv[2]) if len(sys.argv) > 2 else 100)
pos = torch.from_numpy(xi.positions(cfg)).cuda()
g = xp.lattice_plane(cfg.L, cfg.n_plane)
for _ in range(2):
    I = xp.xpcs_intensity_grid(pos, None, g)
torch.cuda.synchronize()
print("ok", float(I[0].max()), cfg.N ** 2)
