"""Small instances of every kernel of libxpcs.so for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


cfg = xi.scaled(xi.CONFIGS["c3"], N=333, T=3)
pos = xi.positions(cfg)
f = xi.form_factors(cfg)
g = xp.qgrid(cfg.L, -70, 140, -60, 130, m0=(0, 0, 1))
for eng in (xp.ENGINE_TENSOR, xp.ENGINE_SIMT):
    xp.xpcs_intensity_grid(t(pos), t(f), g, engine=eng)
xp.xpcs_intensity_grid(t(pos.astype(np.float64)), t(f.astype(np.float64)), xp.qgrid(cfg.L, -8, 16, -8, 16))
q = xp.xpcs_qgrid_ewald(xi.EWALD_WAVELENGTH_SIGMA, 40, 37, xi.EWALD_PITCH_RAD * 10)
xp.xpcs_intensity(t(pos), t(f), q, cfg.L)
xp.xpcs_intensity(t(pos.astype(np.float64)), None, q.double(), cfg.L)
I = torch.rand(23, 4096, device="cuda")
xp.xpcs_g2(I, [0, 1, 3, 7, 22])
xp.xpcs_g2(I, list(range(1, 20)))
bins = xp.xpcs_lattice_bins(xp.lattice_plane(10.0, 64), 32, 1)
xp.xpcs_shell_mean(I, bins, 32)
xp.xpcs_structure_factor_shells(I, t(f[:100]), 100, bins, 32)
xp.xsvs_contrast(I, bins, 33, [1, 2, 5, 23])
xp.xpcs_radial_bins(q, xi.EWALD_QMAX, 32)
torch.cuda.synchronize()
print("sanitize case ok, launches", xp.launch_count())
