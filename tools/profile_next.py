"""One small invocation of each SURVEY 8(f) kernel family for ncu (no timing, no oracle): species combine,
Gaussian form factors, 3-D volume, FFT method (spread + cuFFT + epilogue), speckle histogram, ISF."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402

cfg = xi.scaled(xi.CONFIGS["c2"], T=20)
pos = torch.from_numpy(xi.positions(cfg)).cuda()
g = xp.lattice_plane(cfg.L, 256)
v = xp.qvolume(cfg.L, -128, 256, -128, 256, 0, 1)
sp = xi.species_labels(cfg.N, 2, 1)
a, b, c = xi.gaussian_form_factor_coefficients(2)[0]
fq = torch.stack([xp.xpcs_form_factor_gaussian(*xi.gaussian_form_factor_coefficients(2)[s], vol=v) for s in range(2)])
I = xp.xpcs_intensity_volume(pos, None, v, species=sp, f_q=fq.contiguous())
A = xp.xpcs_intensity_grid(pos, None, g)
bins = xp.xpcs_lattice_bins(g, 32, 4)
H = xp.xpcs_speckle_histogram(A, bins, 32, 5, 64, 4.0)
Am = xp.xpcs_intensity_volume(pos, None, v, amplitude=True)
F = xp.xpcs_isf(Am, list(range(0, 10)))
blk = xp.qvolume(cfg.L, -32, 64, -32, 64, -32, 64)
Ifft = xp.xpcs_intensity_fft(pos[:2], blk, 160, cfg.L / 160)
torch.cuda.synchronize()
print("ok", xp.launch_count())
