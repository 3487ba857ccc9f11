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
# round 2: the integer engine (single chunk, several chunks), species with f_max hints (integer + split-FP16 engines,
# species combine, bright-pixel fix-up), the XSVS gather paths (four pixels per lane, one, the long-series kernel),
# block-streamed g2, XSVS / ring moments
if os.environ.get("SAN_SKIP_TENSOR") != "1":
    xp.xpcs_intensity_grid(t(pos), None, g, engine=xp.ENGINE_TENSOR_I8)
    os.environ["XPCS_CHUNK_ATOMS"] = "128"
    xp.xpcs_intensity_grid(t(pos), None, g, engine=xp.ENGINE_TENSOR_I8)
    del os.environ["XPCS_CHUNK_ATOMS"]
    sp = (f > 1.5).astype(np.int32)
    v = xp.qvolume(cfg.L, -40, 80, -30, 70, 0, 1)
    fq = torch.stack([torch.full((80 * 70,), 1.0), torch.full((80 * 70,), 4.0)]).cuda()
    xp.xpcs_intensity_volume(t(pos), None, v, species=sp, f_q=fq, f_max=[1.0, 4.0])
Iw = torch.rand(37, 256 * 256, device="cuda")
bw = xp.xpcs_lattice_bins(xp.lattice_plane(10.0, 256), 32, 4)
xp.xsvs_contrast(Iw, bw, 33, [1, 2, 3, 8, 36])
xp.xsvs_moments(Iw, bw, 33, [1, 4])
xp.xpcs_ring_moments(Iw, bw, 33)
Il = torch.rand(16500, 64, device="cuda")
bl = torch.arange(64, device="cuda", dtype=torch.int32) % 3
xp.xsvs_contrast(Il, bl, 3, [1, 1000])
S = xp.G2Stream(4096, [0, 1, 3, 7, 12], device="cuda")
for a in range(0, 23, 5):
    S.push(I[a:a + 5].contiguous())
S.result()
torch.cuda.synchronize()
print("sanitize case ok, launches", xp.launch_count())
