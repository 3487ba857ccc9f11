"""Time the generic (explicit-q) kernel on a c4 slice: N = 1M atoms, FRAMES frames (env, default 1), the first PIXELS
Ewald pixels (env, default 262144; 1048576 = the whole c4 detector)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import xpcs_inputs as xi
import paper_2204_13241_b200 as xp
cfg = xi.CONFIGS["c4"]
FR = int(os.environ.get("FRAMES", "1"))
PX = int(os.environ.get("PIXELS", "262144"))
pos = torch.from_numpy(xi.positions(cfg, frames=FR)).cuda()
q = xp.xpcs_qgrid_ewald(xi.EWALD_WAVELENGTH_SIGMA, cfg.detector, cfg.detector, xi.EWALD_PITCH_RAD)[:PX].contiguous()
for _ in range(2):
    I = xp.xpcs_intensity(pos, None, q, cfg.L)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    I = xp.xpcs_intensity(pos, None, q, cfg.L)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
pairs = cfg.N * q.shape[0] * FR
print(json.dumps({"lib": os.environ.get("XPCS_LIB", "main"), "frames": FR, "pixels": PX, "ms": ms, "pairs_per_s": pairs / (ms / 1e3)}))
