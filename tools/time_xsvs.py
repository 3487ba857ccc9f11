"""Time xsvs_contrast alone (CUDA events, 20 calls after warm-up) on the c2 / c5 / c3 shapes: the config's rings and
windows, exponential (fully developed speckle) intensities.  XPCS_LIB selects a variant build."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import xpcs_inputs as xi
import paper_2204_13241_b200 as xp
from paper_2204_13241_b200 import pipeline

res = {"lib": os.path.basename(os.environ.get("XPCS_LIB", "main"))}
for name in sys.argv[1:] or ["c2", "c5", "c3"]:
    cfg = xi.CONFIGS[name]
    wl = pipeline.workload_from_config(cfg)
    P = pipeline.Pipeline(wl)
    n_q = P.bins.numel()
    g = torch.Generator(device="cuda").manual_seed(1)
    I = torch.empty((cfg.T, n_q), device="cuda", dtype=torch.float32).exponential_(generator=g)
    out = torch.empty((len(wl.windows), wl.n_bins), dtype=torch.float64, device="cuda")
    for _ in range(3):
        xp.xsvs_contrast(I, P.bins, wl.n_bins, wl.windows, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        xp.xsvs_contrast(I, P.bins, wl.n_bins, wl.windows, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    n_valid = int(((P.bins >= 0) & (P.bins < wl.n_bins)).sum())
    t_use = max((cfg.T // w) * w for w in wl.windows)
    res[name] = {"ms": round(ms, 4), "hbm_frac": round(t_use * n_valid * 4 / (ms * 1e-3) / 6.55e12, 3),
                 "beta00": float(out[0, 0])}
    P.close()
print(json.dumps(res))
