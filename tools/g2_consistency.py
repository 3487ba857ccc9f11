"""g2 kernel time inside a c3 pipeline step (per-class profile, serial reductions) vs xpcs_g2 timed alone on the same
I (CUDA events) -- one process, one GPU."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import xpcs_inputs as xi
import paper_2204_13241_b200 as xp
from paper_2204_13241_b200 import pipeline

cfg = xi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
wl = pipeline.workload_from_config(cfg)
P = pipeline.Pipeline(wl)
P.serial_reductions = True
pos = torch.from_numpy(xi.positions(cfg)).cuda()
f = torch.from_numpy(xi.form_factors(cfg)).cuda() if cfg.two_species else None
P.run(pos, f)
torch.cuda.synchronize()
res = {}
for rep in range(2):
    xp.profile_reset()
    P.run(pos, f, profile=True)
    torch.cuda.synchronize()
    res[f"pipeline_g2_ms_{rep}"] = xp.profile_query()["g2"][0]
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = torch.empty_like(P.g2)
for rep in range(2):
    a.record()
    xp.xpcs_g2(P.I, wl.lags, out=out, out_dtype=xp.F32)
    b.record()
    torch.cuda.synchronize()
    res[f"alone_g2_ms_{rep}"] = a.elapsed_time(b)
xp.profile_reset()
xp.xpcs_g2(P.I, wl.lags, out=out, out_dtype=xp.F32, profile=True)
torch.cuda.synchronize()
res["alone_profiled_ms"] = xp.profile_query()["g2"][0]
res["I_shape"] = list(P.I.shape)
res["lags"] = [min(wl.lags), max(wl.lags), len(wl.lags)]
print(json.dumps(res))
