"""Where the end-to-end time of the c2 step goes: pinned H2D / D2H bandwidth alone, the device pass, and
Pipeline.run_host with different frame-batch counts (CUDA events, medians of 10)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import xpcs_inputs as xi  # noqa: E402
from paper_2204_13241_b200 import pipeline  # noqa: E402


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


cfg = xi.CONFIGS["c2"]
pos = xi.positions(cfg)
hp = torch.from_numpy(pos).pin_memory()
dp = torch.empty_like(hp, device="cuda")
ho = torch.empty(39361792 // 4, dtype=torch.float32).pin_memory()
do = torch.empty_like(ho, device="cuda")
out = {"h2d_ms": timed(lambda: dp.copy_(hp, non_blocking=True)), "d2h_ms": timed(lambda: ho.copy_(do, non_blocking=True))}
s2 = torch.cuda.Stream()


def both():
    dp.copy_(hp, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


out["h2d_d2h_concurrent_ms"] = timed(both)
out["h2d_GBs"] = hp.numel() * 4 / out["h2d_ms"] / 1e6
out["d2h_GBs"] = ho.numel() * 4 / out["d2h_ms"] / 1e6
wl = pipeline.workload_from_config(cfg)
P = pipeline.Pipeline(wl)
d_pos = torch.from_numpy(pos).cuda()
P.run(d_pos, None)
out["device_ms"] = timed(lambda: P.run(d_pos, None))
for nb in (1, 2, 4, 8, 16):
    P.alloc_host_io(pos, None, batches=nb)
    P.run_host()
    out[f"run_host_b{nb}_ms"] = timed(P.run_host)
print(json.dumps(out))
