"""Time xpcs_g2 alone (CUDA events, 5 calls after warm-up) on the c2 / c3 shapes (the config's lag list, exponential
intensities).  Prints ms and the fraction of the measured FP64 DFMA rate (17.1e12/s).  XPCS_LIB selects a
variant build."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import xpcs_inputs as xi
import paper_2204_13241_b200 as xp

res = {"lib": os.path.basename(os.path.dirname(os.environ["XPCS_LIB"])) if "XPCS_LIB" in os.environ else "main"}
import threading
try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # clocks are optional context
    _h = None


def _sample(stop, out):
    while not stop.is_set():
        out.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
        stop.wait(0.002)
ref = None
for name in sys.argv[1:] or ["c2", "c3"]:
    cfg = xi.CONFIGS[name]
    n_q = cfg.n_plane * cfg.n_plane
    g = torch.Generator(device="cuda").manual_seed(1)
    I = torch.empty((cfg.T, n_q), device="cuda", dtype=torch.float32).exponential_(generator=g)
    out = torch.empty((len(cfg.lags), n_q), dtype=torch.float32, device="cuda")
    for _ in range(2):
        xp.xpcs_g2(I, cfg.lags, out=out, out_dtype=xp.F32)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks, stop = [], threading.Event()
    th = threading.Thread(target=_sample, args=(stop, clocks)) if _h is not None else None
    if th:
        th.start()
    a.record()
    for _ in range(5):
        xp.xpcs_g2(I, cfg.lags, out=out, out_dtype=xp.F32)
    b.record()
    torch.cuda.synchronize()
    if th:
        stop.set()
        th.join()
    ms = a.elapsed_time(b) / 5
    dfma = sum(cfg.T - t for t in cfg.lags) * n_q
    res[name] = {"ms": round(ms, 4), "fp64_frac": round(dfma / (ms * 1e-3) / 17.1e12, 3),
                 "checksum": float(out.double().sum()),
                 "sm_mhz": sorted(clocks)[len(clocks) // 2] if clocks else None}
    for B in (int(b) for b in os.environ.get("XPCS_G2_STREAM", "").split(",") if b):
        # block-streamed g2 of the same series in blocks of B frames (state reset untimed)
        S = xp.G2Stream(n_q, cfg.lags, dtype=torch.float32)
        reps, tot = 3, 0.0
        for rep in range(reps + 1):
            S.acc.zero_(); S.sum.zero_(); S.t = 0
            torch.cuda.synchronize()
            a.record()
            for t in range(0, cfg.T, B):
                S.push(I[t:t + B])
            S.result(out=out, out_dtype=xp.F32)
            b.record()
            torch.cuda.synchronize()
            if rep:
                tot += a.elapsed_time(b)
        res[name][f"stream_{B}_ms"] = round(tot / reps, 4)
        res[name][f"stream_{B}_checksum"] = float(out.double().sum())
print(json.dumps(res))
