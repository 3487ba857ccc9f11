"""Worker of tests/test_dist_cpu.py: one rank of a gloo process group (env RANK / WORLD_SIZE / MASTER_*).

Drives the product's q-sharding plumbing on CPU: the 2-D block decomposition (dist.qblocks), the one flat FP64
moment buffer (pipeline.MomentLayout) and its all-reduce (QShardPipeline._default_allreduce, torch.distributed).  The
per-block moments and the final combine are computed here with numpy from oracle intensities (the library's moment
kernels need a GPU; tests/test_gpu_qslab.py runs them)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import xpcs_inputs as xi  # noqa: E402
from paper_2204_13241_b200 import dist as xd  # noqa: E402
from paper_2204_13241_b200.pipeline import MomentLayout, QShardPipeline  # noqa: E402


def ring_moments(values, bins, n_bins):
    """[rows][n_pix] -> [rows][n_bins][2] (count of finite values, their sum): xpcs_ring_moments' layout."""
    v = np.asarray(values, dtype=np.float64)
    out = np.zeros((v.shape[0], n_bins, 2))
    for b in range(n_bins):
        sel = v[:, bins == b]
        ok = np.isfinite(sel)
        out[:, b, 0] = ok.sum(1)
        out[:, b, 1] = np.where(ok, sel, 0.0).sum(1)
    return out


def xsvs_moments(I, bins, n_bins, windows):
    """[n_slots][n_bins][3] (m0, m1, m2 of I_W over the ring per window and snapshot): xsvs_moments' layout."""
    mom = []
    for W in windows:
        for s in range(I.shape[0] // W):
            IW = I[s * W:(s + 1) * W].sum(0)
            mom.append([[np.sum(bins == b), IW[bins == b].sum(), (IW[bins == b] ** 2).sum()] for b in range(n_bins)])
    return np.array(mom, dtype=np.float64)


def main(out_path):
    dist.init_process_group("gloo")
    rank, world = xd.world()
    try:
        out = {"rank": rank, "world": world}
        out["shard"] = list(xd.shard(101, rank, world))
        out["max"] = xd.max_over_ranks(1.5 + rank)
        out["seed"] = xd.trajectory_seed(220413241, rank)
        cfg = xi.scaled(xi.CONFIGS["c2"], N=400, T=6)
        pos = xi.positions(cfg)
        n, nb, lags, wins = 64, 32, [1, 2], [1, 2, 4]
        (h0, n_h, k0, n_k), (row0, col0, ph, pk) = xd.qblocks(n, n, -n // 2, -n // 2, rank, world)
        out["block"] = [h0, n_h, k0, n_k]
        q = oracle.lattice_q(cfg.L, h0, n_h, k0, n_k)
        I = oracle.intensity(pos, None, q, cfg.L)
        bins = oracle.lattice_bins(n).reshape(n, n)[row0:row0 + n_h, col0:col0 + n_k].ravel()
        g2 = oracle.g2(I, lags)
        lay = MomentLayout(cfg.T, len(lags), sum(cfg.T // w for w in wins), nb)
        m = torch.zeros(lay.total, dtype=torch.float64)
        mS, mG, mX = lay.views(m)
        mS.copy_(torch.from_numpy(ring_moments(I, bins, nb)))
        mG.copy_(torch.from_numpy(ring_moments(g2, bins, nb)))
        mX.copy_(torch.from_numpy(xsvs_moments(I, bins, nb, wins)))
        QShardPipeline._default_allreduce(m)
        mS, mG, mX = (v.numpy() for v in lay.views(m))
        with np.errstate(invalid="ignore", divide="ignore"):
            out["S_rings"] = np.nan_to_num(mS[..., 1] / mS[..., 0] / cfg.N, nan=-1.0).tolist()
            out["g2_rings"] = np.nan_to_num(mG[..., 1] / mG[..., 0], nan=-1.0).tolist()
            beta, k = [], 0
            for W in wins:
                S = cfg.T // W
                mm = mX[k:k + S]
                k += S
                mean = mm[..., 1] / mm[..., 0]
                beta.append(np.where(mm[..., 0].min(0) > 0,
                                     ((mm[..., 2] / mm[..., 0] - mean ** 2) / mean ** 2).mean(0), np.nan))
            out["beta"] = np.nan_to_num(np.array(beta), nan=-1.0).tolist()
        dist.barrier()
    finally:
        dist.destroy_process_group()
    with open(out_path, "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main(sys.argv[1])
