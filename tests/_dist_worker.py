"""Worker of tests/test_dist_cpu.py: one rank of a gloo process group (env RANK / WORLD_SIZE / MASTER_*)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import xpcs_inputs as xi  # noqa: E402
from paper_2204_13241_b200 import dist as xd  # noqa: E402


def main(out_path):
    dist.init_process_group("gloo")
    rank, world = xd.world()
    try:
        out = {"rank": rank, "world": world}
        out["shard"] = list(xd.shard(101, rank, world))
        out["max"] = xd.max_over_ranks(1.5 + rank)
        cfg = xi.scaled(xi.CONFIGS["c2"], N=400, T=2)
        pos = xi.positions(cfg)
        n = 64
        h0, n_h, row0 = xd.qslab(n, -n // 2, rank, world)
        q = oracle.lattice_q(cfg.L, h0, n_h, -n // 2, n)
        I = oracle.intensity(pos, None, q, cfg.L)
        bins = oracle.lattice_bins(n).reshape(n, n)[row0:row0 + n_h].ravel()
        out["rings"] = np.nan_to_num(xd.allreduce_ring_means(I, bins, 32), nan=-1.0).tolist()
        out["seed"] = xd.trajectory_seed(cfg.seed, rank)
        # the q-slab pipeline's moment all-reduce (one flat FP64 buffer) on the gloo group
        import torch
        from paper_2204_13241_b200.pipeline import QSlabPipeline
        t = torch.full((7,), float(rank + 1), dtype=torch.float64)
        QSlabPipeline._default_allreduce(t)
        out["allreduce"] = t.tolist()
        # XSVS from summed per-slab moments (m0, m1, m2 per window / snapshot / ring), the q-slab combine step
        wins = [1, 2]
        mom = []
        for W in wins:
            for sI in range(cfg.T // W):
                IW = I[sI * W:(sI + 1) * W].sum(0)
                for b in range(32):
                    sel = IW[bins == b]
                    mom.append([sel.size, sel.sum(), (sel * sel).sum()])
        tm = torch.tensor(mom, dtype=torch.float64)
        QSlabPipeline._default_allreduce(tm)
        m = tm.numpy().reshape(-1, 32, 3)
        beta, k = [], 0
        for W in wins:
            S = cfg.T // W
            mm = m[k:k + S]
            k += S
            with np.errstate(invalid="ignore", divide="ignore"):
                mean = mm[..., 1] / mm[..., 0]
                beta.append(np.where(mm[..., 0].min(0) > 0, ((mm[..., 2] / mm[..., 0] - mean ** 2) / mean ** 2).mean(0),
                                     np.nan))
        out["beta"] = np.nan_to_num(np.array(beta), nan=-1.0).tolist()
        dist.barrier()
    finally:
        dist.destroy_process_group()
    with open(out_path, "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main(sys.argv[1])
