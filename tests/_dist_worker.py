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
        dist.barrier()
    finally:
        dist.destroy_process_group()
    with open(out_path, "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main(sys.argv[1])
