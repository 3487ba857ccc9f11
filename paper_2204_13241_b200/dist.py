"""Multi-process plumbing for the direct method (one process per GPU, torch.distributed).

The path shards without any data-path exchange over independent problems (frames / trajectories: "parallelized
on 32 CPUs over atomic configurations") and over q ("the computations of scattered intensity for
different q vectors are independent").  The only collectives are
  * the timing reduction (max over ranks) of bench.py, and
  * in the q-slab mode, one all-reduce of the ring moments (count, sum) so that ring averages over a detector that
    is split across ranks equal the single-device result.
Everything here is host logic; it runs on gloo (CPU tests) and nccl (GPU) alike.
"""
from __future__ import annotations

import os

import numpy as np


def world():
    """(rank, world_size) of this process (1 process when torch.distributed is not initialised)."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except ImportError:
        pass
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def shard(n_units: int, rank: int, world_size: int):
    """Contiguous balanced share [lo, hi) of n_units for rank (sizes differ by at most 1)."""
    base, rem = divmod(int(n_units), int(world_size))
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def max_over_ranks(x: float, device=None) -> float:
    """Max of a scalar over all ranks (the bench's device time); identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(a, device=None):
    """Element-wise sum of an array over ranks (returns numpy float64)."""
    import torch
    import torch.distributed as dist
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if not (dist.is_available() and dist.is_initialized()):
        return arr
    t = torch.from_numpy(arr.copy())
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def trajectory_seed(base_seed: int, rank: int) -> int:
    """Weak scaling: rank r processes its own independent trajectory (a different seed)."""
    return int(base_seed) + 1000 * int(rank)


def qslab(n_h: int, h0: int, rank: int, world_size: int):
    """Detector slab of rank: rows [h0 + lo, h0 + hi) of an n_h-row lattice plane -> (h0_r, n_h_r, row offset)."""
    lo, hi = shard(n_h, rank, world_size)
    return h0 + lo, hi - lo, lo


def ring_moments(values, bins, n_bins):
    """Per-row ring moments (count of finite values, their sum) of a [rows][n_pix] slab; the host-side form of
    the combine step (the device reductions produce the same moments per rank)."""
    v = np.asarray(values, dtype=np.float64)
    if v.ndim == 1:
        v = v[None]
    cnt = np.zeros((v.shape[0], n_bins))
    s = np.zeros((v.shape[0], n_bins))
    for b in range(n_bins):
        sel = v[:, bins == b]
        ok = np.isfinite(sel)
        cnt[:, b] = ok.sum(1)
        s[:, b] = np.where(ok, sel, 0.0).sum(1)
    return cnt, s


def ring_means_from_moments(cnt, s):
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(cnt > 0, s / np.where(cnt > 0, cnt, 1), np.nan)


def allreduce_ring_means(values, bins, n_bins, device=None):
    """Ring averages over a detector split across ranks: all-reduce (count, sum), then divide."""
    cnt, s = ring_moments(values, bins, n_bins)
    both = sum_over_ranks(np.stack([cnt, s]), device)
    return ring_means_from_moments(both[0], both[1])
