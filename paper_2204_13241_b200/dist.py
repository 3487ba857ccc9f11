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


# the tensor engines' pair tile (k_lattice_i8.cu / k_lattice_tc.cu): 256 rows h x 128 columns k
TILE_H, TILE_K = 256, 128


def _split_aligned(n: int, parts: int, unit: int, idx: int):
    """[lo, hi) of part idx when n is split into `parts` contiguous ranges: whole multiples of `unit` while there are
    at least as many units as parts (balanced in units), else an even split."""
    units = -(-n // unit)
    if parts <= units:
        ulo, uhi = shard(units, idx, parts)
        return min(n, ulo * unit), min(n, uhi * unit)
    return shard(n, idx, parts)


def qblocks(n_h: int, n_k: int, h0: int, k0: int, rank: int, world_size: int):
    """2-D block of a lattice plane for rank: the factorisation world = ph x pk whose blocks need the fewest pair
    tiles on the busiest rank (ties: the most even pixel split), rows and columns cut at tile boundaries where
    possible.  Returns ((h0_r, n_h_r, k0_r, n_k_r), (row0, col0, ph, pk))."""
    best = None
    for ph in range(1, world_size + 1):
        if world_size % ph:
            continue
        pk = world_size // ph
        tiles, pix = [], []
        for r in range(world_size):
            hl, hh = _split_aligned(n_h, ph, TILE_H, r // pk)
            kl, kh = _split_aligned(n_k, pk, TILE_K, r % pk)
            tiles.append(-(-(hh - hl) // TILE_H) * -(-(kh - kl) // TILE_K))
            pix.append((hh - hl) * (kh - kl))
        key = (max(tiles), max(pix) - min(pix), ph)
        if best is None or key < best[0]:
            best = (key, ph, pk)
    _, ph, pk = best
    hl, hh = _split_aligned(n_h, ph, TILE_H, rank // pk)
    kl, kh = _split_aligned(n_k, pk, TILE_K, rank % pk)
    return (h0 + hl, hh - hl, k0 + kl, kh - kl), (hl, kl, ph, pk)
