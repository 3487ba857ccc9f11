"""The q-sharded single-trajectory mode: a detector split into tile-aligned blocks (lattice planes) or
pixel ranges (explicit q), each block's I, g2 and additive ring / XSVS moments computed separately, the moments
summed (the all-reduce), the ring results formed from the sums.  On one GPU the ranks run one after another (no rank waits on another) and the sum stands in for the
NCCL all-reduce; the result must equal the single-detector reductions up to summation order, and each slab's I must
equal the matching rows of the full-plane I within the per-pixel gate.  Also pins the moment entry points on their
own: moments of the full detector reproduce xpcs_shell_mean / xsvs_contrast."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402
from paper_2204_13241_b200 import pipeline  # noqa: E402
from paper_2204_13241_b200 import dist as xd  # noqa: E402
from _gates import assert_pixels, assert_rel  # noqa: E402

DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    xp.load()
    yield
    xp.release()


def _cfg():
    return xi.scaled(xi.CONFIGS["c2"], N=3000, T=24, n_plane=96, lags=(1, 2, 3, 5), windows=(1, 2, 4, 7), n_bins=8)


def test_moment_entry_points_match_direct_reductions():
    cfg = _cfg()
    wl = pipeline.workload_from_config(cfg, device=DEV)
    P = pipeline.Pipeline(wl, device=DEV)
    out = P.run(torch.from_numpy(xi.positions(cfg)).to(DEV), None)
    torch.cuda.synchronize()
    I, g2 = out["I"], out["g2"]
    mS = xp.xpcs_ring_moments(I, P.bins, wl.n_bins)
    assert_rel(xp.xpcs_ring_means_from_moments(mS, 1.0 / cfg.N).cpu().numpy(), out["S_rings"].cpu().numpy(), 1e-12,
               "S rings from moments")
    mG = xp.xpcs_ring_moments(g2, P.bins, wl.n_bins)
    assert_rel(xp.xpcs_ring_means_from_moments(mG).cpu().numpy(), out["g2_rings"].cpu().numpy(), 1e-12, "g2 rings")
    mX = xp.xsvs_moments(I, P.bins, wl.n_bins, wl.windows)
    assert mX.shape[0] == xp.xsvs_n_slots(cfg.T, wl.windows)
    assert_rel(xp.xsvs_contrast_from_moments(mX, cfg.T, wl.windows).cpu().numpy(), out["beta"].cpu().numpy(), 1e-12,
               "beta from moments")
    # the count moment is the ring's pixel count, the same for every snapshot
    cnt = mX[:, :, 0].cpu().numpy()
    assert np.all(cnt == cnt[0])
    P.close()


def _shape(name):
    """Reduced inputs with the structure of each config: c2 (uniform f), c3 / c5 (two kinds, AUTO's hybrid engine
    split), c4 (explicit Ewald q list)."""
    if name == "c4":
        return xi.scaled(xi.CONFIGS["c4"], N=4000, T=6, detector=64, lags=(1, 2), windows=(1, 2), n_bins=8)
    base = xi.CONFIGS[name]
    return xi.scaled(base, N=3000, T=24, n_plane=96, lags=(1, 2, 3, 5), windows=(1, 2, 4, 7), n_bins=8)


@pytest.mark.parametrize("name,world", [("c2", 2), ("c2", 3), ("c3", 2), ("c3", 4), ("c5", 3), ("c4", 2), ("c4", 3)])
def test_qshard_split_equals_full_detector(name, world):
    """One trajectory, the detector split across `world` ranks run one after another on this GPU (no rank waits on
    another; the sum stands in for the NCCL all-reduce): ring results within the ring gate of the full detector,
    every block's I within the per-pixel gate of the matching full-detector pixels, and the blocks tile it."""
    cfg = _shape(name)
    pos = torch.from_numpy(xi.positions(cfg)).to(DEV)
    f = torch.from_numpy(xi.form_factors(cfg)).to(DEV) if cfg.two_species else None
    wl = pipeline.workload_from_config(cfg, device=DEV)
    P = pipeline.Pipeline(wl, device=DEV)
    full = {k: v.clone() for k, v in P.run(pos, f).items() if torch.is_tensor(v)}
    ranks = [pipeline.QShardPipeline(wl, r, world, device=DEV, allreduce=lambda t: None) for r in range(world)]
    total = None
    for Q in ranks:
        m = Q.local(pos, f).clone()
        total = m if total is None else total + m
    torch.cuda.synchronize()
    res = ranks[0].finish(f, moments=total)
    for key in ("S_rings", "g2_rings", "beta"):
        assert_rel(res[key].cpu().numpy(), full[key].cpu().numpy(), 1e-4, f"q-shard {key} ({name}, world {world})")
    I_full = full["I"].cpu().numpy()
    g2_full = full["g2"].cpu().numpy()
    covered = np.zeros(I_full.shape[1], dtype=int)
    for Q in ranks:
        if Q.grid is not None:
            n = cfg.n_plane
            row0, col0, _, _ = Q.block
            idx = ((np.arange(Q.grid.n_h)[:, None] + row0) * n + col0 + np.arange(Q.grid.n_k)[None, :]).ravel()
        else:
            idx = np.arange(*Q.block)
        covered[idx] += 1
        assert_pixels(Q.I.cpu().numpy(), I_full[:, idx], cfg.N, f"{name} block {Q.rank} I")
        np.testing.assert_allclose(Q.g2.cpu().numpy(), g2_full[:, idx], rtol=1e-3)
        Q.close()
    assert np.all(covered == 1)
    P.close()


def test_qshard_decomposition_exact_on_identical_input():
    """The decomposition itself is exact: the full detector's I split into the blocks, the blocks' moments summed,
    reproduce the full-detector reductions to 1e-12 (only the summation order differs)."""
    cfg = _cfg()
    pos = torch.from_numpy(xi.positions(cfg)).to(DEV)
    wl = pipeline.workload_from_config(cfg, device=DEV)
    P = pipeline.Pipeline(wl, device=DEV)
    full = {k: v.clone() for k, v in P.run(pos, None).items() if torch.is_tensor(v)}
    n = cfg.n_plane
    tot_S = tot_G = tot_X = None
    for r in range(3):
        (h0, n_h, k0, n_k), (row0, col0, _, _) = xd.qblocks(n, n, -n // 2, -n // 2, r, 3)
        idx = torch.from_numpy(((np.arange(n_h)[:, None] + row0) * n + col0 + np.arange(n_k)[None, :]).ravel()).to(DEV)
        I_s = full["I"][:, idx].contiguous()
        g2_s = full["g2"][:, idx].contiguous()
        b_s = P.bins[idx].contiguous()
        mS = xp.xpcs_ring_moments(I_s, b_s, wl.n_bins)
        mG = xp.xpcs_ring_moments(g2_s, b_s, wl.n_bins)
        mX = xp.xsvs_moments(I_s, b_s, wl.n_bins, wl.windows)
        tot_S = mS if tot_S is None else tot_S + mS
        tot_G = mG if tot_G is None else tot_G + mG
        tot_X = mX if tot_X is None else tot_X + mX
    assert_rel(xp.xpcs_ring_means_from_moments(tot_S, 1.0 / cfg.N).cpu().numpy(), full["S_rings"].cpu().numpy(),
               1e-12, "block-summed S rings")
    assert_rel(xp.xpcs_ring_means_from_moments(tot_G).cpu().numpy(), full["g2_rings"].cpu().numpy(), 1e-12,
               "block-summed g2 rings")
    assert_rel(xp.xsvs_contrast_from_moments(tot_X, cfg.T, wl.windows).cpu().numpy(), full["beta"].cpu().numpy(),
               1e-12, "block-summed beta")
    P.close()
