"""The q-sharded single-trajectory mode: a detector split into slabs of rows, each slab's I, g2 and
additive ring / XSVS moments computed separately, the moments summed (the all-reduce), the ring results formed from
the sums.  On one GPU the ranks run one after another (no rank waits on another) and the sum stands in for the
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


@pytest.mark.parametrize("world", [2, 3])
def test_qslab_split_equals_full_detector(world):
    cfg = _cfg()
    pos = torch.from_numpy(xi.positions(cfg)).to(DEV)
    wl = pipeline.workload_from_config(cfg, device=DEV)
    P = pipeline.Pipeline(wl, device=DEV)
    full = {k: v.clone() for k, v in P.run(pos, None).items() if torch.is_tensor(v)}
    ranks = [pipeline.QSlabPipeline(wl, r, world, device=DEV, allreduce=lambda t: None) for r in range(world)]
    total = None
    for Q in ranks:
        m = Q.local(pos, None).clone()
        total = m if total is None else total + m
    torch.cuda.synchronize()
    res = ranks[0].finish(None, moments=total)
    # each slab's I comes from its own engine launch (its own tiling and atom chunking), so the ring results agree
    # with the full detector's within the ring gate (1e-4, north_star), not bitwise; the decomposition itself is
    # pinned exactly below on identical input
    for key in ("S_rings", "g2_rings", "beta"):
        assert_rel(res[key].cpu().numpy(), full[key].cpu().numpy(), 1e-4, f"q-slab {key} (world {world})")
    # exact decomposition: the full-detector I split into the same slabs, moments summed over slabs == full moments
    n = cfg.n_plane
    tot_S = tot_G = tot_X = None
    for Q in ranks:
        lo, hi = Q.row0 * n, (Q.row0 + Q.grid.n_h) * n
        I_s = full["I"][:, lo:hi].contiguous()
        g2_s = full["g2"][:, lo:hi].contiguous()
        b_s = P.bins[lo:hi].contiguous()
        mS = xp.xpcs_ring_moments(I_s, b_s, wl.n_bins)
        mG = xp.xpcs_ring_moments(g2_s, b_s, wl.n_bins)
        mX = xp.xsvs_moments(I_s, b_s, wl.n_bins, wl.windows)
        tot_S = mS if tot_S is None else tot_S + mS
        tot_G = mG if tot_G is None else tot_G + mG
        tot_X = mX if tot_X is None else tot_X + mX
    assert_rel(xp.xpcs_ring_means_from_moments(tot_S, 1.0 / cfg.N).cpu().numpy(), full["S_rings"].cpu().numpy(),
               1e-12, "slab-summed S rings")
    assert_rel(xp.xpcs_ring_means_from_moments(tot_G).cpu().numpy(), full["g2_rings"].cpu().numpy(), 1e-12,
               "slab-summed g2 rings")
    assert_rel(xp.xsvs_contrast_from_moments(tot_X, cfg.T, wl.windows).cpu().numpy(), full["beta"].cpu().numpy(),
               1e-12, "slab-summed beta")
    I_full = full["I"].cpu().numpy().reshape(cfg.T, cfg.n_plane, cfg.n_plane)
    g2_full = full["g2"].cpu().numpy().reshape(len(cfg.lags), cfg.n_plane, cfg.n_plane)
    rows = 0
    for Q in ranks:
        n_h = Q.grid.n_h
        Ir = Q.I.cpu().numpy().reshape(cfg.T, n_h, cfg.n_plane)
        assert_pixels(Ir, I_full[:, Q.row0:Q.row0 + n_h], cfg.N, f"slab {Q.rank} I")
        g2r = Q.g2.cpu().numpy().reshape(len(cfg.lags), n_h, cfg.n_plane)
        np.testing.assert_allclose(g2r, g2_full[:, Q.row0:Q.row0 + n_h], rtol=1e-3)
        rows += n_h
        Q.close()
    assert rows == cfg.n_plane
    P.close()
