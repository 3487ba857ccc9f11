"""CUDA-graph capture of one pipeline step (Pipeline.capture / capture_host): a replay recomputes every output of
the step from the current contents of the input buffers and gives the same bits as the eager calls (same kernels,
same plans, same fixed-order reductions).  Covers the integer engine (uniform f), the species path (two kinds: host
tables cached on the device, so the capture holds no pageable copy) and the end-to-end host path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402
from paper_2204_13241_b200 import pipeline  # noqa: E402

DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    xp.load()
    yield
    xp.release()


def _cfg(two_species):
    base = xi.CONFIGS["c3" if two_species else "c2"]
    return xi.scaled(base, N=3000, T=24, n_plane=96, lags=(1, 2, 3, 5), windows=(1, 2, 4), n_bins=8)


def _snap(out):
    return {k: v.detach().cpu().clone() for k, v in out.items()}


def _same(a, b):
    assert a.keys() == b.keys()
    for k in a:
        x, y = a[k].numpy(), b[k].numpy()
        assert np.array_equal(x, y, equal_nan=True), k


@pytest.mark.parametrize("two_species", [False, True])
def test_graph_replay_matches_eager(two_species):
    cfg = _cfg(two_species)
    wl = pipeline.workload_from_config(cfg, device=DEV)
    P = pipeline.Pipeline(wl, device=DEV)
    pos = xi.positions(cfg)
    f = torch.from_numpy(xi.form_factors(cfg)).to(DEV) if cfg.two_species else None
    pos_d = torch.from_numpy(pos).to(DEV)
    g, out_g = P.capture(pos_d, f)
    assert P.capture_launches > 0
    # new trajectory into the same buffer: the replay must see it
    pos2 = xi.positions(xi.scaled(cfg, seed=cfg.seed + 17))
    pos_d.copy_(torch.from_numpy(pos2))
    g.replay()
    torch.cuda.synchronize()
    got = _snap(out_g)
    eager = _snap(P.run(pos_d, f))
    torch.cuda.synchronize()
    _same(got, eager)
    # and the replayed step is not the stale one
    pos_d.copy_(torch.from_numpy(pos))
    g.replay()
    torch.cuda.synchronize()
    assert not np.array_equal(out_g["I"].cpu().numpy(), got["I"].numpy())
    P.close()


def test_graph_end_to_end_host_path():
    cfg = _cfg(False)
    wl = pipeline.workload_from_config(cfg, device=DEV)
    P = pipeline.Pipeline(wl, device=DEV)
    pos = xi.positions(cfg)
    P.alloc_host_io(pos, None, batches=3)
    P.run_host()
    torch.cuda.synchronize()
    ref = {k: v.clone() for k, v in P.h_out.items()}
    g, _ = P.capture_host()
    for v in P.h_out.values():
        v.zero_()
    g.replay()
    torch.cuda.synchronize()
    _same({k: v for k, v in P.h_out.items()}, ref)
    P.close()


def test_host_step_explicit_q_matches_device_run():
    """xpcs_step_host with an explicit q list (an Ewald detector, the generic SFU kernel): the host-buffer step equals
    the device-buffer pipeline within the per-pixel gate (frame batches may chunk the atoms differently)."""
    from _gates import assert_pixels
    cfg = xi.scaled(xi.CONFIGS["c4"], N=2000, T=6, detector=48)
    wl = pipeline.workload_from_config(cfg, device=DEV)
    P = pipeline.Pipeline(wl, device=DEV)
    pos = xi.positions(cfg)
    dev_out = P.run(torch.from_numpy(pos).to(DEV), None)
    I_dev = dev_out["I"].cpu().numpy().copy()
    S_dev = dev_out["S_rings"].cpu().numpy().copy()
    P.alloc_host_io(pos, None, batches=3)
    h = P.run_host()
    torch.cuda.synchronize()
    assert_pixels(h["I"].numpy(), I_dev, cfg.N, "host step, explicit q")
    np.testing.assert_allclose(h["S_rings"].numpy(), S_dev, rtol=1e-5, equal_nan=True)
    P.close()


def test_host_step_edge_cases():
    """xpcs_step_host: pageable (unpinned) host buffers, more batches than frames, no lags / windows, NULL outputs,
    rings that are empty (NaN), and f64 positions (FP64 path) -- each against the device-buffer calls."""
    cfg = xi.scaled(xi.CONFIGS["c2"], N=1500, T=3, n_plane=64, lags=(), windows=(), n_bins=40)
    pos = xi.positions(cfg)
    g = xp.lattice_plane(cfg.L, 64)
    bins = xp.xpcs_lattice_bins(g, 40, 2, DEV)          # rings of width 2 up to r < 80: r <= 45 fills rings 0..22
    I_dev = xp.xpcs_intensity_grid(torch.from_numpy(pos).to(DEV), None, g).cpu().numpy()
    S_dev = xp.xpcs_structure_factor_shells(torch.from_numpy(I_dev).to(DEV), None, cfg.N, bins, 40).cpu().numpy()
    hp = torch.from_numpy(pos.copy())                   # pageable
    hI = torch.empty((cfg.T, 64 * 64), dtype=torch.float32)
    hS = torch.empty((cfg.T, 40), dtype=torch.float64)
    xp.xpcs_step_host(hp, None, g, bins, 40, I_out=hI, S_rings=hS, batches=7)
    torch.cuda.synchronize()
    np.testing.assert_allclose(hI.numpy(), I_dev, rtol=2e-5, atol=2e-5 * np.abs(I_dev).max())
    np.testing.assert_allclose(hS.numpy(), S_dev, rtol=1e-5, equal_nan=True)
    assert np.isnan(hS.numpy()[:, 23:]).all()           # empty rings
    # nothing requested but I: NULL reductions outputs are skipped
    hI2 = torch.zeros_like(hI)
    xp.xpcs_step_host(hp, None, g, bins, 40, I_out=hI2, batches=1)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hI2.numpy(), xp.xpcs_intensity_grid(torch.from_numpy(pos).to(DEV), None, g).cpu().numpy())
    # FP64 positions -> FP64 kernels, FP64 output
    p64 = torch.from_numpy(pos.astype(np.float64))
    hI64 = torch.empty((cfg.T, 64 * 64), dtype=torch.float64)
    xp.xpcs_step_host(p64, None, g, bins, 40, I_out=hI64, batches=2)
    torch.cuda.synchronize()
    ref64 = xp.xpcs_intensity_grid(p64.to(DEV), None, g).cpu().numpy()
    np.testing.assert_allclose(hI64.numpy(), ref64, rtol=1e-12, atol=1e-9)


def test_moments_empty_rings_are_nan():
    cfg = xi.scaled(xi.CONFIGS["c2"], N=800, T=8, n_plane=32, lags=(1,), windows=(1, 2), n_bins=24)
    g = xp.lattice_plane(cfg.L, 32)
    bins = xp.xpcs_lattice_bins(g, 24, 1, DEV)           # r <= 22.6: rings 23 empty
    I = xp.xpcs_intensity_grid(torch.from_numpy(xi.positions(cfg)).to(DEV), None, g)
    m = xp.xpcs_ring_moments(I, bins, 24)
    means = xp.xpcs_ring_means_from_moments(m, 1.0).cpu().numpy()
    assert np.isnan(means[:, 23:]).all() and np.isfinite(means[:, 1:15]).all()
    mx = xp.xsvs_moments(I, bins, 24, [1, 2])
    beta = xp.xsvs_contrast_from_moments(mx, cfg.T, [1, 2]).cpu().numpy()
    ref = xp.xsvs_contrast(I, bins, 24, [1, 2]).cpu().numpy()
    assert np.array_equal(np.isnan(beta), np.isnan(ref))
    ok = ~np.isnan(ref)
    np.testing.assert_allclose(beta[ok], ref[ok], rtol=1e-12)


def test_graph_survives_scratch_growth_and_stream_reuse():
    """a captured graph holds raw scratch pointers.  After the capture, a larger eager call on the SAME
    stream and workspace grows the same scratch slots: the buffers the graph uses must be retired (kept until
    xpcs_release), not freed, so replaying the graph still gives the eager result bit for bit.  A pipeline with its
    own workspace on a (possibly recycled) stream must not disturb it either."""
    cfg = _cfg(False)
    pos = torch.from_numpy(xi.positions(cfg)).to(DEV)
    grid = xp.lattice_plane(cfg.L, 96)
    ws = xp.new_workspace()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with xp.workspace(ws), torch.cuda.stream(s):
        ref = xp.xpcs_intensity_grid(pos, None, grid, stream=s).clone()       # sizes the scratch (eager)
        g2ref = xp.xpcs_g2(ref, [1, 2, 3], stream=s).clone()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with xp.workspace(ws), torch.cuda.graph(g, stream=s):
        out = xp.xpcs_intensity_grid(pos, None, grid, stream=s)
        g2 = xp.xpcs_g2(out, [1, 2, 3], stream=s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref) and torch.equal(g2, g2ref)
    big = xi.scaled(cfg, N=9000, T=60)
    pos_big = torch.from_numpy(xi.positions(big)).to(DEV)
    with xp.workspace(ws), torch.cuda.stream(s):                            # same key: the slots grow
        Ib = xp.xpcs_intensity_grid(pos_big, None, xp.lattice_plane(big.L, 200), stream=s)
        xp.xpcs_g2(Ib, list(range(1, 40)), stream=s)
    Q = pipeline.Pipeline(pipeline.workload_from_config(big))
    Q.run(pos_big, None)
    torch.cuda.synchronize()
    out.zero_()
    g2.zero_()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref) and torch.equal(g2, g2ref)
    Q.close()
