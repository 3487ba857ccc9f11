"""Full-size configs (BASELINE.json configs[1..4]) in the launch configuration bench.py times
(paper_2204_13241_b200.pipeline), checked three ways:

  1. sampled parity: I(q,t) of seeded pixels (plus the centre / axis / corner pixels) and frames against the FP64
     oracle, gate |dI| <= 1e-3 N + 1e-5 I (R11);
  2. reduction parity on the GPU's own I: g2 (per pixel on the sampled pixels), ring-averaged S(q,t) and g2, XSVS
     beta against the oracle's reductions (1e-10 relative, R12);
  3. the statistical pins of SURVEY 8(c) applied to the *full* GPU outputs (the only end-to-end check at full scale
     that the CPU oracle cannot afford): the Siegert + diffusion law of the g2 numerator (Eq. 24-25), mean S = 1 for
     the ideal gas, the discrete Eq.(28) XSVS law, and the off-lattice expectation with the box shape transform.
  4. END-TO-END ring-level acceptance (north_star: <= 1e-4 relative on the azimuthally averaged S(q) and on g2,
     DESIGN.md R12; XSVS beta at the same 1e-4): the oracle computes I itself on whole rings (the
     SURVEY 8(d) parity subsets) and its S_b(t), ring g2 and beta are compared with the GPU pipeline's outputs --
     c2 full plane x frames {0, 49, 99} (S_b) and shells 0-3 x 100 frames (ring g2), c3 shell 0 x 1000 frames
     (ring g2, S_b), c5 shells {0, 1} x 200 frames (beta); every oracle pixel-frame also passes the per-pixel gate.
Plus the perfect-crystal Bragg variant of every config at its own N (I = N^2 at peaks within the gate, ~0 elsewhere).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
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


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _run(cfg, repeat=False):
    """Generate the config's inputs, run the whole pipeline, return (outputs as numpy, positions, f, q, bins).
    repeat: run the step a second time on the same inputs and require bit-identical outputs (the deterministic
    engines, folds and reductions at full size: many frame batches on two streams, every reduction)."""
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg)
    wl = pipeline.workload_from_config(cfg)
    P = pipeline.Pipeline(wl)
    pos_d = _t(pos)
    f_d = _t(f) if cfg.two_species else None
    out = P.run(pos_d, f_d)
    torch.cuda.synchronize()
    if repeat:
        first = {k: v.clone() for k, v in out.items()}
        out = P.run(pos_d, f_d)
        torch.cuda.synchronize()
        for k, v in out.items():
            a, b = v, first[k]
            same = (a == b) | (torch.isnan(a) & torch.isnan(b))
            assert bool(same.all()), f"{cfg.name}: {k} differs between two runs of the same step"
        del first
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["bins"] = P.bins.cpu().numpy()
    del pos_d
    if cfg.n_plane:
        q = oracle.lattice_q(cfg.L, **oracle.plane_grid(cfg.n_plane))
        n = cfg.n_plane
        c = (n // 2) * n + n // 2
        include = [c, c + 1, c - 1, c + n, c - n, 0, n - 1, n * n - 1, c + n // 4]
    else:
        q = wl.q.cpu().numpy().astype(np.float64)
        d = cfg.detector
        c = (d // 2) * d + d // 2
        include = [c, c - d - 1, 0, d - 1, d * d - 1] + [c + k for k in range(1, 40)] + [c + k * d for k in range(1, 20)]
    return res, pos, f, q, include


def _pixel_parity(cfg, res, pos, f, q, include, frames, n_pix, seed):
    pix = xi.pixel_subset(q.shape[0], n_pix, seed, include)
    ref = oracle.intensity(pos[frames], f.astype(np.float64) if cfg.two_species else None, q[pix], cfg.L)
    assert_pixels(res["I"][frames][:, pix], ref, cfg.N, cfg.name)
    return pix


def _reductions(cfg, res, pix):
    I, bins = res["I"], res["bins"]
    f = xi.form_factors(cfg) if cfg.two_species else None
    assert_rel(res["S_rings"], oracle.structure_factor_shells(I, f, cfg.N, bins, cfg.n_bins), 1e-10, "S rings")
    if cfg.lags:
        g2 = res["g2"]
        # per-pixel g2 on the sampled pixels (fp32 output of an FP64 accumulation)
        assert_rel(g2[:, pix], oracle.g2(I[:, pix], cfg.lags).astype(np.float32), 1e-6, "g2 per pixel")
        assert_rel(res["g2_rings"], oracle.shell_mean(g2, bins, cfg.n_bins), 1e-10, "g2 rings")
    if cfg.windows:
        assert_rel(res["beta"], oracle.xsvs_beta(I, bins, cfg.n_bins, cfg.windows), 1e-10, "beta")


def _oracle_I(cfg, pos, f, q_sel, frames=None, chunk=100):
    """Oracle I(q, t) at the selected q for the given frames (all by default), in frame chunks (bounded memory)."""
    frames = np.arange(pos.shape[0]) if frames is None else np.asarray(frames)
    ff = f.astype(np.float64) if cfg.two_species else None
    out = [oracle.intensity(pos[frames[i:i + chunk]], ff, q_sel, cfg.L) for i in range(0, len(frames), chunk)]
    return np.concatenate(out, 0)


def _shell_pixels(bins, shells):
    return np.flatnonzero(np.isin(bins, list(shells)))


def _ring_mean(values, bins_sel, shells):
    """Mean over each shell's pixels (values [rows][n_sel], bins_sel [n_sel]) -> [rows][len(shells)]."""
    return np.stack([values[:, bins_sel == b].mean(1) for b in shells], 1)


def _species(cfg):
    f = xi.form_factors(cfg).astype(np.float64)
    return f.sum(), (f ** 2).sum(), (f ** 4).sum()


def _g2_numerator_pin(cfg, res, q, lags, shells):
    """SURVEY 8(c) 'g2 (Brownian)': per shell, mean over pixels of num(tau)/S2^2 - 1 vs beta0 mean phi^2,
    phi = exp(-D q^2 tau dt) (Eq. 24 + 25, exact as a ratio of expectations, A.7); 5 sigma with sigma = the
    across-pixel std / sqrt(n_pix / 2) (I(q) = I(-q) pairs)."""
    I, bins = res["I"].astype(np.float64), res["bins"]
    _, S2, S4 = _species(cfg)
    beta0 = 1 - S4 / S2 ** 2
    q2 = (q ** 2).sum(1)
    den = I.mean(0) ** 2
    li_of = {tau: i for i, tau in enumerate(cfg.lags)}
    worst = 0.0
    for tau in lags:
        num = res["g2"][li_of[tau]].astype(np.float64) * den
        for b in shells:
            sel = bins == b
            v = num[sel] / S2 ** 2 - 1.0
            pred = beta0 * np.mean(np.exp(-2 * cfg.D * q2[sel] * tau * cfg.dt))
            z = abs(v.mean() - pred) / (v.std() / np.sqrt(sel.sum() / 2))
            worst = max(worst, z)
            assert z < 5.0, (cfg.name, tau, b, v.mean(), pred, z)
    # denominator: <I>/S2 = 1 over the whole disk (ideal gas, lattice q != 0)
    m = I[:, bins >= 0].mean() / S2
    assert abs(m - 1) < 0.01, m
    return worst


# ------------------------------------------------------------------------------------------------ configs
def test_config2_full_size():
    cfg = xi.CONFIGS["c2"]
    res, pos, f, q, inc = _run(cfg, repeat=True)
    bins = res["bins"]
    # full plane at frames {0, 49, 99}: per-pixel gate on every pixel and S_b(t) end to end (SURVEY 8(d) subset)
    frames = [0, 49, 99]
    Io = _oracle_I(cfg, pos, f, q, frames)
    assert_pixels(res["I"][frames], Io, cfg.N, "c2 full plane")
    S_o = oracle.structure_factor_shells(Io, None, cfg.N, bins, cfg.n_bins)
    assert_rel(res["S_rings"][frames], S_o, 1e-4, "c2 S_b(t) vs oracle I (end to end)")
    # shells 0-3 x all 100 frames: per-pixel gate and the ring-averaged g2 end to end
    shells = range(4)
    pix = _shell_pixels(bins, shells)
    Ir = _oracle_I(cfg, pos, f, q[pix])
    assert_pixels(res["I"][:, pix], Ir, cfg.N, "c2 shells 0-3 x 100 frames")
    g2_ring_o = _ring_mean(oracle.g2(Ir, cfg.lags), bins[pix], shells)
    assert_rel(res["g2_rings"][:, :4], g2_ring_o, 1e-4, "c2 ring g2 vs oracle I (end to end)")
    pix_s = _pixel_parity(cfg, res, pos, f, q, inc, [0, 49, 99], 384, 2)
    _reductions(cfg, res, pix_s)
    _g2_numerator_pin(cfg, res, q, cfg.lags, range(cfg.n_bins))
    assert abs(np.nanmean(res["S_rings"][:, 4:]) - 1) < 0.01


@pytest.mark.slow
def test_config3_full_size():
    """1000 frames x 262144 atoms x 512^2 pixels (6.9e13 pairs), two species, g2 for tau = 1..200.  End to end: the
    oracle's I on shell 0 (~200 pixels) x all 1000 frames (5e10 pairs, ~2 min on 16 cores): per-pixel gate on 2e5
    pixel-frames, ring g2 and S_b(t) of shell 0 within 1e-4."""
    cfg = xi.CONFIGS["c3"]
    res, pos, f, q, inc = _run(cfg, repeat=True)
    bins = res["bins"]
    pix0 = _shell_pixels(bins, [0])
    Ir = _oracle_I(cfg, pos, f, q[pix0])
    assert Ir.size >= 1e5
    assert_pixels(res["I"][:, pix0], Ir, cfg.N, "c3 shell 0 x 1000 frames")
    assert_rel(res["g2_rings"][:, :1], _ring_mean(oracle.g2(Ir, cfg.lags), bins[pix0], [0]), 1e-4,
               "c3 ring g2 (shell 0) vs oracle I (end to end)")
    _, S2, _ = _species(cfg)
    assert_rel(res["S_rings"][:, :1], _ring_mean(Ir, bins[pix0], [0]) / S2, 1e-4, "c3 S_b(t) (shell 0) end to end")
    pix = _pixel_parity(cfg, res, pos, f, q, inc, [0, 999], 64, 3)
    del pos
    _reductions(cfg, res, pix)
    _g2_numerator_pin(cfg, res, q, [1, 2, 4, 8, 16, 32, 64, 128, 200], range(cfg.n_bins))
    assert abs(np.nanmean(res["S_rings"][:, 4:]) - 1) < 0.005


@pytest.mark.slow
def test_config4_full_size():
    """Ewald detector (1024^2 fp32 q), 2^20 atoms, 20 independent frames: sampled parity, ring parity, and the
    off-lattice expectation E[I(q)] = S2 + (S1^2 - S2) prod_c sinc^2(q_c L / 2) ring by ring (5 sigma; the
    speckle is oversampled ~1.4x per axis, so n_eff = pixels x frames / 4)."""
    cfg = xi.CONFIGS["c4"]
    res, pos, f, q, inc = _run(cfg)
    pix = _pixel_parity(cfg, res, pos, f, q, inc, list(range(20)), 512, 4)     # 512 pixels x 20 frames = 1e4
    del pos
    _reductions(cfg, res, pix)
    S1, S2, _ = _species(cfg)
    sinc2 = np.prod(np.sinc(q * cfg.L / 2 / np.pi) ** 2, axis=1)
    E = S2 + (S1 ** 2 - S2) * sinc2
    r = res["I"].astype(np.float64) / E[None, :]
    bins = res["bins"]
    for b in range(1, cfg.n_bins):
        sel = bins == b
        x = r[:, sel]
        n_eff = x.size / 4
        z = abs(x.mean() - 1) / (x.std() / np.sqrt(n_eff))
        assert z < 5, (b, x.mean(), z)


@pytest.mark.slow
def test_config5_full_size():
    """XSVS workload: 200 frames x 524288 atoms x 512^2 (2.7e13 pairs).  Parity, beta reduction parity, and the
    discrete Eq.(28) law beta_W = beta0 mean[(W + 2 S_W(x)) / W^2] (1 - 2/n_eff), x = exp(-2 D q^2 dt), on the
    rings with 2 D q^2 dt T >= 20 for W <= 64 (SURVEY 8(c) XSVS pin, A.11)."""
    cfg = xi.CONFIGS["c5"]
    res, pos, f, q, inc = _run(cfg, repeat=True)
    bins = res["bins"]
    # end to end: the oracle's I on shells {0, 1} (~800 pixels) x 200 frames (8e10 pairs, ~3 min on 16 cores):
    # per-pixel gate on 1.6e5 pixel-frames and beta of both shells for every window within 1e-4
    shells = [0, 1]
    pixr = _shell_pixels(bins, shells)
    Ir = _oracle_I(cfg, pos, f, q[pixr])
    assert_pixels(res["I"][:, pixr], Ir, cfg.N, "c5 shells 0-1 x 200 frames")
    beta_o = oracle.xsvs_beta(Ir, bins[pixr], cfg.n_bins, cfg.windows)[:, :2]
    assert_rel(res["beta"][:, :2], beta_o, 1e-4, "c5 beta (shells 0, 1) vs oracle I (end to end)")
    pix = _pixel_parity(cfg, res, pos, f, q, inc, [0, 199], 64, 5)
    del pos
    _reductions(cfg, res, pix)
    _, S2, S4 = _species(cfg)
    beta0 = 1 - S4 / S2 ** 2
    bins = res["bins"]
    q2 = (q ** 2).sum(1)
    checked = 0
    for b in range(cfg.n_bins):
        sel = bins == b
        if np.min(2 * cfg.D * q2[sel] * cfg.dt * cfg.T) < 20:
            continue
        x = np.exp(-2 * cfg.D * q2[sel] * cfg.dt)
        n_eff = sel.sum() / 2
        for wi, W in enumerate(cfg.windows):
            if W > 64:
                continue
            SW = x * (W * (1 - x) - 1 + x ** W) / (1 - x) ** 2
            pred = beta0 * np.mean((W + 2 * SW) / W ** 2) * (1 - 2 / n_eff)
            assert abs(res["beta"][wi, b] - pred) < 0.03 * pred, (b, W, res["beta"][wi, b], pred)
            checked += 1
    assert checked >= 20 * 7


# ------------------------------------------------------------------------------------------------ Bragg variants
@pytest.mark.parametrize("kind,n_cells,cfg_name,n", [("sc", 64, "c3", 512), ("bcc", 64, "c5", 512),
                                                     ("fcc", 64, "c4", 1024)])
def test_bragg_variant_at_config_size(kind, n_cells, cfg_name, n):
    """SURVEY 8(c) perfect-lattice pin at each config's own N and L: SC 64^3 (c3), BCC 2 x 64^3 (c5),
    FCC 4 x 64^3 (c4, on a 1024^2 lattice plane).  I = N^2 at the crystal's reciprocal lattice, 0 elsewhere."""
    cfg = xi.CONFIGS[cfg_name]
    pos = xi.crystal(kind, n_cells, cfg.L, "f32")
    N = pos.shape[0]
    assert N == cfg.N
    g = xp.lattice_plane(cfg.L, n)
    I = xp.xpcs_intensity_grid(_t(pos), None, g).cpu().numpy().reshape(n, n).astype(np.float64)
    h = np.arange(-n // 2, n // 2)
    H, K = np.meshgrid(h, h, indexing="ij")
    period = 2 * n_cells if kind == "fcc" else n_cells
    peak = (H % period == 0) & (K % period == 0)
    if kind == "bcc":
        peak &= ((H // period + K // period) % 2 == 0)
    qp = (2 * np.pi / cfg.L) * np.stack([H[peak], K[peak], np.zeros(peak.sum())], -1)
    assert_pixels(I[peak], oracle.intensity(pos.astype(np.float64), None, qp, cfg.L)[0], N, f"{kind} Bragg peaks")
    assert np.max(I[~peak]) <= 1e-3 * N
