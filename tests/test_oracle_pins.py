"""Pins of the FP64 oracle against what the paper and the mathematics fix (CPU only).

Each test names the passage it checks.  None of them re-types the oracle's formula: they use the
O(N^2) pair sum (Eq. 2), closed forms (single atoms, forward limit, Bragg peaks of perfect crystals,
the ideal-gas expectation with the box shape transform, the Brownian g2 and XSVS laws), invariants
(inversion, PBC shift, permutation) and numbers printed in the paper (tests/golden/).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import xpcs_inputs as xi

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def _hkl_q(L, hkl):
    return (2 * np.pi / L) * np.asarray(hkl, dtype=np.float64)


# ------------------------------------------------------------------ worked examples (golden)
@pytest.mark.parametrize("case", ["single_atom_origin", "single_atom_half_box"])
def test_golden_amplitude_sign(case):
    g = _gold("spec_examples.json")[case]
    A = oracle.amplitude(np.array(g["pos"]), np.array(g["f"]), _hkl_q(g["L"], g["hkl"]), g["L"])
    np.testing.assert_allclose(A.real, g["amplitude_re"], atol=1e-12)
    np.testing.assert_allclose(A.imag, g["amplitude_im"], atol=1e-12)


@pytest.mark.parametrize("case", ["one_atom_f", "forward"])
def test_golden_intensity(case):
    g = _gold("spec_examples.json")[case]
    I = oracle.intensity(np.array(g["pos"]), np.array(g["f"]), _hkl_q(g["L"], g["hkl"]), g["L"])[0]
    np.testing.assert_allclose(I, g["intensity"], rtol=1e-12)


def test_paper_q_point_is_a_lattice_vector():
    """PAPER.md:414 prints q = (0, 1.481, -1.164) A^-1 for the L = 59.19 A box;
    Algorithm 1 only allows reciprocal-lattice q: lattice_q must reproduce the printed
    point as (2 pi / L)(0, 14, -11) to the printed 3 decimals."""
    g = _gold("paper_parameters.json")
    L = g["box_L_angstrom"]["value"]
    hkl = g["q_point_fig3"]["hkl"]
    q = oracle.lattice_q(L, h0=hkl[1], n_h=1, k0=hkl[2], n_k=1, m0=(hkl[0], 0, 0), ma=(0, 1, 0), mb=(0, 0, 1))[0]
    np.testing.assert_allclose(q, g["q_point_fig3"]["value"], atol=6e-3)


def test_two_atoms_closed_form():
    """Eq.(2) with N = 2: I = f1^2 + f2^2 + 2 f1 f2 cos(q . (r1 - r2))."""
    L = 9.0
    pos = np.array([[1.1, 2.2, 3.3], [7.7, 0.4, 5.9]])
    f = np.array([1.5, 0.7])
    q = oracle.lattice_q(L, -5, 11, -5, 11, m0=(2, 0, 0), ma=(0, 1, 0), mb=(0, 0, 1))
    d = pos[0] - pos[1]
    expect = f[0] ** 2 + f[1] ** 2 + 2 * f[0] * f[1] * np.cos(q @ d)
    np.testing.assert_allclose(oracle.intensity(pos, f, q, L)[0], expect, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ brute force
@pytest.mark.parametrize("N,two", [(8, False), (50, True), (100, True)])
def test_direct_equals_pair_sum(N, two):
    """Single sum Eq.(7)+(8) == O(N^2) pair sum Eq.(2) to 1e-10 relative on all lattice q, |q| <= 3
    (SPEC.md:596 acceptance #1; PAPER.md:280-284 derivation)."""
    L = 6.0
    rng = np.random.default_rng(N)
    pos = rng.uniform(0, L, (N, 3))
    f = np.where(np.arange(N) % 2 == 1, 2.0, 1.0) if two else np.ones(N)
    q = np.concatenate([oracle.lattice_q(L, -3, 7, -3, 7, m0=(l, 0, 0), ma=(0, 1, 0), mb=(0, 0, 1))
                        for l in range(-3, 4)])
    q = q[np.linalg.norm(q, axis=1) <= 3.0]
    a = oracle.intensity(pos, f, q, L)[0]
    b = oracle.pair_sum_intensity(pos, f, q, L)
    scale = max(1.0, float(np.max(np.abs(b))))
    assert np.max(np.abs(a - b)) <= 1e-10 * scale


def test_forward_limit_and_inversion():
    """I(0) = (sum f)^2; I(q) = I(-q) (conjugate symmetry of Eq. 7)."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=600, T=1)
    pos = xi.positions(cfg)[0]
    f = xi.form_factors(cfg).astype(np.float64)
    n = 16
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(n))
    I = oracle.intensity(pos, f, q, cfg.L)[0].reshape(n, n)
    assert abs(I[n // 2, n // 2] - f.sum() ** 2) <= 1e-12 * f.sum() ** 2
    inner = I[1:, 1:]                       # h, k in [-n/2+1, n/2-1] has its mirror inside the grid
    np.testing.assert_allclose(inner, inner[::-1, ::-1], rtol=1e-12, atol=1e-9)


def test_pbc_shift_and_permutation_invariance():
    """Lattice q: any periodic image gives the same I -> a rigid shift of all atoms,
    re-wrapped, leaves I unchanged; so does relabelling atoms."""
    L = 8.0
    rng = np.random.default_rng(7)
    pos = rng.uniform(0, L, (300, 3))
    f = rng.uniform(0.5, 2.0, 300)
    q = oracle.lattice_q(L, -6, 12, -6, 12, m0=(3, 0, 0), ma=(0, 1, 0), mb=(0, 0, 1))
    I0 = oracle.intensity(pos, f, q, L)[0]
    shifted = pos + np.array([3.7, -12.25, 101.5])      # the oracle wraps into [0, L)
    I1 = oracle.intensity(shifted, f, q, L)[0]
    np.testing.assert_allclose(I1, I0, rtol=1e-9, atol=1e-9 * 300)
    perm = rng.permutation(300)
    I2 = oracle.intensity(pos[perm], f[perm], q, L)[0]
    np.testing.assert_allclose(I2, I0, rtol=1e-11, atol=1e-10)


# ------------------------------------------------------------------ Bragg peaks (closed form)
@pytest.mark.parametrize("kind,n_cells,L,n,period,rule", [
    ("sc", 10, 10.0, 64, 10, "all"),           # config 1's own size: SC 10^3, L = 10
    ("fcc", 6, 12.0, 64, 12, "all"),           # FCC: h, k in 2 n_c Z (l = 0)
    ("bcc", 8, 20.0, 64, 8, "even"),           # BCC: H + K even, H = h / n_c
])
def test_bragg_peaks(kind, n_cells, L, n, period, rule):
    """Perfect crystal, f = 1: geometric lattice sums give I = N^2 on the reciprocal lattice of the
    crystal and 0 elsewhere (Eq. 7 as a lattice sum; PAPER.md:285-288 reciprocal lattice)."""
    pos = xi.crystal(kind, n_cells, L)
    N = pos.shape[0]
    q = oracle.lattice_q(L, **oracle.plane_grid(n))
    I = oracle.intensity(pos, None, q, L)[0].reshape(n, n)
    h = np.arange(-n // 2, n // 2)
    H, K = np.meshgrid(h, h, indexing="ij")
    peak = (H % period == 0) & (K % period == 0)
    if rule == "even":
        peak &= ((H // period + K // period) % 2 == 0)
    assert peak.sum() > 4
    np.testing.assert_allclose(I[peak], float(N) ** 2, rtol=1e-12)
    assert np.max(I[~peak]) < 1e-6 * N


# ------------------------------------------------------------------ ideal-gas statistics
def test_random_positions_plane_mean():
    """Uniform random positions, lattice q != 0: E[I] = sum f^2 (Eq. 12 with S = 1 for an ideal gas);
    plane mean of I / sum f^2 = 1 +- 5/sqrt(n_q/2) (pairs +-q identical)."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=2000, T=1)
    pos = xi.positions(cfg)[0]
    f = xi.form_factors(cfg).astype(np.float64)
    n = 48
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(n))
    I = oracle.intensity(pos, f, q, cfg.L)[0]
    nz = np.linalg.norm(q, axis=1) > 0
    m = I[nz].mean() / np.sum(f ** 2)
    assert abs(m - 1.0) < 5.0 / np.sqrt(nz.sum() / 2)


def test_random_positions_off_lattice_expectation():
    """Off-lattice q (R3): for iid uniform atoms in [0, L)^3,
    E[I(q)] = S2 + (S1^2 - S2) prod_c sinc^2(q_c L / 2)  (characteristic function of U[0, L)),
    checked at 5 sigma over independent frames, including near-forward q where the box term dominates."""
    N, L, frames = 60, 5.0, 400
    f = np.where(np.arange(N) % 2 == 1, 2.0, 1.0)
    S1, S2 = f.sum(), (f ** 2).sum()
    q = np.array([[0.3, 0.1, -0.2], [0.9, 0.0, 0.0], [1.7, -0.6, 0.4], [0.05, 0.05, 0.05], [2.5, 2.5, -1.0]])
    Is = np.stack([oracle.intensity(xi.uniform_frame(1000 + s, N, L), f, q, L)[0] for s in range(frames)])
    sinc2 = np.prod(np.sinc(q * L / 2 / np.pi) ** 2, axis=1)   # np.sinc(x) = sin(pi x)/(pi x)
    expect = S2 + (S1 ** 2 - S2) * sinc2
    sigma = Is.std(0) / np.sqrt(frames)
    assert np.all(np.abs(Is.mean(0) - expect) < 5 * sigma + 1e-9)


def test_contrast_of_single_snapshot():
    """Fully coherent speckle: beta = 1, precisely beta0 = 1 - S4/S2^2 for N random
    phasors (SPEC 8(c) 'intensity statistics'); XSVS W = 1 on one frame over large rings, 5 sigma."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=1500, T=1)
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg).astype(np.float64)
    n = 64
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(n))
    I = oracle.intensity(pos, f, q, cfg.L)
    bins = oracle.lattice_bins(n, n_bins=4)
    beta = oracle.xsvs_beta(I, bins, 4, [1])[0]
    beta0 = 1 - np.sum(f ** 4) / np.sum(f ** 2) ** 2
    for b in (2, 3):
        n_eff = np.sum(bins == b) / 2
        # exponential intensities: var of the sample contrast ~ 8 / n_eff (4th moment of Exp)
        assert abs(beta[b] - beta0 * (1 - 2 / n_eff)) < 5 * np.sqrt(8.0 / n_eff), (b, beta[b])


# ------------------------------------------------------------------ Brownian dynamics: g2 and XSVS
def _brownian(N, L, T, D, dt, seed):
    cfg = xi.Config("pin", N, L, T, D, dt, 0, True, "f64", (), (), seed=seed)
    return xi.positions(cfg), xi.form_factors(cfg).astype(np.float64)


def test_g2_brownian_numerator_and_denominator():
    """Siegert + diffusion (Eq. 24 + Eq. 25): for independent Brownian particles on
    lattice q != 0, E[I_t I_{t+tau}] = S2^2 + phi^2 (S2^2 - S4), phi = exp(-D q^2 tau dt), i.e.
    g2 - 1 = beta0 exp(-2 D q^2 tau).  The literal Eq.(14) ratio is biased at finite T (R6),
    so the unbiased numerator (per shell, 5 sigma) and the denominator mean I / S2 = 1 are pinned."""
    N, L, T, D, dt = 300, 7.0, 500, 0.05, 1.0
    pos, f = _brownian(N, L, T, D, dt, seed=4242)
    n = 16
    q = oracle.lattice_q(L, **oracle.plane_grid(n))
    I = oracle.intensity(pos, f, q, L)
    S2, S4 = np.sum(f ** 2), np.sum(f ** 4)
    beta0 = 1 - S4 / S2 ** 2
    lags = [1, 2, 4, 8]
    bins = oracle.lattice_bins(n, n_bins=4)
    q2 = (q ** 2).sum(1)
    # numerator = g2 * den  (use oracle.g2 so the function under test is exercised)
    den = (I.mean(0)) ** 2
    G = oracle.g2(I, lags)
    num = G * den[None, :]
    worst = 0.0
    for li, tau in enumerate(lags):
        for b in range(4):
            sel = bins == b
            v = num[li, sel] / S2 ** 2 - 1.0
            pred = beta0 * np.mean(np.exp(-2 * D * q2[sel] * tau * dt))
            sigma = v.std() / np.sqrt(sel.sum() / 2)
            z = abs(v.mean() - pred) / sigma
            worst = max(worst, z)
    assert worst < 5.0, worst
    m = I[:, bins >= 0].mean() / S2
    assert abs(m - 1) < 5 * I[:, bins >= 0].std() / S2 / np.sqrt(T * (bins >= 0).sum() / 2 / 10)


def test_xsvs_brownian_closed_form():
    """XSVS contrast vs exposure (Eq. 28) in discrete form for diffusion:
    beta_W = beta0 mean_q[(W + 2 S_W(x)) / W^2], x = exp(-2 D q^2 dt),
    S_W(x) = x (W (1 - x) - 1 + x^W) / (1 - x)^2; literal estimator on fast rings, 5 sigma of the snapshot spread."""
    N, L, T, D, dt = 400, 12.0, 240, 0.05, 0.1
    pos, f = _brownian(N, L, T, D, dt, seed=777)
    n = 48
    q = oracle.lattice_q(L, **oracle.plane_grid(n))
    I = oracle.intensity(pos, f, q, L)
    nb = 4
    bins = oracle.lattice_bins(n, n_bins=nb)
    windows = [1, 2, 4, 8, 16]
    beta, detail = oracle.xsvs_beta(I, bins, nb, windows, per_window=True)
    S2, S4 = np.sum(f ** 2), np.sum(f ** 4)
    beta0 = 1 - S4 / S2 ** 2
    q2 = (q ** 2).sum(1)
    for b in (2, 3):
        sel = bins == b
        x = np.exp(-2 * D * q2[sel] * dt)
        assert np.min(2 * D * q2[sel] * dt * T) >= 20
        for wi, W in enumerate(windows):
            SW = x * (W * (1 - x) - 1 + x ** W) / (1 - x) ** 2
            pred = beta0 * np.mean((W + 2 * SW) / W ** 2)
            n_eff = sel.sum() / 2
            pred *= (1 - 2 / n_eff)                    # finite-ring bias of the literal estimator
            bs = detail[wi][b]                         # per-snapshot contrasts (S of them)
            sigma = bs.std() / np.sqrt(len(bs)) if len(bs) > 1 else 0.1 * pred
            assert abs(beta[wi, b] - pred) < max(5 * sigma, 0.03 * pred), (b, W, beta[wi, b], pred, sigma)


# ------------------------------------------------------------------ reductions: invariants
def test_g2_invariants():
    """Eq.(14): constant series -> g2 = 1; scale invariance; time reversal symmetry of the
    numerator; zero-mean pixel -> NaN."""
    rng = np.random.default_rng(3)
    I = rng.exponential(1.0, (60, 40))
    I[:, 5] = 3.0
    I[:, 6] = 0.0
    lags = [0, 1, 5, 20]
    G = oracle.g2(I, lags)
    np.testing.assert_allclose(G[:, 5], 1.0, rtol=1e-14)
    assert np.all(np.isnan(G[:, 6]))
    np.testing.assert_allclose(oracle.g2(7.5 * I, lags), G, rtol=1e-13)
    np.testing.assert_allclose(oracle.g2(I[::-1], lags), G, rtol=1e-13)
    # tau = 0 gives beta0 + 1 = <I^2>/<I>^2 (Eq. 19)
    m = I[:, :5].mean(0)
    np.testing.assert_allclose(G[0, :5], (I[:, :5] ** 2).mean(0) / m ** 2, rtol=1e-13)


def test_xsvs_invariants():
    """Eq.(15)/(17): W = 1 on a static series equals the single-frame contrast for every W;
    constant field -> beta = 0; Exp(1) pixels -> 1 +- 5 sigma; empty ring -> NaN."""
    rng = np.random.default_rng(11)
    n_q = 4000
    bins = (np.arange(n_q) % 3).astype(np.int32)
    bins[:10] = -1
    frame = rng.exponential(2.0, n_q)
    frame[bins == 2] = 5.0
    I = np.repeat(frame[None], 16, 0)
    beta = oracle.xsvs_beta(I, bins, 4, [1, 2, 4, 16])
    np.testing.assert_allclose(beta[:, 0], beta[0, 0], rtol=1e-12)
    np.testing.assert_allclose(beta[:, 2], 0.0, atol=1e-14)
    assert np.all(np.isnan(beta[:, 3]))
    m = np.sum(bins == 0)
    assert abs(beta[0, 0] - 1) < 5 * np.sqrt(8.0 / m)


def test_lattice_bins():
    """Rings q - dq/2 <= |q| < q + dq/2: integer bins agree with a float evaluation away
    from bin edges, are symmetric under q -> -q, and exclude q = 0 and the corners."""
    for n in (64, 256):
        b = oracle.lattice_bins(n)
        h = np.arange(-n // 2, n // 2)
        H, K = np.meshgrid(h, h, indexing="ij")
        r = np.sqrt(H ** 2 + K ** 2).ravel()
        w = n / 64
        fb = np.floor(r / w)
        ok = (r > 0) & (r < n / 2)
        assert np.all(b[~ok] == -1)
        assert np.all(b[ok] == fb[ok])
        B = b.reshape(n, n)
        np.testing.assert_array_equal(B[1:, 1:], B[1:, 1:][::-1, ::-1])
        assert b.max() == 31


def test_ewald_geometry():
    """Eq.(1): elastic scattering, |k_f| = |k_i| = 2 pi / lambda, so every detector q
    satisfies |q + k z| = k; the centre of an even detector is 4 half-pixels off the beam; the corner
    of the config-4 detector reaches q_max = 8 pi / sigma (R4)."""
    lam, pitch, npx = xi.EWALD_WAVELENGTH_SIGMA, xi.EWALD_PITCH_RAD, 64
    q = oracle.ewald_q(lam, npx, npx, pitch * 16)
    k = 2 * np.pi / lam
    kf = q + np.array([0, 0, k])
    np.testing.assert_allclose(np.linalg.norm(kf, axis=1), k, rtol=1e-13)
    assert np.all(q[:, 2] <= 0)
    qf = oracle.ewald_q(lam, 1024, 1024, pitch)
    r = np.linalg.norm(qf, axis=1)
    assert abs(r.max() - xi.EWALD_QMAX) / xi.EWALD_QMAX < 2e-3
    c = r.reshape(1024, 1024)[511, 511]
    np.testing.assert_allclose(c, 2 * k * np.sin(np.arccos(np.cos(pitch / 2) ** 2) / 2), rtol=1e-9)


def test_shell_mean_and_structure_factor():
    """Eq.(12)-(13): S = I / sum f^2 ring-averaged; NaNs excluded; empty ring NaN."""
    I = np.array([[1.0, 2.0, 3.0, np.nan, 10.0], [4.0, 4.0, 4.0, 4.0, 4.0]])
    bins = np.array([0, 0, 1, 1, -1], np.int32)
    out = oracle.shell_mean(I, bins, 3)
    np.testing.assert_allclose(out[:, :2], [[1.5, 3.0], [4.0, 4.0]])
    assert np.all(np.isnan(out[:, 2]))
    S = oracle.structure_factor_shells(I, np.array([1.0, 2.0]), 2, bins, 3)
    np.testing.assert_allclose(S[:, :2], out[:, :2] / 5.0)


# ------------------------------------------------------------------ intermediate scattering function (8(f) rank 1)
def test_isf_brownian_and_siegert():
    """Eq.(22)-(25): for independent Brownian particles on lattice q != 0, E[p(t) p*(t+tau)] / S2 =
    exp(-D q^2 tau dt) (real); F(0) = S(q) (Eq. 12 vs Eq. 22); and the Siegert relation Eq.(24),
    g2 - 1 = beta0 |F^|^2, holds for the unbiased g2 numerator (Fig. 4b)."""
    N, L, T, D, dt = 300, 7.0, 500, 0.05, 1.0
    pos, f = _brownian(N, L, T, D, dt, seed=99)
    n = 16
    q = oracle.lattice_q(L, **oracle.plane_grid(n))
    A = oracle.amplitudes(pos, f, q, L)
    S2, S4 = np.sum(f ** 2), np.sum(f ** 4)
    lags = [0, 1, 2, 4, 8]
    F = oracle.isf(A, lags, S2)
    I = oracle.intensity(pos, f, q, L)
    np.testing.assert_allclose(F[0].real, I.mean(0) / S2, rtol=1e-12)     # F(q, 0) = <S(q, t)>_t
    np.testing.assert_allclose(F[0].imag, 0.0, atol=1e-12 * N)
    bins = oracle.lattice_bins(n, n_bins=4)
    q2 = (q ** 2).sum(1)
    beta0 = 1 - S4 / S2 ** 2
    den = I.mean(0) ** 2
    G = oracle.g2(I, lags)
    for li, tau in enumerate(lags[1:], start=1):
        for b in range(4):
            sel = bins == b
            phi = np.exp(-D * q2[sel] * tau * dt)
            for comp, pred in ((F[li, sel].real, phi), (F[li, sel].imag, 0 * phi)):
                z = (comp.mean() - pred.mean()) / (comp.std() / np.sqrt(sel.sum() / 2))
                assert abs(z) < 5, (tau, b, z)
            # Siegert: the unbiased numerator num/S2^2 - 1 vs beta0 |F|^2 with E|F|^2 ~ phi^2 (ring level)
            num = G[li, sel] * den[sel] / S2 ** 2 - 1
            sieg = beta0 * phi ** 2
            z = (num.mean() - sieg.mean()) / (num.std() / np.sqrt(sel.sum() / 2))
            assert abs(z) < 5, (tau, b, z)


# ------------------------------------------------------------------ q-dependent form factors, 3-D q blocks
def _two_species_fq(q, n_species=2):
    """Synthetic Gaussian-sum form factors (PAPER.md:94-95 form; the coefficients are made up, not tabulated data)."""
    coef = [([2.0, 1.0], [3.0, 20.0], 0.5), ([0.8, 0.3], [1.5, 9.0], 0.1), ([1.2], [6.0], 0.0)]
    return np.stack([oracle.form_factor_gaussian(q, *coef[s]) for s in range(n_species)])


@pytest.mark.parametrize("N,S", [(7, 2), (40, 3)])
def test_species_direct_equals_pair_sum(N, S):
    """Eq.(2) with f_i(q) f_j(q) as an O(N^2) pair sum == the single-sum species oracle."""
    L = 5.5
    rng = np.random.default_rng(100 + N)
    pos = rng.uniform(0, L, (N, 3))
    sp = rng.integers(0, S, N)
    q = np.concatenate([oracle.lattice_q(L, -3, 7, -3, 7, m0=(l, 0, 0), ma=(0, 1, 0), mb=(0, 0, 1))
                        for l in range(-2, 3)])
    fq = _two_species_fq(q, S)
    a = oracle.species_intensity(pos, sp, fq, q, L)[0]
    b = oracle.pair_sum_species(pos, sp, fq, q, L)
    np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-10 * np.max(np.abs(b)))


def test_species_two_atoms_closed_form_and_constant_limit():
    """Two atoms of different kinds: I = fa(q)^2 + fb(q)^2 + 2 fa fb cos(q . (ra - rb)); q-independent tables reduce
    to the per-atom-f direct method (oracle.intensity, a separate routine)."""
    L = 7.0
    pos = np.array([[0.3, 1.9, 4.4], [5.1, 6.2, 0.7]])
    q = oracle.lattice_q(L, -4, 9, -4, 9, m0=(1, 0, 0), ma=(0, 1, 0), mb=(0, 0, 1))
    fq = _two_species_fq(q)
    I = oracle.species_intensity(pos, [0, 1], fq, q, L)[0]
    expect = fq[0] ** 2 + fq[1] ** 2 + 2 * fq[0] * fq[1] * np.cos(q @ (pos[0] - pos[1]))
    np.testing.assert_allclose(I, expect, rtol=1e-12, atol=1e-12)
    A = oracle.species_intensity(pos, [0, 1], fq, q, L, amp=True)[0]
    np.testing.assert_allclose(A, fq[0] * np.exp(-1j * (q @ pos[0])) + fq[1] * np.exp(-1j * (q @ pos[1])), atol=1e-12)
    rng = np.random.default_rng(3)
    pos = rng.uniform(0, L, (200, 3))
    sp = rng.integers(0, 3, 200)
    c = np.array([1.0, 2.5, 0.75])
    fq_const = np.repeat(c[:, None], q.shape[0], 1)
    np.testing.assert_allclose(oracle.species_intensity(pos, sp, fq_const, q, L)[0],
                               oracle.intensity(pos, c[sp], q, L)[0], rtol=1e-11, atol=1e-9)


def test_form_factor_is_fourier_transform_of_gaussian_density():
    """f(q) is the Fourier transform of the atom's electron density.  A density that is a sum of
    isotropic Gaussians n_i N(0, s_i^2 I) plus a point charge c has, by radial quadrature of
    f(q) = int 4 pi r^2 rho(r) sin(qr)/(qr) dr, the Gaussian-sum form c + sum a_i exp(-b_i (q/4pi)^2) with
    a_i = n_i and b_i = 8 pi^2 s_i^2."""
    from scipy.integrate import quad
    n_i, s_i, c = [2.0, 1.0], [0.2, 0.5], 0.5
    a = n_i
    b = [8 * np.pi ** 2 * s * s for s in s_i]
    for qm in [0.0, 0.7, 2.0, 5.5, 11.0]:
        def integrand(r):
            rho = sum(n * np.exp(-r * r / (2 * s * s)) / (2 * np.pi * s * s) ** 1.5 for n, s in zip(n_i, s_i))
            k = 1.0 if qm == 0 else np.sin(qm * r) / (qm * r)
            return 4 * np.pi * r * r * rho * k
        f_num = quad(integrand, 0, 10, limit=400, epsabs=1e-13)[0] + c
        f_or = oracle.form_factor_gaussian(np.array([[0.0, 0.0, qm]]), a, b, c)[0]
        assert abs(f_num - f_or) < 1e-9, (qm, f_num, f_or)


def test_volume_bragg_peaks_and_table1_grid():
    """3-D reciprocal-lattice block (Algorithm 1 step 1; Table 1's 81^3 grid): an SC
    crystal of n^3 atoms has I = N^2 exactly at h, k, l in n Z and 0 elsewhere -- pins the (l, h, k) index order.
    The Table 1 grid of the L = 59.19 A box has 531441 q with |q_c| <= 40 (2 pi / L)."""
    n_c, L = 4, 6.0
    pos = xi.crystal("sc", n_c, L)
    N = pos.shape[0]
    q = oracle.lattice_volume_q(L, -5, 11, -6, 12, -4, 9)
    I = oracle.intensity(pos, None, q, L)[0].reshape(9, 11, 12)
    l, h, k = np.meshgrid(np.arange(-4, 5), np.arange(-5, 6), np.arange(-6, 6), indexing="ij")
    peak = (h % n_c == 0) & (k % n_c == 0) & (l % n_c == 0)
    np.testing.assert_allclose(I[peak], float(N) ** 2, rtol=1e-12)
    assert np.max(I[~peak]) < 1e-8 * N
    g = _gold("paper_parameters.json")
    Lp = g["box_L_angstrom"]["value"]
    qt = oracle.lattice_volume_q(Lp, -40, 81, -40, 81, -40, 81)
    assert qt.shape == (81 ** 3, 3)
    np.testing.assert_allclose(np.abs(qt).max(0), 40 * 2 * np.pi / Lp, rtol=1e-15)


# ------------------------------------------------------------------ speckle statistics, Eq.(37)-(38)
@pytest.mark.parametrize("case", ["one_ring_M1", "two_rings_M2_remainder", "two_snapshots_per_snapshot_mean"])
def test_speckle_histogram_worked_examples(case):
    g = _gold("speckle_histogram.json")[case]
    counts, amb = oracle.speckle_histogram(np.array(g["I"]), np.array(g["bins"]), len(g["counts"]), g["M"],
                                           g["n_hist"], g["kappa_max"])
    np.testing.assert_array_equal(counts, g["counts"])


def test_erlang_pdf_is_the_gamma_law():
    """Eq.(38) is the Gamma(M, 1/M) density (sum of M iid Exp(1) normalised by M); M = 1 is
    Eq.(37)."""
    from scipy import stats
    k = np.linspace(0.01, 6, 200)
    for M in (1, 2, 5, 10, 20):
        np.testing.assert_allclose(oracle.erlang_pdf(k, M), stats.gamma(a=M, scale=1.0 / M).pdf(k), rtol=1e-12)


def test_speckle_histogram_follows_erlang_law():
    """Ideal-gas independent frames on lattice q: |p|^2 is exponential (fully coherent) and the sum of
    M independent patterns is Erlang.  The pooled histogram of kappa over rings and snapshots must
    match the bin integrals of Eq.(38) within 5 sigma (+ a 3% allowance for normalising by the ring's sample mean)."""
    from scipy import stats
    N, L, T, n = 400, 8.0, 48, 40
    pos = np.stack([xi.uniform_frame(500 + s, N, L) for s in range(T)])
    I = oracle.intensity(pos, None, oracle.lattice_q(L, **oracle.plane_grid(n)), L)
    bins = oracle.lattice_bins(n, n_bins=4)
    bins[bins == 0] = -1                                   # innermost ring: too few pixels
    for M in (1, 3, 6):
        n_hist, kmax = 16, 4.0
        counts, _ = oracle.speckle_histogram(I, bins, 4, M, n_hist, kmax)
        tot = counts.sum(0)
        n_all = int((bins >= 0).sum()) * (T // M)
        edges = np.linspace(0, kmax, n_hist + 1)
        cdf = stats.gamma(a=M, scale=1.0 / M).cdf(edges)
        expect = n_all * np.diff(cdf)
        assert np.all(np.abs(tot - expect) <= 5 * np.sqrt(expect + 1) + 0.03 * expect), (M, tot, expect)
        # invariants: every kappa < kmax is counted once; scaling I leaves kappa unchanged
        assert tot.sum() <= n_all
        c2, _ = oracle.speckle_histogram(I * 3.5, bins, 4, M, n_hist, kmax)
        np.testing.assert_array_equal(c2, counts)


# ------------------------------------------------------------------ Algorithm 2, the FFT method
def test_fft_method_shift_theorem():
    """An atom on a grid point n*dx deposits the origin Gaussian shifted by whole grid steps, so its FFT is
    f^eta(q) e^{-i q . r} exactly (DFT shift theorem): I = 1 at every q; two such atoms give 2 + 2 cos(q . dr)."""
    L, n, eta = 6.0, 24, 0.3
    dx = L / n
    one = np.array([[5 * dx, 17 * dx, 2 * dx]])
    I = oracle.fft_intensity(one, L, n, eta)
    np.testing.assert_allclose(I, 1.0, rtol=1e-7)      # ratio of Gaussian tails ~1e-3 at the grid edge
    two = np.array([[5 * dx, 17 * dx, 2 * dx], [11 * dx, 0.0, 23 * dx]])
    I = oracle.fft_intensity(two, L, n, eta)
    m = np.fft.fftfreq(n, 1.0 / n)
    H, K, Lq = np.meshgrid(m, m, m, indexing="ij")
    d = two[0] - two[1]
    expect = 2 + 2 * np.cos((2 * np.pi / L) * (H * d[0] + K * d[1] + Lq * d[2]))
    np.testing.assert_allclose(I, expect, atol=1e-7)


def test_fft_method_matches_direct_method_at_low_q():
    """Algorithm 2 approximates Algorithm 1: with eta ~ one grid spacing (the paper's 0.1485 A at
    N_grid = 400, L = 59.19 A) the two agree on the low-|q| block of the grid to < 1e-3 N per pixel;
    the kernel width follows the 10 eta rule (k = 11 for eta = dx)."""
    L, n, N = 10.0, 64, 300
    eta = L / n
    assert oracle.fft_kernel_width(L, n, eta) == 11
    pos = xi.uniform_frame(31, N, L)
    I = oracle.fft_intensity(pos, L, n, eta)
    h = n // 8
    Ib = oracle.fft_block(I, -h, 2 * h, -h, 2 * h, -h, 2 * h)
    Id = oracle.intensity(pos, None, oracle.lattice_volume_q(L, -h, 2 * h, -h, 2 * h, -h, 2 * h), L)[0]
    assert np.max(np.abs(Ib - Id)) < 1e-3 * N
    assert abs(Ib.reshape(2 * h, 2 * h, 2 * h)[h, h, h] - N * N) < 1e-3 * N * N    # forward point ~ N^2


# ------------------------------------------------------------------ hand-computed estimator examples (golden)
# tests/golden/estimators.json holds worked examples written by hand from the definitions; each fixes a choice a
# plausible estimator could get wrong (symmetric g2 normalisation, sample variance, a kept remainder window,
# binning |q|^2, the conjugate amplitude).
def _nan(a):
    return np.array([[np.nan if v is None else v for v in row] for row in a], dtype=np.float64)


def test_golden_g2_literal_eq14():
    """Eq.(14), literal normalisation (R6): hand-computed g2 of a 4-frame series."""
    g = _gold("estimators.json")["g2_literal"]
    out = oracle.g2(np.array(g["I"]), g["lags"])
    np.testing.assert_allclose(out, _nan(g["g2"]), rtol=1e-14, atol=1e-15, equal_nan=True)


def test_golden_xsvs_population_variance_and_dropped_remainder():
    """Eq.(15)+(17): hand-computed beta with T = 5 not divisible by W = 2, 3,
    a 3-pixel ring, a single-pixel ring (population variance 0) and an empty ring (NaN)."""
    g = _gold("estimators.json")["xsvs_population_variance_remainder_dropped"]
    out = oracle.xsvs_beta(np.array(g["I"]), np.array(g["bins"]), g["n_bins"], g["windows"])
    np.testing.assert_allclose(out, _nan(g["beta"]), rtol=1e-13, atol=1e-15, equal_nan=True)


def test_golden_radial_bins_edges():
    """PAPER.md:192 half-open rings of |q|: explicit |q| values at and either side of the bin edges."""
    g = _gold("estimators.json")["radial_bins_edges"]
    out = oracle.radial_bins(np.array(g["q"]), g["q_max"], g["n_bins"])
    np.testing.assert_array_equal(out, g["bins"])


def test_golden_amplitude_sign_quarter_box():
    """Eq.(7): e^{-i q.r}; an atom at L/4 with q = 2 pi / L x gives p = -i."""
    g = _gold("estimators.json")["amplitude_sign"]
    L = g["L"]
    for c in g["cases"]:
        A = oracle.amplitude(np.array(c["pos"]), np.array(c["f"]), _hkl_q(L, c["hkl"]), L)
        np.testing.assert_allclose(A.real, c["re"], atol=1e-12)
        np.testing.assert_allclose(A.imag, c["im"], atol=1e-12)


def test_golden_isf_order_and_pair_count():
    """Eq.(22)-(23): p(t) p*(t + tau) (not p*(t) p(t + tau)), averaged over the T - tau pairs;
    hand-computed 3-frame, 2-pixel series."""
    g = _gold("estimators.json")["isf_order_and_pair_count"]
    A = np.array(g["A_re"]) + 1j * np.array(g["A_im"])
    F = oracle.isf(A, g["lags"], g["S2"])
    np.testing.assert_allclose(F.real, g["F_re"], atol=1e-15)
    np.testing.assert_allclose(F.imag, g["F_im"], atol=1e-15)


def test_golden_ewald_orientation():
    """Eq.(1), PAPER.md:74-77 with reading R4: hand-computed q of off-axis pixels of a 3 x 3 detector (fixes which
    pixel index runs along x and y, and the sign of each component)."""
    g = _gold("estimators.json")["ewald_orientation"]
    q = oracle.ewald_q(g["wavelength"], g["npx"], g["npy"], g["pitch"])
    np.testing.assert_allclose(q[g["pixels"]], g["q"], atol=1e-15)
