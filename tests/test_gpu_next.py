"""GPU tests of the SURVEY 8(f) rows built so far: complex amplitude output (Eq. 7), the intermediate scattering
function F(q, tau) (Eq. 22) and the paper's Fig. 4 / Fig. 8 relations evaluated on GPU outputs:
  * Siegert relation g2 = 1 + beta0 |F^|^2 (Eq. 24),
  * beta from q-space (Eq. 17) = beta0 from time (Eq. 19) for an ergodic system,
  * incoherent superposition of M independent patterns: beta = 1/M."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402

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


def _cplx(A):
    a = A.cpu().numpy().astype(np.float64)
    return a[..., 0] + 1j * a[..., 1]


def _amp_gate(A_gpu, A_or, N):
    """|dp| <= 1e-3 sqrt(N) + 1e-5 |p|: the amplitude form of the intensity gate (R11)."""
    err = np.abs(A_gpu - A_or)
    ratio = np.max(err / (1e-3 * np.sqrt(N) + 1e-5 * np.abs(A_or)))
    assert ratio <= 1.0, ratio
    return ratio


@pytest.mark.parametrize("engine", [xp.ENGINE_TENSOR, xp.ENGINE_SIMT])
def test_amplitude_grid_parity(engine):
    cfg = xi.scaled(xi.CONFIGS["c3"], N=6001, T=3)
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg)
    g = xp.qgrid(cfg.L, -100, 200, -70, 140, m0=(0, 0, 3))
    A = _cplx(xp.xpcs_amplitude_grid(_t(pos), _t(f), g, engine=engine))
    q = oracle.lattice_q(g.L, g.h0, g.n_h, g.k0, g.n_k, (0, 0, 3))
    ref = oracle.amplitudes(pos, f.astype(np.float64), q, cfg.L)
    _amp_gate(A, ref, cfg.N)
    I = xp.xpcs_intensity_grid(_t(pos), _t(f), g, engine=engine).cpu().numpy()
    np.testing.assert_allclose(np.abs(A) ** 2, I, rtol=2e-6, atol=1e-6 * cfg.N)


def test_amplitude_explicit_q_and_fp64():
    N, L = 3000, 15.0
    pos = np.stack([xi.uniform_frame(40 + s, N, L, "f32") for s in range(2)])
    q = np.random.default_rng(2).uniform(-9, 9, (700, 3)).astype(np.float32)
    A = _cplx(xp.xpcs_amplitude(_t(pos), None, _t(q), L))
    _amp_gate(A, oracle.amplitudes(pos, None, q.astype(np.float64), L), N)
    pos64 = pos.astype(np.float64)
    g = xp.qgrid(L, -9, 18, -9, 18)
    A64 = _cplx(xp.xpcs_amplitude_grid(_t(pos64), None, g))
    ref = oracle.amplitudes(pos64, None, oracle.lattice_q(L, -9, 18, -9, 18), L)
    np.testing.assert_allclose(A64, ref, rtol=1e-9, atol=1e-9 * N)


def test_isf_reduction_parity():
    rng = np.random.default_rng(12)
    T, n_q = 90, 2000
    A = (rng.standard_normal((T, n_q)) + 1j * rng.standard_normal((T, n_q))) * 30
    Af = np.stack([A.real, A.imag], -1).astype(np.float32)
    lags = [0, 1, 2, 3, 10, 44, 89] + list(range(20, 40))
    f = np.where(np.arange(500) % 2 == 1, 2.0, 1.0).astype(np.float32)
    F = _cplx(xp.xpcs_isf(_t(Af), lags, _t(f), 500))
    ref = oracle.isf(Af[..., 0].astype(np.float64) + 1j * Af[..., 1].astype(np.float64), lags, float(np.sum(f.astype(np.float64) ** 2)))
    np.testing.assert_allclose(F, ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())
    F1 = _cplx(xp.xpcs_isf(_t(Af), lags, None, 500))
    np.testing.assert_allclose(F1, ref * np.sum(f.astype(np.float64) ** 2) / 500, rtol=1e-10,
                               atol=1e-12 * np.abs(ref).max())


def test_siegert_relation_on_gpu_outputs():
    """Fig. 4b analogue: (g2 - 1)/beta0 vs |F^|^2 ring by ring for Brownian frames (all quantities from the GPU).
    Both estimate exp(-2 D q^2 tau); the literal g2 is biased by O(1/T) on fast rings, hence the tolerance."""
    cfg = xi.scaled(xi.CONFIGS["c2"], N=4000, T=400)
    pos = xi.positions(cfg)
    n = 64
    g = xp.qgrid(cfg.L, -n // 2, n, -n // 2, n)
    A = xp.xpcs_amplitude_grid(_t(pos), None, g)
    I = xp.xpcs_intensity_grid(_t(pos), None, g)
    lags = [0, 1, 2, 4]
    F = _cplx(xp.xpcs_isf(A, lags, None, cfg.N))
    G = xp.xpcs_g2(I, lags).cpu().numpy()
    bins = oracle.lattice_bins(n, n_bins=8)
    q2 = (oracle.lattice_q(cfg.L, **oracle.plane_grid(n)) ** 2).sum(1)
    Fhat2 = np.abs(F / F[0]) ** 2
    for b in range(3, 8):
        sel = bins == b
        beta0 = np.mean(G[0, sel] - 1)
        for li in (1, 2, 3):
            lhs = np.mean((G[li, sel] - 1)) / beta0
            rhs = np.mean(Fhat2[li, sel])
            pred = np.mean(np.exp(-2 * cfg.D * q2[sel] * lags[li] * cfg.dt))
            assert abs(lhs - rhs) < 0.05 + 0.1 * pred, (b, li, lhs, rhs, pred)
            assert abs(rhs - pred) < 0.05 + 0.1 * pred, (b, li, rhs, pred)


def test_beta_q_space_equals_beta_time_and_superposition():
    """Eq.(17) vs Eq.(19): the contrast over a ring of one frame equals g2(0) - 1 over time;
    for independent configurations, the XSVS window sum of M frames is the incoherent M-superposition
     whose contrast is beta0 / M (Erlang statistics)."""
    cfg = xi.scaled(xi.CONFIGS["c4"], N=3000, T=64)
    pos = xi.positions(cfg)                       # independent uniform frames (ideal gas)
    n = 128
    g = xp.qgrid(cfg.L, -n // 2, n, -n // 2, n)
    I = xp.xpcs_intensity_grid(_t(pos), None, g)
    bins = _t(oracle.lattice_bins(n, n_bins=8))
    windows = [1, 2, 4, 8]
    beta = xp.xsvs_contrast(I, bins, 8, windows).cpu().numpy()
    G0 = xp.xpcs_g2(I, [0])
    beta_t = xp.xpcs_shell_mean(G0, bins, 8).cpu().numpy()[0] - 1.0
    beta0 = 1 - 1.0 / cfg.N                       # single species: S4 / S2^2 = 1/N
    for b in range(3, 8):
        n_eff = int((oracle.lattice_bins(n, n_bins=8) == b).sum()) / 2
        assert abs(beta[0, b] - beta0) < 0.08, (b, beta[0, b])                 # q-space contrast ~ 1
        assert abs(beta_t[b] - beta0) < 0.08, (b, beta_t[b])                   # time contrast ~ 1
        assert abs(beta[0, b] - beta_t[b]) < 0.1
        for wi, M in enumerate(windows):
            assert abs(beta[wi, b] * M - beta0 * (1 - 2 / n_eff)) < 0.15, (b, M, beta[wi, b])


def _hist_close(got, counts, amb):
    """Exact integer counts; a value within 1e-9 of a bin edge e may sit on either side (different FP64 summation
    order of the ring mean): allow moves between bins e-1 and e bounded by ambiguous[e]."""
    d = got.astype(np.int64) - counts
    if not d.any():
        return
    carry = np.zeros(d.shape[0], dtype=np.int64)
    for e in range(d.shape[1]):
        carry = carry + d[:, e]
        assert np.all(np.abs(carry) <= amb[:, e + 1]), (e, d, amb)


@pytest.mark.parametrize("M,n_hist,kmax", [(1, 40, 8.0), (3, 25, 5.0), (7, 1000, 3.0)])
def test_speckle_histogram_reduction_parity(M, n_hist, kmax):
    rng = np.random.default_rng(M)
    T, n = 45, 96
    I = rng.exponential(1.0, (T, n * n)).astype(np.float32) * 37.0
    bins = oracle.lattice_bins(n, n_bins=16)
    got = xp.xpcs_speckle_histogram(_t(I), _t(bins), 16, M, n_hist, kmax).cpu().numpy()
    counts, amb = oracle.speckle_histogram(I, bins, 16, M, n_hist, kmax)
    _hist_close(got, counts, amb)


def test_erlang_statistics_on_gpu_outputs():
    """PAPER.md:560-572 (Fig. 8 analogue): M independent ideal-gas patterns superposed -> Erlang(M) intensity law
    (Eq. 38) and contrast 1/M, all from GPU outputs (I by the tensor engine, histogram and XSVS by the library)."""
    from scipy import stats
    cfg = xi.scaled(xi.CONFIGS["c4"], N=2000, T=40)
    pos = xi.positions(cfg)
    n = 128
    I = xp.xpcs_intensity_grid(_t(pos), None, xp.qgrid(cfg.L, -n // 2, n, -n // 2, n))
    bins_h = oracle.lattice_bins(n, n_bins=8)
    bins_h[bins_h < 2] = -1
    bins = _t(bins_h)
    n_hist, kmax = 20, 4.0
    edges = np.linspace(0, kmax, n_hist + 1)
    for M in (1, 5, 10, 20):
        got = xp.xpcs_speckle_histogram(I, bins, 8, M, n_hist, kmax).cpu().numpy().sum(0)
        n_all = int((bins_h >= 0).sum()) * (cfg.T // M)
        expect = n_all * np.diff(stats.gamma(a=M, scale=1.0 / M).cdf(edges))
        assert np.all(np.abs(got - expect) <= 5 * np.sqrt(expect + 1) + 0.04 * expect), (M, got, expect)
    beta = xp.xsvs_contrast(I, bins, 8, [1, 5, 10, 20]).cpu().numpy()
    for wi, M in enumerate((1, 5, 10, 20)):
        assert np.all(np.abs(beta[wi, 2:] * M - 1.0) < 0.12), (M, beta[wi])


def test_registered_ring_plan_gives_identical_reductions():
    """xpcs_rings_register: the cached plan gives bit-identical ring reductions; unregister frees it."""
    rng = np.random.default_rng(5)
    T, n = 20, 64
    I = _t(rng.exponential(1.0, (T, n * n)).astype(np.float32))
    bins = _t(oracle.lattice_bins(n, n_bins=8))
    a = [xp.xsvs_contrast(I, bins, 8, [1, 2, 5]), xp.xpcs_shell_mean(I, bins, 8),
         xp.xpcs_speckle_histogram(I, bins, 8, 2, 16, 4.0)]
    xp.xpcs_rings_register(bins, 8)
    b = [xp.xsvs_contrast(I, bins, 8, [1, 2, 5]), xp.xpcs_shell_mean(I, bins, 8),
         xp.xpcs_speckle_histogram(I, bins, 8, 2, 16, 4.0)]
    xp.xpcs_rings_unregister(bins)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    with pytest.raises(xp.XpcsError, match="not registered"):
        xp.xpcs_rings_unregister(bins)
