"""Invariants of the reductions evaluated directly on the GPU kernels (SPEC S:349-360, S:376-377,
S:435-437), independent of the oracle:
  * g2 of a constant series is exactly 1; g2 and beta are invariant to a global intensity scale (powers of two:
    exact in floating point);
  * a static series (every frame the same pattern) has beta_W = beta_1 for every window W (I_W = W I);
  * a constant field has beta = 0 (population variance of equal values);
  * the ring means of a constant field equal it, and S(q) of f = 1 atoms is I / N."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_13241_b200 as xp  # noqa: E402

DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    xp.load()
    yield
    xp.release()


def _bins(n, n_bins):
    g = xp.lattice_plane(10.0, n)
    return xp.xpcs_lattice_bins(g, n_bins, n // (2 * n_bins), DEV)


def test_g2_constant_series_and_scale_invariance():
    rng = np.random.default_rng(5)
    T, n_q = 40, 64 * 64
    const = torch.full((T, n_q), 3.5, dtype=torch.float32, device=DEV)
    g = xp.xpcs_g2(const, [0, 1, 7, 39]).cpu().numpy()
    assert np.all(g == 1.0)
    I = torch.from_numpy(rng.exponential(1.0, (T, n_q)).astype(np.float32)).to(DEV)
    a = xp.xpcs_g2(I, [0, 1, 2, 5, 11]).cpu().numpy()
    b = xp.xpcs_g2(I * 8.0, [0, 1, 2, 5, 11]).cpu().numpy()
    np.testing.assert_allclose(a, b, rtol=1e-14)


def test_xsvs_static_series_and_constant_field():
    rng = np.random.default_rng(6)
    n, nb, T = 64, 16, 64
    bins = _bins(n, nb)
    frame = rng.exponential(1.0, n * n).astype(np.float32)
    static = torch.from_numpy(np.tile(frame, (T, 1))).to(DEV)
    beta = xp.xsvs_contrast(static, bins, nb, [1, 2, 4, 8, 16, 32, 64]).cpu().numpy()
    ok = np.isfinite(beta[0])
    assert ok.sum() >= nb - 2
    np.testing.assert_allclose(beta[:, ok], np.broadcast_to(beta[0, ok], beta[:, ok].shape), rtol=1e-12)
    # the window-1 contrast of an Exp(1) field is ~1: averaged over the rings (each ring's estimate has a relative
    # spread of ~sqrt(20 / n_ring) for Exp(1) pixels)
    assert abs(np.mean(beta[0, 4:nb - 1]) - 1.0) < 0.15
    const = torch.full((T, n * n), 2.0, dtype=torch.float32, device=DEV)
    b0 = xp.xsvs_contrast(const, bins, nb, [1, 3, 8]).cpu().numpy()
    assert np.all(np.abs(b0[:, ok]) < 1e-14)
    S = xp.xpcs_shell_mean(const, bins, nb).cpu().numpy()
    assert np.all(S[:, ok] == 2.0)
    Sq = xp.xpcs_structure_factor_shells(const, None, 4, bins, nb).cpu().numpy()
    np.testing.assert_allclose(Sq[:, ok], 0.5, rtol=1e-15)
