"""Tolerances of the parity gates.

Per pixel (north_star, R11):  |I_gpu - I_oracle| <= 1e-3 * N + 1e-5 * I_oracle
  N is the atom count (stricter than sum f^2 for two species); the relative branch only matters where
  I > 100 N (Bragg peaks, the forward box term of off-lattice detectors), where fp32 output rounding alone
  exceeds 1e-3 N.
Ring-averaged S(q) and g2: <= 1e-4 relative (north_star); reductions on identical input: <= 1e-10 relative.
"""
import numpy as np

ABS_PER_ATOM = 1e-3
REL = 1e-5


def pixel_gate(I_gpu, I_or, N):
    """Returns (worst ratio |err| / allowed, max |err| / N, #pixels that needed the relative branch)."""
    I_gpu = np.asarray(I_gpu, dtype=np.float64)
    I_or = np.asarray(I_or, dtype=np.float64)
    err = np.abs(I_gpu - I_or)
    allowed = ABS_PER_ATOM * N + REL * np.abs(I_or)
    ratio = float(np.max(err / allowed)) if err.size else 0.0
    needed_rel = int(np.sum(err > ABS_PER_ATOM * N))
    return ratio, float(np.max(err) / N) if err.size else 0.0, needed_rel


def assert_pixels(I_gpu, I_or, N, what=""):
    ratio, worst, n_rel = pixel_gate(I_gpu, I_or, N)
    assert np.all(np.isfinite(I_gpu)), what
    assert ratio <= 1.0, f"{what}: worst err/allowed = {ratio:.3g}, max |dI|/N = {worst:.3g}, rel-branch pixels {n_rel}"
    return ratio, worst


def assert_rel(a, b, tol, what=""):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    nan_a, nan_b = np.isnan(a), np.isnan(b)
    assert np.array_equal(nan_a, nan_b), f"{what}: NaN pattern differs"
    ok = ~nan_a
    if ok.any():
        rel = np.max(np.abs(a[ok] - b[ok]) / np.maximum(np.abs(b[ok]), 1e-300))
        assert rel <= tol, f"{what}: max rel err {rel:.3g} > {tol}"
        return float(rel)
    return 0.0
