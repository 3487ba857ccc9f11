"""GPU path against the hand-computed worked examples of tests/golden/estimators.json (no oracle in between).

The same examples pin the oracle (tests/test_oracle_pins.py); here the CUDA kernels, called through the C ABI,
must reproduce the paper-derived numbers directly: the literal Eq.(14) g2, the Eq.(15)/(17) contrast with the
population variance and dropped remainder, the half-open |q| rings and the e^{-iq.r} sign of Eq.(7) (every
amplitude engine, including the tensor engines whose partials hold conj(p)).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2204_13241_b200 as xp  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "estimators.json")
DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    xp.load()
    yield
    xp.release()


def _g(name):
    with open(GOLD) as fh:
        return json.load(fh)[name]


def _nan(a):
    return np.array([[np.nan if v is None else v for v in row] for row in a], dtype=np.float64)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_gpu_g2_literal_eq14(dtype):
    g = _g("g2_literal")
    I = torch.tensor(g["I"], dtype=dtype, device=DEV)
    out = xp.xpcs_g2(I, g["lags"]).cpu().numpy()
    np.testing.assert_allclose(out, _nan(g["g2"]), rtol=1e-14, atol=1e-15, equal_nan=True)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_gpu_xsvs_population_variance_remainder_dropped(dtype):
    g = _g("xsvs_population_variance_remainder_dropped")
    I = torch.tensor(g["I"], dtype=dtype, device=DEV)
    bins = torch.tensor(g["bins"], dtype=torch.int32, device=DEV)
    out = xp.xsvs_contrast(I, bins, g["n_bins"], g["windows"]).cpu().numpy()
    np.testing.assert_allclose(out, _nan(g["beta"]), rtol=1e-13, atol=1e-15, equal_nan=True)


def test_gpu_radial_bins_edges():
    g = _g("radial_bins_edges")
    q = torch.tensor(g["q"], dtype=torch.float64, device=DEV)
    out = xp.xpcs_radial_bins(q, g["q_max"], g["n_bins"]).cpu().numpy()
    np.testing.assert_array_equal(out, g["bins"])


def test_gpu_amplitude_sign_explicit_q():
    g = _g("amplitude_sign")
    L = g["L"]
    for c in g["cases"]:
        pos = torch.tensor([c["pos"]], dtype=torch.float64, device=DEV)
        f = torch.tensor(c["f"], dtype=torch.float64, device=DEV)
        q = torch.tensor((2 * np.pi / L) * np.asarray(c["hkl"], np.float64), device=DEV)
        A = xp.xpcs_amplitude(pos, f, q, L).cpu().numpy()[0]
        np.testing.assert_allclose(A[:, 0], c["re"], atol=1e-12)
        np.testing.assert_allclose(A[:, 1], c["im"], atol=1e-12)


@pytest.mark.parametrize("engine", [xp.ENGINE_AUTO, xp.ENGINE_SIMT, xp.ENGINE_TENSOR, xp.ENGINE_TENSOR_I8])
def test_gpu_amplitude_sign_lattice_engines(engine):
    """The quarter-box atom on a lattice plane through every fp32 engine: p(h = 1, k = 0) = -i, p(-1, 0) = +i, and
    p(h, k) = exp(-i pi h / 2) for the whole plane (the atom sits on the x axis)."""
    L = 8.0
    pos = torch.tensor([[[2.0, 0.0, 0.0]]], dtype=torch.float32, device=DEV)
    grid = xp.qgrid(L, -4, 8, -3, 6)
    A = xp.xpcs_amplitude_grid(pos, None, grid, engine=engine).cpu().numpy()[0]
    h = np.arange(-4, 4)[:, None] * np.ones((1, 6))
    expect = np.exp(-0.5j * np.pi * h).reshape(-1)
    tol = 2e-4 if engine in (xp.ENGINE_TENSOR_I8, xp.ENGINE_AUTO) else 1e-5
    np.testing.assert_allclose(A[:, 0], expect.real, atol=tol)
    np.testing.assert_allclose(A[:, 1], expect.imag, atol=tol)


def test_gpu_isf_order_and_pair_count():
    """Eq.(22)-(23): p(t) p*(t + tau) over the T - tau pairs, hand-computed (estimators.json)."""
    g = _g("isf_order_and_pair_count")
    A = torch.stack([torch.tensor(g["A_re"], dtype=torch.float64), torch.tensor(g["A_im"], dtype=torch.float64)], -1)
    F = xp.xpcs_isf(A.to(DEV).contiguous(), g["lags"], None, N=int(g["S2"])).cpu().numpy()   # f = 1: sum f^2 = N
    np.testing.assert_allclose(F[..., 0], g["F_re"], atol=1e-15)
    np.testing.assert_allclose(F[..., 1], g["F_im"], atol=1e-15)


def test_gpu_ewald_orientation():
    """Eq.(1), PAPER.md:74-77 with reading R4: hand-computed q of off-axis pixels of a 3 x 3 detector."""
    g = _g("ewald_orientation")
    q = xp.xpcs_qgrid_ewald(g["wavelength"], g["npx"], g["npy"], g["pitch"], out_dtype=xp.F64, device=DEV)
    np.testing.assert_allclose(q.cpu().numpy()[g["pixels"]], g["q"], atol=1e-14)


@pytest.mark.parametrize("case", ["one_ring_M1", "two_rings_M2_remainder", "two_snapshots_per_snapshot_mean"])
def test_gpu_speckle_histogram_worked_examples(case):
    """Eq.(37)-(38) statistics: hand-computed histograms (speckle_histogram.json)."""
    with open(os.path.join(os.path.dirname(__file__), "golden", "speckle_histogram.json")) as fh:
        g = json.load(fh)[case]
    I = torch.tensor(g["I"], dtype=torch.float64, device=DEV)
    bins = torch.tensor(g["bins"], dtype=torch.int32, device=DEV)
    out = xp.xpcs_speckle_histogram(I, bins, len(g["counts"]), g["M"], g["n_hist"], g["kappa_max"]).cpu().numpy()
    np.testing.assert_array_equal(out, g["counts"])
