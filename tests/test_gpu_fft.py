"""GPU parity of SURVEY 8(f) rank 4: Algorithm 2, the FFT-based method, through the C ABI, against
the FP64 numpy oracle (oracle.fft_intensity) and -- within the method's own discretisation error -- the direct method."""
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


@pytest.mark.parametrize("n,eta,k,dtype", [(32, 0.35, 0, "f64"), (48, 0.2, 0, "f32"), (40, 0.3, 7, "f64")])
def test_fft_method_parity(n, eta, k, dtype):
    """Full grid, several frames (batched cuFFT), ragged block, negative l (Hermitian half spectrum)."""
    L, N, T = 8.0, 257, 3
    pos = np.stack([xi.uniform_frame(700 + s, N, L, dtype) for s in range(T)])
    h = n // 2
    blk = xp.qvolume(L, -h, n, -h + 3, n - 5, -h, n)
    I = xp.xpcs_intensity_fft(_t(pos), blk, n, eta, k, out_dtype=xp.F64).cpu().numpy()
    # I = |p^eta|^2 / f^eta^2: where f^eta ~ exp(-q^2 eta^2 / 2) is tiny (grid corners) both sides divide FFT round-off
    # by it; compare where f^eta > 1e-3 (the usable part of the grid), require finite values elsewhere
    q = oracle.lattice_volume_q(L, -h, n, -h + 3, n - 5, -h, n)
    usable = np.exp(-(q * q).sum(1) * eta * eta / 2) > 1e-3
    assert usable.mean() > 0.2
    for t in range(T):
        ref = oracle.fft_block(oracle.fft_intensity(pos[t].astype(np.float64), L, n, eta, k), -h, n, -h + 3, n - 5, -h, n)
        np.testing.assert_allclose(I[t][usable], ref[usable], rtol=1e-7, atol=1e-10 * N)
        assert np.all(np.isfinite(I[t]))


def test_fft_method_shift_theorem_and_direct_method():
    L, n = 10.0, 64
    dx = L / n
    one = np.array([[[7 * dx, 33 * dx, 60 * dx]]])
    blk = xp.qvolume(L, -32, 64, -32, 64, -32, 64)
    I = xp.xpcs_intensity_fft(_t(one), blk, n, dx, out_dtype=xp.F64).cpu().numpy()
    np.testing.assert_allclose(I, 1.0, rtol=1e-7)
    N = 600
    pos = xi.uniform_frame(17, N, L)[None]
    h = n // 8
    blk = xp.qvolume(L, -h, 2 * h, -h, 2 * h, -h, 2 * h)
    I = xp.xpcs_intensity_fft(_t(pos), blk, n, dx, out_dtype=xp.F64).cpu().numpy()[0]
    Id = oracle.intensity(pos[0], None, oracle.lattice_volume_q(L, -h, 2 * h, -h, 2 * h, -h, 2 * h), L)[0]
    assert np.max(np.abs(I - Id)) < 1e-3 * N
    Ig = xp.xpcs_intensity_volume(_t(pos.astype(np.float32)), None, blk).cpu().numpy()[0]
    assert np.max(np.abs(I - Ig)) < 2e-3 * N


def test_fft_method_form_factor():
    L, n, N = 8.0, 32, 100
    pos = xi.uniform_frame(4, N, L)[None]
    blk = xp.qvolume(L, -5, 10, -5, 10, 0, 3)
    fq = oracle.form_factor_gaussian(oracle.lattice_volume_q(L, -5, 10, -5, 10, 0, 3), [2.0], [10.0], 0.5)
    I1 = xp.xpcs_intensity_fft(_t(pos), blk, n, 0.3, out_dtype=xp.F64).cpu().numpy()
    If = xp.xpcs_intensity_fft(_t(pos), blk, n, 0.3, f_q=_t(fq), out_dtype=xp.F64).cpu().numpy()
    np.testing.assert_allclose(If, I1 * fq ** 2, rtol=1e-12)
