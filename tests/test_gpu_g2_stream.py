"""Block-streamed g2 (include/xpcs.h xpcs_g2_accumulate / xpcs_g2_finalize; SURVEY 8(d) K4 "update in blocks of B
frames"): a series pushed in blocks of any sizes must give Eq.(14) of the whole series -- the FP64 oracle's g2 at
1e-10, and xpcs_g2 on the resident series up to summation order (1e-12).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402
from _gates import assert_rel  # noqa: E402

DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    xp.load()
    yield
    xp.release()


def _stream(I, lags, blocks, dtype):
    S = xp.G2Stream(I.shape[1], lags, dtype=dtype, device=DEV)
    t = 0
    for b in blocks:
        S.push(I[t:t + b])
        t += b
    assert t == I.shape[0]
    return S.result()


@pytest.mark.parametrize("lags,blocks", [
    ((0, 1, 2, 3, 5, 8, 13, 40, 100), (1, 37, 100, 64, 55)),          # non-consecutive lags, blocks < and > max lag
    (tuple(range(1, 65)), (50, 50, 50, 50, 57)),                       # 64 consecutive lags: 16 lags per warp
    (tuple(range(0, 20)), (257,)),                                     # one block
    ((7,), (3, 3, 3, 3, 245)),                                         # blocks shorter than the lag
])
def test_streamed_g2_equals_whole_series(lags, blocks):
    rng = np.random.default_rng(len(lags) + len(blocks))
    T, n_q = sum(blocks), 3000                                         # ragged pixel count (not a multiple of 32)
    I_h = rng.exponential(2.0, (T, n_q)).astype(np.float32)
    I_h[:, 17] = 0.0                                                   # a dark pixel: NaN
    I = torch.from_numpy(I_h).to(DEV)
    g = _stream(I, lags, blocks, torch.float32).cpu().numpy()
    whole = xp.xpcs_g2(I, lags).cpu().numpy()
    assert_rel(g, whole, 1e-12, "streamed vs resident g2")
    assert_rel(g, oracle.g2(I_h, lags), 1e-10, "streamed g2 vs oracle")


def test_streamed_g2_fp64_input_and_float_output():
    rng = np.random.default_rng(3)
    T, n_q, lags = 90, 700, (1, 2, 3, 4, 30, 89)
    I_h = rng.exponential(1.0, (T, n_q))
    I = torch.from_numpy(I_h).to(DEV)
    S = xp.G2Stream(n_q, lags, dtype=torch.float64, device=DEV)
    for t in range(0, T, 29):
        S.push(I[t:t + 29])
    g32 = S.result(out_dtype=xp.F32)
    assert g32.dtype == torch.float32
    np.testing.assert_allclose(g32.cpu().numpy(), oracle.g2(I_h, lags), rtol=1e-6)
    assert_rel(S.result().cpu().numpy(), oracle.g2(I_h, lags), 1e-10, "fp64 streamed g2")


def test_ring_too_small_is_rejected():
    I = torch.ones((4, 64), device=DEV)
    ring = torch.empty((2, 64), device=DEV)
    acc = torch.zeros((1, 64), dtype=torch.float64, device=DEV)
    s = torch.zeros((64,), dtype=torch.float64, device=DEV)
    with pytest.raises(xp.XpcsError):
        xp.xpcs_g2_accumulate(I, 0, (3,), ring, acc, s)
