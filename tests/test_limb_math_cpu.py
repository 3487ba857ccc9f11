"""CPU checks of the integer engine's limb arithmetic (k_lattice_i8.cu), emulated bit-exactly in
numpy: one FP32 FMA t = fma(v, 32512, 1.5 * 2^23 + 128) (exact product, one rounding: emulated in FP64, where
v * 32512 + M is exact, then rounded once to FP32) must leave y = rint(32512 v) + 128 in the low 16 bits of t, with
byte 1 = hi and byte 0 = lo + 128; the two limbs must reconstruct x = 256 hi + lo exactly, stay inside int8, and
the three-product form must approximate v w within the stated bound.  These pin the kernel's encoding, not the
physics (the GPU parity tests compare whole intensities with the FP64 oracle)."""
import numpy as np

QS = 32512.0
M = 12582912.0          # 1.5 * 2^23


def _fma_f32(v, a, c):
    # FP32 FMA: v and a, c exact in FP64; v * a + c is exact in FP64 for |v| <= 1 (24 + 15 bits), one rounding to FP32
    return (v.astype(np.float64) * a + c).astype(np.float32)


def _limbs(v, scale=QS):
    t = _fma_f32(v, scale, M + 128.0)
    bits = t.view(np.uint32)
    hi = ((bits >> 8) & 0xFF).astype(np.int64)
    lo = (((bits & 0xFF) ^ 0x80)).astype(np.int64)
    hi = np.where(hi >= 128, hi - 256, hi)
    lo = np.where(lo >= 128, lo - 256, lo)
    return hi, lo


def _grid():
    rng = np.random.default_rng(2204)
    dense = np.linspace(-1.0, 1.0, 200001, dtype=np.float64).astype(np.float32)
    rand = rng.uniform(-1.0, 1.0, 200000).astype(np.float32)
    # exact ties of 32512 v (half-integers) and the range ends
    ties = ((np.arange(-32512, 32512) + 0.5) / QS).astype(np.float32)
    ends = np.array([-1.0, -0.99999994, 0.0, -0.0, 0.99999994, 1.0], dtype=np.float32)
    return np.concatenate([dense, rand, ties, ends])


def test_q16_bytes_reconstruct_rint():
    v = _grid()
    hi, lo = _limbs(v)
    x = np.rint(v.astype(np.float64) * QS).astype(np.int64)   # round-half-even, like the FMA's rounding
    assert np.array_equal(256 * hi + lo, x)
    assert hi.min() >= -127 and hi.max() <= 127
    assert lo.min() >= -128 and lo.max() <= 127


def test_q16_representation_error():
    v = _grid()
    hi, lo = _limbs(v)
    err = np.abs(v.astype(np.float64) - (256 * hi + lo) / QS)
    assert err.max() <= 1.0 / (2 * QS) + 1e-12          # 1/65024 = 1.54e-5


def test_q16_negation_is_exact():
    # the -Ws rows use fma(s, -32512, M + 128): limbs of -x, never the unrepresentable -(-128)
    v = _grid()
    hi, lo = _limbs(v)
    nhi, nlo = _limbs(v, -QS)
    assert np.array_equal(256 * nhi + nlo, -(256 * hi + lo))


def test_three_product_form_bound():
    rng = np.random.default_rng(7)
    v = rng.uniform(-1, 1, 100000).astype(np.float32)
    w = rng.uniform(-1, 1, 100000).astype(np.float32)
    hv, lv = _limbs(v)
    hw, lw = _limbs(w)
    approx = (65536.0 * hv * hw + 256.0 * (hv * lw + lv * hw)) / QS**2
    exact = v.astype(np.float64) * w.astype(np.float64)
    # |v - xv/QS| <= 1/65024 each, plus the dropped lo.lo' <= 128^2 / QS^2
    bound = 2.0 / (2 * QS) + (1.0 / (2 * QS)) ** 2 + 128.0**2 / QS**2
    assert np.abs(approx - exact).max() <= bound
    # the dropped lo.lo' term is zero-mean (lo symmetric): no coherent bias over many atoms
    assert abs(np.mean(lv * lw)) / 128.0**2 < 0.01


def test_int32_accumulation_bound():
    # per atom: HH <= 2 * 127^2 (two MMAs), X <= 4 * 127 * 128; chunks of <= 32768 atoms (kI8MaxChunk)
    assert 2 * 127 * 127 * 32768 < 2**31
    assert 4 * 127 * 128 * 32768 < 2**31
