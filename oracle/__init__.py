"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct FP64 CPU implementation of what the CUDA path computes, written from
PAPER.md (arXiv 2204.13241).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import it.  It shares no code with
``paper_2204_13241_b200`` (neither imports the other); both consume only ``xpcs_inputs``.

Contents (each function cites the passage it follows):
  * liboracle.so (oracle.c): the direct sum Eq.(7)/(8) and the pair sum Eq.(2), FP64, OpenMP over q.
  * lattice_q       -- reciprocal-lattice q = (2 pi / L) (m0 + h ma + k mb), Algorithm 1 step 1.
  * ewald_q         -- Ewald-sphere detector q = k (u - z), Eq.(1) + Fig. 5 (reading R4).
  * g2              -- Eq.(14) literal estimator (reading R6).
  * amplitudes / isf -- Eq.(7) per frame, Eq.(22) intermediate scattering function.
  * lattice_bins / radial_bins / shell_mean / structure_factor_shells -- ring average, Eq.(12).
  * xsvs_beta       -- Eq.(15) + Eq.(17), per-snapshot then averaged.
  * lattice_volume_q -- 3-D reciprocal-lattice block (Table 1's 81^3 grid).
  * species_intensity / pair_sum_species -- Eq.(2)/(7) with q-dependent form factors f_s(q).
  * form_factor_gaussian -- f(q) as a sum of Gaussians.
  * fft_intensity / fft_block -- Algorithm 2, the FFT-based method, FP64 numpy FFT.
  * speckle_histogram / erlang_pdf -- kappa = I_M / <I_M>_ring statistics, Eq.(37)-(38).
Every function is pinned by tests/test_oracle_pins.py (no function here is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", _SRC, "-o", _LIB, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        L.oracle_amplitude.argtypes = [dp, i64, dp, dp, i64, ctypes.c_double, dp, dp]
        L.oracle_intensity.argtypes = [dp, i64, dp, dp, i64, i64, ctypes.c_double, dp]
        L.oracle_pair_sum.argtypes = [dp, i64, dp, dp, i64, ctypes.c_double, dp]
        ip = ctypes.POINTER(ctypes.c_int32)
        L.oracle_species.argtypes = [dp, i64, ip, dp, dp, i64, i64, ctypes.c_double, ctypes.c_int, dp]
        L.oracle_pair_sum_species.argtypes = [dp, i64, ip, dp, dp, i64, ctypes.c_double, dp]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def threads() -> int:
    return int(lib().oracle_max_threads())


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's loops (timing on all host cores)."""
    lib().oracle_set_threads(int(n))


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f(f):
    if f is None:
        return None, None
    return _d(f)


# ----------------------------------------------------------------------------------------------
# q geometry
# ----------------------------------------------------------------------------------------------
def lattice_q(L, h0, n_h, k0, n_k, m0=(0, 0, 0), ma=(1, 0, 0), mb=(0, 1, 0)) -> np.ndarray:
    """Algorithm 1 step 1: q on the reciprocal lattice of the cubic box, components
    integer multiples of 2 pi / L.  Pixel (ih, ik) -> h = h0 + ih, k = k0 + ik,
    q = (2 pi / L) (m0 + h ma + k mb), pixel index ih * n_k + ik.  FP64."""
    h = np.arange(h0, h0 + n_h, dtype=np.float64)[:, None, None]
    k = np.arange(k0, k0 + n_k, dtype=np.float64)[None, :, None]
    m = (np.asarray(m0, np.float64)[None, None, :] + h * np.asarray(ma, np.float64)[None, None, :]
         + k * np.asarray(mb, np.float64)[None, None, :])
    return (2.0 * np.pi / L) * m.reshape(-1, 3)


def lattice_volume_q(L, h0, n_h, k0, n_k, l0, n_l, m0=(0, 0, 0), ma=(1, 0, 0), mb=(0, 1, 0), mc=(0, 0, 1)):
    """Algorithm 1 step 1 on a 3-D block of the reciprocal lattice (the 81 x 81 x 81 grid of
    Table 1): q = (2 pi / L) (m0 + h ma + k mb + l mc), index ((il * n_h) + ih) * n_k + ik, i.e.
    the l-planes of lattice_q stacked.  FP64."""
    planes = [lattice_q(L, h0, n_h, k0, n_k, tuple(np.asarray(m0) + (l0 + il) * np.asarray(mc)), ma, mb)
              for il in range(n_l)]
    return np.concatenate(planes, 0)


def form_factor_gaussian(q, a, b, c):
    """Atomic form factor as a sum of Gaussians ('well parameterized by a sum of Gaussians'):
    f(q) = c + sum_i a_i exp(-b_i s^2) with s = |q| / (4 pi) (= sin(theta) / lambda).  q [n_q][3] -> [n_q] FP64."""
    q = np.asarray(q, dtype=np.float64)
    s2 = (q * q).sum(1) / (4.0 * np.pi) ** 2
    out = np.full(q.shape[0], float(c))
    for ai, bi in zip(a, b):
        out += float(ai) * np.exp(-float(bi) * s2)
    return out


def plane_grid(n):
    """The configs' detector plane: h, k in [-n/2, n/2 - 1], l = 0 (reading R7)."""
    return dict(h0=-(n // 2), n_h=n, k0=-(n // 2), n_k=n)


def ewald_q(wavelength, npx, npy, pitch) -> np.ndarray:
    """Detector pixels on the Ewald sphere (Eq.(1): |k_i| = |k_f| = 2 pi / lambda,
    q = k_f - k_i; Fig. 5 'spherical slice ... to keep |k_f| = |k_i|').
    Reading R4: k_i = k z, pixel (i, j) at lon-lat angles
    psi_x = (i - (npx-1)/2) pitch, psi_y = (j - (npy-1)/2) pitch,
    u = (sin psi_x cos psi_y, sin psi_y, cos psi_x cos psi_y), q = k (u - z).  FP64, index i*npy + j."""
    k = 2.0 * np.pi / wavelength
    px = (np.arange(npx, dtype=np.float64) - (npx - 1) / 2.0) * pitch
    py = (np.arange(npy, dtype=np.float64) - (npy - 1) / 2.0) * pitch
    PX, PY = np.meshgrid(px, py, indexing="ij")
    u = np.stack([np.sin(PX) * np.cos(PY), np.sin(PY), np.cos(PX) * np.cos(PY)], -1)
    q = k * (u - np.array([0.0, 0.0, 1.0]))
    return q.reshape(-1, 3)


# ----------------------------------------------------------------------------------------------
# the direct method
# ----------------------------------------------------------------------------------------------
def amplitude(pos, f, q, L):
    """Eq.(7): complex p^e(q) for one frame [N][3] (positions promoted to FP64)."""
    pos, pp = _d(pos)
    N = pos.shape[0]
    f, fp = _f(f)
    q, qp = _d(q)
    n_q = q.shape[0]
    re = np.zeros(n_q)
    im = np.zeros(n_q)
    lib().oracle_amplitude(pp, N, fp, qp, n_q, float(L), _d(re)[1], _d(im)[1])
    return re + 1j * im


def intensity(pos, f, q, L):
    """Eq.(8) I(q,t) = |p^e(q,t)|^2 for positions [T][N][3] (or [N][3]); returns [T][n_q]."""
    pos = np.asarray(pos)
    if pos.ndim == 2:
        pos = pos[None]
    pos, pp = _d(pos)
    T, N = pos.shape[0], pos.shape[1]
    f, fp = _f(f)
    q, qp = _d(q)
    n_q = q.shape[0]
    out = np.zeros((T, n_q))
    lib().oracle_intensity(pp, N, fp, qp, n_q, T, float(L), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def amplitudes(pos, f, q, L):
    """Eq.(7) for every frame: complex p^e [T][n_q] (positions [T][N][3] or [N][3])."""
    pos = np.asarray(pos)
    if pos.ndim == 2:
        pos = pos[None]
    return np.stack([amplitude(p, f, q, L) for p in pos])


def isf(A, lags, S2):
    """Eq.(22): F(q, tau) = <p(t) p*(t + tau)>_t / sum_j f_j^2, the time average taken over the
    T - tau available pairs.  A complex [T][n_q] -> complex [n_lags][n_q]."""
    A = np.asarray(A, dtype=np.complex128)
    T = A.shape[0]
    out = np.empty((len(lags), A.shape[1]), dtype=np.complex128)
    for i, tau in enumerate(lags):
        out[i] = (A[: T - tau] * np.conj(A[tau:])).sum(0) / (T - tau) / S2
    return out


def _species_args(species, fq, n_q):
    sp = np.ascontiguousarray(species, dtype=np.int32)
    fq = np.ascontiguousarray(fq, dtype=np.float64)
    assert fq.ndim == 2 and fq.shape[1] == n_q and sp.min() >= 0 and sp.max() < fq.shape[0]
    return sp, sp.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), fq, fq.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def species_intensity(pos, species, fq, q, L, amp=False):
    """Eq.(2)/(7)/(8) with q-dependent form factors f_{s(j)}(q): p = sum_j f_{s(j)}(q) e^{-i q.r_j},
    I = |p|^2.  pos [T][N][3] (or [N][3]), species [N] int, fq [n_species][n_q].  Returns I [T][n_q] or, with
    amp=True, complex p [T][n_q]."""
    pos = np.asarray(pos)
    if pos.ndim == 2:
        pos = pos[None]
    pos, pp = _d(pos)
    T, N = pos.shape[0], pos.shape[1]
    q, qp = _d(q)
    n_q = q.shape[0]
    sp, spp, fq, fqp = _species_args(species, fq, n_q)
    out = np.zeros((T, n_q, 2) if amp else (T, n_q))
    lib().oracle_species(pp, N, spp, fqp, qp, n_q, T, float(L), 1 if amp else 0,
                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out[..., 0] + 1j * out[..., 1] if amp else out


def pair_sum_species(pos, species, fq, q, L):
    """Eq.(2) with f_i(q): the O(N^2) pair sum (tiny N only)."""
    pos, pp = _d(pos)
    N = pos.shape[0]
    q, qp = _d(q)
    n_q = q.shape[0]
    sp, spp, fq, fqp = _species_args(species, fq, n_q)
    out = np.zeros(n_q)
    lib().oracle_pair_sum_species(pp, N, spp, fqp, qp, n_q, float(L), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def pair_sum_intensity(pos, f, q, L):
    """Eq.(2): I(q) by the O(N^2) double sum over atom pairs (tiny N only)."""
    pos, pp = _d(pos)
    N = pos.shape[0]
    f, fp = _f(f)
    q, qp = _d(q)
    n_q = q.shape[0]
    out = np.zeros(n_q)
    lib().oracle_pair_sum(pp, N, fp, qp, n_q, float(L), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


# ----------------------------------------------------------------------------------------------
# speckle statistics
# ----------------------------------------------------------------------------------------------
def g2(I, lags):
    """Eq.(14), literal estimator (R6):
    num(tau) = 1/(T - tau) sum_{t=0}^{T-1-tau} I_t I_{t+tau},  den = ((1/T) sum_t I_t)^2,
    g2 = num / den; NaN where den == 0.  I [T][n_q] -> [n_lags][n_q] FP64."""
    I = np.asarray(I, dtype=np.float64)
    T = I.shape[0]
    mean = I.sum(0) / T
    den = mean * mean
    out = np.empty((len(lags), I.shape[1]))
    for i, tau in enumerate(lags):
        num = (I[: T - tau] * I[tau:]).sum(0) / (T - tau)
        with np.errstate(divide="ignore", invalid="ignore"):
            out[i] = np.where(den > 0, num / np.where(den > 0, den, 1.0), np.nan)
    return out


def lattice_bins(n, n_bins=32, h0=None, k0=None):
    """q-ring membership q - dq/2 <= |q| < q + dq/2 on the n x n lattice plane,
    in exact integer arithmetic (R8): radius unit w = n / (2 n_bins) pixels,
    b = floor(sqrt(h^2 + k^2) / w) = isqrt(h^2 + k^2) // w; q = 0 and h^2 + k^2 >= (n/2)^2 excluded (-1)."""
    h0 = -(n // 2) if h0 is None else h0
    k0 = -(n // 2) if k0 is None else k0
    w = n // (2 * n_bins)
    assert w * 2 * n_bins == n
    out = np.full(n * n, -1, dtype=np.int32)
    lim = (n // 2) ** 2
    for ih in range(n):
        h = h0 + ih
        for ik in range(n):
            k = k0 + ik
            r2 = h * h + k * k
            if r2 == 0 or r2 >= lim:
                continue
            out[ih * n + ik] = math.isqrt(r2) // w
    return out


def radial_bins(q, q_max, n_bins=32):
    """Shells of |q| for an explicit q list (config 4): b = floor(|q| / q_max * n_bins) in FP64 from the
    (fp32) q array; |q| >= q_max and q = 0 excluded (-1)."""
    q = np.asarray(q, dtype=np.float64)
    r = np.sqrt((q * q).sum(1))
    b = np.floor(r / q_max * n_bins).astype(np.int64)
    b[(r >= q_max) | (r == 0.0)] = -1
    return b.astype(np.int32)


def shell_mean(values, bins, n_bins):
    """Average over all detector pixels in each ring, per row; non-finite values
    (e.g. g2 of a zero-mean pixel) are excluded; empty ring -> NaN.  values [rows][n_q] -> [rows][n_bins]."""
    v = np.asarray(values, dtype=np.float64)
    if v.ndim == 1:
        v = v[None]
    out = np.full((v.shape[0], n_bins), np.nan)
    for b in range(n_bins):
        sel = v[:, bins == b]
        for r in range(v.shape[0]):
            x = sel[r][np.isfinite(sel[r])]
            if x.size:
                out[r, b] = x.sum() / x.size
    return out


def structure_factor_shells(I, f, N, bins, n_bins):
    """Eq.(12)/(13): S(q,t) = I(q,t) / sum_j f_j^2, ring-averaged per frame -> [T][n_bins]."""
    s2 = float(N) if f is None else float(np.sum(np.asarray(f, np.float64) ** 2))
    return shell_mean(I, bins, n_bins) / s2


def xsvs_beta(I, bins, n_bins, windows, per_window=False):
    """Optical contrast vs exposure (XSVS).  Eq.(15) as a discrete, unnormalised
    sum over non-overlapping windows of W frames aligned at t = 0 (remainder dropped):
        I_W(q, s) = sum_{t = sW}^{sW + W - 1} I(q, t),  s = 0 .. floor(T/W) - 1;
    Eq.(17) per snapshot s and ring b with the population variance
        beta_{W,b,s} = (<I_W^2>_b - <I_W>_b^2) / <I_W>_b^2,
    then averaged over snapshots.  Returns [n_windows][n_bins] FP64 (NaN: empty ring)."""
    I = np.asarray(I, dtype=np.float64)
    T = I.shape[0]
    out = np.full((len(windows), n_bins), np.nan)
    detail = []
    for wi, W in enumerate(windows):
        S = T // W
        IW = I[: S * W].reshape(S, W, -1).sum(1)          # [S][n_q]
        row = []
        for b in range(n_bins):
            x = IW[:, bins == b]                           # [S][m0]
            m0 = x.shape[1]
            if m0 == 0:
                row.append(None)
                continue
            m1 = x.sum(1)
            m2 = (x * x).sum(1)
            mean = m1 / m0
            beta_s = (m2 / m0 - mean * mean) / (mean * mean)
            out[wi, b] = beta_s.sum() / S
            row.append(beta_s)
        detail.append(row)
    return (out, detail) if per_window else out


def speckle_histogram(I, bins, n_bins, M, n_hist, kappa_max, edge_tol=1e-9):
    """Speckle intensity statistics (PAPER.md:540-546 and Eq.(37)-(38)).  The incoherent
    superposition of M patterns (sum over intensity) of consecutive frames,
        I_M(q, s) = sum_{t=sM}^{sM+M-1} I(q, t),  s = 0 .. floor(T/M) - 1,
    normalised per ring b and snapshot s, kappa(q) = I_M(q, s) / <I_M(., s)>_{q in b} (the paper's
    kappa = I / <I>_q), is histogrammed over the ring's pixels and all snapshots into n_hist bins of width
    kappa_max / n_hist on [0, kappa_max) (kappa >= kappa_max dropped): h = floor(kappa * n_hist / kappa_max).
    Returns (counts int64 [n_bins][n_hist], ambiguous int64 [n_bins][n_hist + 1]) where ambiguous counts values
    whose kappa * n_hist / kappa_max lies within edge_tol (relative) of an integer edge e (slot e), the only
    decisions a different FP64 summation order of the ring mean could flip."""
    I = np.asarray(I, dtype=np.float64)
    T = I.shape[0]
    S = T // M
    IM = I[: S * M].reshape(S, M, -1).sum(1)                    # [S][n_q]
    counts = np.zeros((n_bins, n_hist), dtype=np.int64)
    amb = np.zeros((n_bins, n_hist + 1), dtype=np.int64)
    for b in range(n_bins):
        sel = IM[:, bins == b]                                   # [S][m0]
        if sel.shape[1] == 0:
            continue
        for s in range(S):
            x = sel[s]
            mean = x.sum() / x.size
            if not mean > 0:
                continue
            u = (x / mean) * n_hist / kappa_max
            for v in u:
                h = int(math.floor(v))
                if h < n_hist:
                    counts[b, h] += 1
                e = int(round(v))
                if abs(v - e) <= edge_tol * max(1.0, abs(v)) and e <= n_hist:
                    amb[b, e] += 1
    return counts, amb


def erlang_pdf(kappa, M):
    """Eq.(38): P_M(kappa) = M^M kappa^(M-1) exp(-M kappa) / (M-1)!  (M = 1: Eq.(37) exp(-kappa))."""
    kappa = np.asarray(kappa, dtype=np.float64)
    return M ** M * kappa ** (M - 1) * np.exp(-M * kappa) / math.factorial(M - 1)


# ----------------------------------------------------------------------------------------------
# Algorithm 2 (FFT-based method) -- SURVEY 8(f) rank 4, the paper's cross-check path
# ----------------------------------------------------------------------------------------------
def fft_kernel_width(L, n_grid, eta, k=0):
    """k = 'the nearest integer greater than 10 eta' in grid spacings, made odd so the k points
    nearest the origin are centred (reading R16); an explicit k > 0 is used as given (must be odd)."""
    if k <= 0:
        k = int(math.floor(10.0 * eta / (L / n_grid))) + 1
        if k % 2 == 0:
            k += 1
    assert k % 2 == 1
    return k


def _spread(pos, L, n_grid, eta, k):
    """Algorithm 2 steps 1-2: rho^eta on the n_grid^3 grid, each atom's Gaussian (Eq. 30) evaluated on the k x k x k
    grid points nearest to it (periodic wrap of the indices), grid point n at r = n L / n_grid."""
    d = L / n_grid
    rho = np.zeros((n_grid, n_grid, n_grid))
    c = (1.0 / (math.sqrt(2.0 * math.pi) * eta)) ** 3
    for r in np.asarray(pos, dtype=np.float64):
        idx = []
        for a in range(3):
            u = r[a] / d
            n0 = int(math.floor(u - k / 2.0)) + 1              # the k integers nearest to u
            idx.append(np.arange(n0, n0 + k))
        X, Y, Z = np.meshgrid(*idx, indexing="ij")
        r2 = (X * d - r[0]) ** 2 + (Y * d - r[1]) ** 2 + (Z * d - r[2]) ** 2
        np.add.at(rho, (X % n_grid, Y % n_grid, Z % n_grid), c * np.exp(-r2 / (2.0 * eta * eta)))
    return rho


def fft_intensity(pos, L, n_grid, eta, k=0, f=1.0):
    """Algorithm 2 for one frame [N][3]: rho^eta (steps 1-2), p^eta = FFT (step 3, with the
    e^{-i q.r} sign of Eq. 31: numpy's forward transform), f^eta = FFT of the truncated Gaussian centred at the origin
    (step 4), I = f^2 |p^eta|^2 / |f^eta|^2 (Eq. 35, step 5).  Returns I on the full FFT grid [n][n][n], axis index
    m <-> frequency h = m (m < n/2) or m - n; q = (2 pi / L)(h, k, l).  FP64."""
    k = fft_kernel_width(L, n_grid, eta, k)
    P = np.fft.fftn(_spread(pos, L, n_grid, eta, k))
    G = np.fft.fftn(_spread(np.zeros((1, 3)), L, n_grid, eta, k))
    return f * f * np.abs(P) ** 2 / np.abs(G) ** 2


def fft_block(I_full, h0, n_h, k0, n_k, l0, n_l):
    """Block of a full FFT-grid array in (l, h, k) output order (as xpcs_qvolume / lattice_volume_q): entry
    [il][ih][ik] = I at frequencies (h0 + ih, k0 + ik, l0 + il) on axes (x, y, z)."""
    n = I_full.shape[0]
    hh = (np.arange(h0, h0 + n_h)) % n
    kk = (np.arange(k0, k0 + n_k)) % n
    ll = (np.arange(l0, l0 + n_l)) % n
    return I_full[np.ix_(hh, kk, ll)].transpose(2, 0, 1).reshape(-1)
