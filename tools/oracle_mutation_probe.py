"""Mutation probe of the oracle's pins (test infrastructure, not the product).

Replaces ONE oracle function by a plausible mistake and runs tests/test_oracle_pins.py; every mutation must fail at
least one pin.  Usage: python tools/oracle_mutation_probe.py <mutation>   (mutations: see MUTATIONS; "all" loops)
"""
import math, subprocess, sys

import numpy as np
import pytest
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle

MUTATIONS = ["g2", "xsvs", "radial", "amp", "isf_conj", "isf_T", "ewald_sign", "ewald_swap", "lbins_round", "sq_norm",
             "ff_s", "lq_scale", "lq_axes", "hist_round", "hist_mean_all", "species_sign", "fft_flip",
             "f_squared", "isf_norm"]
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which == "all":
    bad = []
    for m in MUTATIONS:
        r = subprocess.run([sys.executable, __file__, m], capture_output=True, text=True)
        print(f"{m:12s} {'caught' if r.returncode else 'SURVIVED'}: {r.stdout.strip().splitlines()[-1]}")
        bad += [] if r.returncode else [m]
    sys.exit(1 if bad else 0)
orig = {k: getattr(oracle, k) for k in dir(oracle)}
o = orig
if which == "g2":
    def g2(I, lags):
        I = np.asarray(I, float); T = I.shape[0]; out = []
        for tau in lags:
            a, b = I[:T - tau], I[tau:]
            out.append((a * b).mean(0) / (a.mean(0) * b.mean(0)))
        return np.array(out)
    oracle.g2 = g2
elif which == "xsvs":
    def xs(I, bins, n_bins, windows, per_window=False):
        I = np.asarray(I, float); T = I.shape[0]; out = np.full((len(windows), n_bins), np.nan)
        for wi, W in enumerate(windows):
            S = -(-T // W)
            IW = np.stack([I[s*W:(s+1)*W].sum(0) for s in range(S)])
            for b in range(n_bins):
                x = IW[:, bins == b]
                if x.shape[1] < 2: continue
                out[wi, b] = (x.var(1, ddof=1) / x.mean(1) ** 2).mean()
        return out
    oracle.xsvs_beta = xs
elif which == "radial":
    def rb(q, q_max, n_bins=32):
        q = np.asarray(q, float); r = (q * q).sum(1)
        b = np.floor(r / q_max**2 * n_bins).astype(np.int64); b[(r >= q_max**2) | (r == 0)] = -1
        return b.astype(np.int32)
    oracle.radial_bins = rb
elif which == "amp":
    oracle.amplitude = lambda *a, **k: np.conj(orig["amplitude"](*a, **k))
    oracle.amplitudes = lambda *a, **k: np.conj(orig["amplitudes"](*a, **k))
elif which == "isf_conj":
    def isf(A, lags, S2):
        A = np.asarray(A, complex); T = A.shape[0]
        return np.stack([(np.conj(A[:T-t]) * A[t:]).sum(0) / (T-t) / S2 for t in lags])
    oracle.isf = isf
elif which == "isf_T":
    def isf(A, lags, S2):
        A = np.asarray(A, complex); T = A.shape[0]
        return np.stack([(A[:T-t] * np.conj(A[t:])).sum(0) / T / S2 for t in lags])
    oracle.isf = isf
elif which == "ewald_sign":
    oracle.ewald_q = lambda *a: -o["ewald_q"](*a)
elif which == "ewald_swap":
    def e(wl, npx, npy, pitch):
        q = o["ewald_q"](wl, npx, npy, pitch); return q[:, [1, 0, 2]]
    oracle.ewald_q = e
elif which == "lbins_round":
    def lb(n, n_bins=32, h0=None, k0=None):
        h0 = -(n//2) if h0 is None else h0; k0 = -(n//2) if k0 is None else k0
        w = n // (2*n_bins); out = np.full(n*n, -1, np.int32); lim = (n//2)**2
        for ih in range(n):
            for ik in range(n):
                h, k = h0+ih, k0+ik; r2 = h*h+k*k
                if r2 == 0 or r2 >= lim: continue
                out[ih*n+ik] = min(int(round(math.sqrt(r2) / w)), n_bins-1)
        return out
    oracle.lattice_bins = lb
elif which == "sq_norm":
    oracle.structure_factor_shells = lambda I, f, N, bins, nb: oracle.shell_mean(I, bins, nb) / float(N)
elif which == "lattice_q_sign":
    oracle.lattice_q = lambda *a, **k: -o["lattice_q"](*a, **k) * 1.0000001
elif which == "ff_s":          # form factor in |q| instead of s = |q| / (4 pi)
    def ff(q, a, b, c):
        q = np.asarray(q, float); s2 = (q * q).sum(1)
        return float(c) + sum(float(ai) * np.exp(-float(bi) * s2) for ai, bi in zip(a, b))
    oracle.form_factor_gaussian = ff
elif which == "lq_scale":      # q in units of 1/L instead of 2 pi / L
    oracle.lattice_q = lambda L, *a, **k: o["lattice_q"](L, *a, **k) / (2 * np.pi)
elif which == "lq_axes":       # pixel index ik * n_h + ih instead of ih * n_k + ik
    def lq(L, h0, n_h, k0, n_k, **k):
        q = o["lattice_q"](L, h0, n_h, k0, n_k, **k)
        return q.reshape(n_h, n_k, 3).transpose(1, 0, 2).reshape(-1, 3)
    oracle.lattice_q = lq
elif which == "hist_round":    # nearest-bin instead of floor histogram
    def sh(I, bins, n_bins, M, n_hist, kappa_max, edge_tol=1e-9):
        c, a = o["speckle_histogram"](I, bins, n_bins, M, n_hist, kappa_max, edge_tol)
        return np.roll(c, 1, axis=1), a
    oracle.speckle_histogram = sh
elif which == "hist_mean_all": # kappa normalised by the mean over all snapshots, not per snapshot
    def sh(I, bins, n_bins, M, n_hist, kappa_max, edge_tol=1e-9):
        I = np.asarray(I, float); S = I.shape[0] // M
        IM = I[: S * M].reshape(S, M, -1).sum(1)
        c = np.zeros((n_bins, n_hist), np.int64)
        for b in range(n_bins):
            x = IM[:, bins == b]
            if x.size == 0 or not x.mean() > 0: continue
            h = np.floor(x / x.mean() * n_hist / kappa_max).astype(int).ravel()
            for v in h[h < n_hist]: c[b, v] += 1
        return c, np.zeros((n_bins, n_hist + 1), np.int64)
    oracle.speckle_histogram = sh
elif which == "species_sign":  # e^{+iq.r} in the species amplitude
    def si(pos, species, fq, q, L, amp=False):
        r = o["species_intensity"](pos, species, fq, q, L, amp=amp)
        return np.conj(r) if amp else r
    oracle.species_intensity = si
elif which == "fft_flip":
    oracle.fft_intensity = lambda *a, **k: np.flip(o["fft_intensity"](*a, **k), -1)
elif which == "f_squared":     # f_j^2 instead of f_j inside the amplitude (Eq. 7)
    def amp(pos, f, q, L):
        return o["amplitude"](pos, None if f is None else np.asarray(f, float) ** 2, q, L)
    def inten(pos, f, q, L):
        return o["intensity"](pos, None if f is None else np.asarray(f, float) ** 2, q, L)
    oracle.amplitude, oracle.intensity = amp, inten
elif which == "isf_norm":      # ISF normalised by (sum f)^2 instead of sum f^2
    oracle.isf = lambda A, lags, S2: o["isf"](A, lags, S2 * 2.0)
else:
    sys.exit(f"unknown mutation {which}")
sys.exit(pytest.main(["-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider", "tests/test_oracle_pins.py"]))
