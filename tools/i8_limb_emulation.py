"""Numpy emulation of the integer engine's arithmetic (k_lattice_i8.cu), used to choose its design.

Emulates: exact 32-bit phase turns, conjugate row pairs around the tile centre c (rows c +- d, d half-integer),
the global rotation Gamma on W, Q16 limbs (x = rint(32512 v) = 256 hi + lo), exact integer sums HH and X (the
lo.lo' term dropped), and the conjugate-pair combination; against the exact amplitude (float64, same turns).
Prints the relative error of I at coherent pixels (q = 0 of random frames, Bragg peaks of perfect crystals with and
without a rigid shift) and the rms / max |dI| / N at random pixels of a random frame, for the variants:
  old   -- the round-1 design (rows h, complex MAC, no pairing): exact at phase 0 only
  conj  -- conjugate pairs, no rotation
  rot   -- conjugate pairs + the rotation on W (the shipped kernel)
Not a test: the GPU tests measure the kernel itself.  Usage: python tools/i8_limb_emulation.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import xpcs_inputs as xi  # noqa: E402

QS = 32512.0
GAMMA = 0x3147AE14 / 2.0 ** 32


def limbs(v):
    x = np.rint(QS * v).astype(np.int64)
    hi = np.floor_divide(x + 128, 256)
    return hi, x - 256 * hi


def rdot(a, w):
    ha, la = limbs(a)
    hw, lw = limbs(w)
    return (65536.0 * (ha * hw).sum() + 256.0 * (ha * lw + la * hw).sum()) / QS ** 2


def amp(variant, tha, thb, th0, h, k, c):
    if variant == "old":
        px, pw = 2 * np.pi * ((h * tha) % 1.0), 2 * np.pi * ((th0 + k * thb) % 1.0)
        a, b, wr, wi = np.cos(px), np.sin(px), np.cos(pw), np.sin(pw)
        return complex(rdot(a, wr) - rdot(b, wi), rdot(a, wi) + rdot(b, wr))
    g = GAMMA if variant == "rot" else 0.0
    d = abs(h - c)
    px, pw = 2 * np.pi * ((d * tha) % 1.0), 2 * np.pi * ((th0 + k * thb + c * tha + g) % 1.0)
    a, b, wr, wi = np.cos(px), np.sin(px), np.cos(pw), np.sin(pw)
    AR, AI, BR, BI = rdot(a, wr), rdot(a, wi), rdot(b, wr), rdot(b, wi)
    q = complex(AR - BI, AI + BR) if h > c else complex(AR + BI, AI - BR)
    return q * np.exp(-2j * np.pi * g)


def exact(tha, thb, th0, h, k):
    return np.exp(2j * np.pi * ((h * tha + k * thb + th0) % 1.0)).sum()


def turns(pos, L):
    X = np.mod(np.rint(pos * (2.0 ** 32 / L)), 2.0 ** 32) / 2.0 ** 32
    return X[:, 0], X[:, 1], np.zeros(len(X))


def main():
    rng = np.random.default_rng(11)
    variants = ["old", "conj", "rot"]
    L = 40.0
    print("relative error of I at q = 0 (random frame, N = 32000), tile centres -0.5 (n = 256) and 127.5 (n = 512):")
    tha, thb, th0 = turns(rng.uniform(0, L, (32000, 3)), L)
    for c in (-0.5, 127.5):
        I0 = abs(exact(tha, thb, th0, 0, 0)) ** 2
        print("  c =", c, {v: f"{abs(abs(amp(v, tha, thb, th0, 0, 0, c)) ** 2 / I0 - 1):.1e}" for v in variants})
    print("max relative error of I at Bragg peaks (n = 256 plane, c = -0.5):")
    for kind, nc in [("fcc", 20), ("sc", 32), ("sc", 20)]:
        for shift in (False, True):
            base = xi.crystal(kind, nc, L, "f64")
            pos = np.mod(base + (rng.uniform(0, L, 3) if shift else 0.0), L).astype(np.float32).astype(np.float64)
            tha, thb, th0 = turns(pos, L)
            period = 2 * nc if kind == "fcc" else nc
            hs = [h for h in range(-128, 128) if h % period == 0]
            worst = {v: 0.0 for v in variants}
            for h in hs:
                for k in hs[:3]:
                    I0 = abs(exact(tha, thb, th0, h, k)) ** 2
                    for v in variants:
                        worst[v] = max(worst[v], abs(abs(amp(v, tha, thb, th0, h, k, -0.5)) ** 2 / I0 - 1))
            print(f"  {kind}{nc}{' shifted' if shift else ''}:", {v: f"{e:.1e}" for v, e in worst.items()})
    print("random pixels of a random frame (N = 32000): rms and max |dI| / N")
    tha, thb, th0 = turns(rng.uniform(0, L, (32000, 3)), L)
    for v in variants:
        e = []
        for h in range(-120, 128, 13):
            for k in range(-120, 128, 17):
                if h == 0 and k == 0:
                    continue
                e.append((abs(amp(v, tha, thb, th0, h, k, -0.5)) ** 2 - abs(exact(tha, thb, th0, h, k)) ** 2) / 32000)
        e = np.array(e)
        print(f"  {v}: rms {np.sqrt((e * e).mean()):.2e}, max {np.abs(e).max():.2e}")


if __name__ == "__main__":
    main()
