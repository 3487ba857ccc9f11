"""Seeded synthetic inputs shared by the CUDA path, the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no phases, no q vectors, no intensities,
no statistics).  It only draws atom positions / form factors and describes the five
BASELINE.json workloads.  Both sides (oracle/ and the CUDA library) consume its arrays.

Workload recipe:
  * reduced Lennard-Jones units (sigma = 1), number density 0.8 for configs 2-5, the reduced analogue
    of the paper's liquid-Ar box (rho*sigma^3 = 0.762);
  * frame 0 uniform in [0, L)^3; Brownian frames add N(0, 2 D dt) per axis (variance)
    and wrap back into the box;
  * two-species configs: f_j = 1 for even j, f_j = 2 for odd j;
  * config 4: 20 independent uniform (ideal-gas) frames;
  * seed = 220413241 + config number, numpy PCG64.
The paper's own trajectories (LJ Ar, TIP4P/2005 water) are not available; these synthetic inputs
stand in for them (same N/L/density class, no structure: S(q) = 1).
"""
from __future__ import annotations

import dataclasses
import numpy as np

SEED_BASE = 220413241

# Ewald-detector workload parameters for config 4 (reading B):
# wavelength 1.0 Angstrom expressed in sigma = 3.405 Angstrom units, 1024 x 1024 lon-lat pixels.
EWALD_WAVELENGTH_SIGMA = 1.0 / 3.405
EWALD_PITCH_RAD = 1.916535e-3
EWALD_QMAX = 8.0 * np.pi  # = 4 * 2 pi / sigma, the shell range used for config-4 binning


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    N: int
    L: float
    T: int
    D: float            # diffusion coefficient (0 => independent uniform frames)
    dt: float
    n_plane: int        # lattice plane n x n (0 => Ewald detector)
    two_species: bool
    dtype: str          # "f32" | "f64": positions / q / form factors as handed to the library
    lags: tuple         # g2 lags (Eq. 14)
    windows: tuple      # XSVS exposure windows in frames (Eq. 15)
    n_bins: int = 32
    seed: int = 0
    detector: int = 0   # Ewald detector pixels per side (config 4)


def _L(N, density=0.8):
    return float((N / density) ** (1.0 / 3.0))


CONFIGS = {
    "c1": Config("c1", 1000, 10.0, 1, 0.0, 1.0, 64, False, "f64", (), (), seed=SEED_BASE + 1),
    "c2": Config("c2", 32000, _L(32000), 100, 0.05, 1.0, 256, False, "f32",
                 tuple(range(1, 51)), (1, 2, 4, 8, 16, 32, 64), seed=SEED_BASE + 2),
    "c3": Config("c3", 262144, _L(262144), 1000, 0.02, 1.0, 512, True, "f32",
                 tuple(range(1, 201)), (1, 2, 4, 8, 16, 32, 64, 128), seed=SEED_BASE + 3),
    "c4": Config("c4", 1048576, _L(1048576), 20, 0.0, 1.0, 0, False, "f32", (), (),
                 seed=SEED_BASE + 4, detector=1024),
    "c5": Config("c5", 524288, _L(524288), 200, 0.05, 0.1, 512, True, "f32",
                 (), (1, 2, 4, 8, 16, 32, 64, 128), seed=SEED_BASE + 5),
}


def scaled(cfg: Config, **kw) -> Config:
    """Same workload class with some sizes replaced (used for small parity cases)."""
    d = dataclasses.asdict(cfg)
    d.update(kw)
    if "N" in kw and "L" not in kw and cfg.name != "c1":
        d["L"] = _L(d["N"])
    return Config(**d)


def rng_for(cfg: Config, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([cfg.seed, stream]))


def _wrap(x, L):
    # generator-side periodic wrap (keeps generated coordinates inside [0, L))
    x = x - L * np.floor(x / L)
    x[x >= L] = 0.0
    return x


def _cast(x64, L, dtype):
    if dtype == "f64":
        return x64.copy()
    x = x64.astype(np.float32)
    # rounding to fp32 may land exactly on L: re-wrap in fp32
    x[x >= np.float32(L)] = np.float32(0.0)
    return x


def positions(cfg: Config, frames: int | None = None) -> np.ndarray:
    """Positions [T][N][3] in cfg.dtype, inside [0, L)^3.

    D > 0: frame 0 uniform, then Brownian steps with per-axis variance 2 D dt.
    D == 0: independent uniform frames (ideal gas)."""
    T = cfg.T if frames is None else frames
    rng = rng_for(cfg)
    out = np.empty((T, cfg.N, 3), dtype=np.float32 if cfg.dtype == "f32" else np.float64)
    x = rng.uniform(0.0, cfg.L, size=(cfg.N, 3))
    out[0] = _cast(x, cfg.L, cfg.dtype)
    sigma = np.sqrt(2.0 * cfg.D * cfg.dt)
    for t in range(1, T):
        if cfg.D > 0:
            x = _wrap(x + sigma * rng.standard_normal(size=(cfg.N, 3)), cfg.L)
        else:
            x = rng.uniform(0.0, cfg.L, size=(cfg.N, 3))
        out[t] = _cast(x, cfg.L, cfg.dtype)
    return out


def form_factors(cfg: Config) -> np.ndarray:
    f = np.ones(cfg.N, dtype=np.float64)
    if cfg.two_species:
        f[1::2] = 2.0
    return f.astype(np.float32 if cfg.dtype == "f32" else np.float64)


BASES = {
    "sc": [(0.0, 0.0, 0.0)],
    "bcc": [(0.0, 0.0, 0.0), (0.5, 0.5, 0.5)],
    "fcc": [(0.0, 0.0, 0.0), (0.5, 0.5, 0.0), (0.5, 0.0, 0.5), (0.0, 0.5, 0.5)],
}


def crystal(kind: str, n_cells: int, L: float, dtype: str = "f64") -> np.ndarray:
    """Perfect cubic crystal (SC/BCC/FCC) filling the periodic box: positions [N][3]."""
    a = L / n_cells
    idx = np.arange(n_cells, dtype=np.float64)
    cells = np.stack(np.meshgrid(idx, idx, idx, indexing="ij"), -1).reshape(-1, 3)
    pts = np.concatenate([(cells + np.array(b)) * a for b in BASES[kind]], 0)
    return _cast(pts, L, dtype)


def uniform_frame(seed: int, N: int, L: float, dtype: str = "f64") -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return _cast(rng.uniform(0.0, L, size=(N, 3)), L, dtype)


def pixel_subset(n_q: int, count: int, seed: int, include=()) -> np.ndarray:
    """Sorted, de-duplicated seeded subset of pixel indices (plus any forced ones)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pick = rng.choice(n_q, size=min(count, n_q), replace=False)
    return np.unique(np.concatenate([pick, np.asarray(include, dtype=np.int64)])).astype(np.int64)


def species_labels(N: int, n_species: int, seed: int) -> np.ndarray:
    """Seeded atom kinds in [0, n_species) (int32), for the q-dependent form-factor path."""
    rng = np.random.Generator(np.random.PCG64([seed, 77]))
    return rng.integers(0, n_species, N).astype(np.int32)


# Table 1 of the paper: one liquid-Ar frame, N = 4000 atoms in a cubic box of L = 59.19 Angstrom
# (PAPER.md:385), Algorithm 1 on an 81 x 81 x 81 reciprocal-lattice grid, h, k, l in [-40, 40].
# The Ar configuration itself is not available: a seeded uniform frame of the same N, L stands in for it.
TABLE1 = dict(N=4000, L=59.19, n=81, seed=SEED_BASE + 10)


def gaussian_form_factor_coefficients(n_species: int):
    """Synthetic Gaussian-sum coefficients (a, b, c) per kind for f(q) = c + sum a_i exp(-b_i (q / 4 pi)^2)
    (the PAPER.md:94-95 form; NOT tabulated element data -- values made up for testing, in sigma units)."""
    table = [([9.0, 6.0, 2.0], [1.5, 12.0, 45.0], 1.0),
             ([3.0, 2.0], [4.0, 25.0], 0.3),
             ([0.5], [8.0], 0.0),
             ([5.0, 1.0, 0.5, 0.25], [2.0, 8.0, 30.0, 90.0], 0.2)]
    return [table[s % len(table)] for s in range(n_species)]
