"""GPU parity of the integer tensor engine (XPCS_ENGINE_TENSOR_I8: tcgen05 kind::i8, two int8 limbs per phasor
component, exact int32 accumulation) against the FP64 oracle, at the north_star per-pixel gate (R11), on
ragged tiles / chunks, per-atom and per-kind form factors, amplitudes, 3-D blocks, Bragg crystals and the full c2
workload (sampled pixels, all frames)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402
from _gates import assert_pixels, pixel_gate  # noqa: E402

DEV = "cuda"
I8 = xp.ENGINE_TENSOR_I8


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    xp.load()
    if not xp.engine_available(I8):
        pytest.skip("no tcgen05")
    yield
    xp.release()


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _grid_q(g):
    return oracle.lattice_q(g.L, g.h0, g.n_h, g.k0, g.n_k, tuple(g.m0), tuple(g.ma), tuple(g.mb))


@pytest.mark.parametrize("N,f_kind", [(9001, "two"), (777, "none"), (40000, "none")])
def test_i8_ragged_parity(N, f_kind):
    """Ragged tiles (n_h, n_k not multiples of 256 / 128), tilted plane, N not a multiple of the 32-atom stage,
    several atom chunks (N = 40000 > one 32768-atom chunk)."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=N, T=2)
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg) if f_kind == "two" else None
    g = xp.qgrid(cfg.L, -37, 300, -75, 150, m0=(0, 0, 2), ma=(1, 0, 0), mb=(0, 1, 1))
    I = xp.xpcs_intensity_grid(_t(pos), _t(f) if f is not None else None, g, engine=I8).cpu().numpy()
    ref = oracle.intensity(pos, f.astype(np.float64) if f is not None else None, _grid_q(g), cfg.L)
    ratio, worst = assert_pixels(I, ref, cfg.N, f"i8 ragged N={N}")
    print(f"i8 N={N} f={f_kind}: worst err/allowed {ratio:.3f}, max |dI|/N {worst:.2e}")


def test_i8_matches_split_fp16_engine_statistically():
    """Same input on both tensor engines: the difference is the int8 limb quantisation, rms ~ 3e-5 N per pixel."""
    cfg = xi.scaled(xi.CONFIGS["c2"], N=32000, T=4)
    pos = _t(xi.positions(cfg))
    g = xp.lattice_plane(cfg.L, 256)
    a = xp.xpcs_intensity_grid(pos, None, g, engine=I8, out_dtype=xp.F64).cpu().numpy()
    b = xp.xpcs_intensity_grid(pos, None, g, engine=xp.ENGINE_TENSOR, out_dtype=xp.F64).cpu().numpy()
    d = (a - b) / cfg.N
    rms = float(np.sqrt(np.mean(d * d)))
    assert rms < 8e-5, rms
    assert np.max(np.abs(d)) < 1e-3
    # the forward point is exact in both (all phases 0): I(0) = N^2
    c = (128 * 256 + 128)
    assert abs(a[0, c] - cfg.N ** 2) <= 1e-6 * cfg.N ** 2


def test_i8_amplitude_volume_and_species():
    cfg = xi.scaled(xi.CONFIGS["c2"], N=5003, T=2)
    pos = xi.positions(cfg)
    v = xp.qvolume(cfg.L, -40, 80, -30, 100, -2, 3, mc=(0, 0, 1))
    q = oracle.lattice_volume_q(cfg.L, -40, 80, -30, 100, -2, 3)
    A = xp.xpcs_intensity_volume(_t(pos), None, v, engine=I8, amplitude=True).cpu().numpy().astype(np.float64)
    ref = oracle.amplitudes(pos, None, q, cfg.L)
    err = np.abs(A[..., 0] + 1j * A[..., 1] - ref)
    assert np.max(err / (1e-3 * np.sqrt(cfg.N) + 1e-5 * np.abs(ref))) <= 1.0
    sp = xi.species_labels(cfg.N, 2, 3)
    coef = xi.gaussian_form_factor_coefficients(2)
    fq = np.stack([oracle.form_factor_gaussian(q, *coef[s]) for s in range(2)]).astype(np.float32)
    I = xp.xpcs_intensity_volume(_t(pos), None, v, species=sp, f_q=_t(fq), engine=I8).cpu().numpy()
    Iref = oracle.species_intensity(pos, sp, fq.astype(np.float64), q, cfg.L)
    counts = np.bincount(sp, minlength=2).astype(np.float64)
    S2 = (counts[:, None] * fq.astype(np.float64) ** 2).sum(0)
    assert np.max(np.abs(I - Iref) / (1e-3 * S2 + 1e-5 * Iref)) <= 1.0


@pytest.mark.parametrize("kind,n_cells,shift", [("fcc", 20, False), ("sc", 32, False), ("fcc", 20, True),
                                                 ("sc", 32, True), ("bcc", 16, True)])
def test_i8_bragg(kind, n_cells, shift):
    """Perfect crystals at c2/c3-class N, at the origin and rigidly shifted (PBC): I = N^2 on the
    crystal's reciprocal lattice within the per-pixel gate (|dI| <= 1e-3 N + 1e-5 I, R11), ~0 elsewhere.
    A crystal repeats few phasor values, so the integer engine's limb errors add coherently at its peaks; the
    bright-pixel recompute (k_fixup.cu) must bring them to the gate."""
    L = 40.0
    pos = xi.crystal(kind, n_cells, L, "f64")
    if shift:
        pos = np.mod(pos + np.array([3.3170, 11.0731, 27.6006]), L)
    pos = pos.astype(np.float32)
    N = pos.shape[0]
    n = 256
    I = xp.xpcs_intensity_grid(_t(pos[None]), None, xp.lattice_plane(L, n), engine=I8).cpu().numpy()[0].reshape(n, n)
    h = np.arange(-n // 2, n // 2)
    H, K = np.meshgrid(h, h, indexing="ij")
    if kind == "fcc":      # F = 1 + (-1)^(H+K) + (-1)^H + (-1)^K on l = 0: H, K both even
        peak = (H % (2 * n_cells) == 0) & (K % (2 * n_cells) == 0)
    elif kind == "bcc":    # F = 1 + (-1)^(H+K): H + K even
        peak = (H % n_cells == 0) & (K % n_cells == 0) & ((H // n_cells + K // n_cells) % 2 == 0)
    else:
        peak = (H % n_cells == 0) & (K % n_cells == 0)
    qp = (2 * np.pi / L) * np.stack([H[peak], K[peak], np.zeros(peak.sum())], -1).astype(np.float64)
    ref = oracle.intensity(pos.astype(np.float64), None, qp, L)[0]
    np.testing.assert_allclose(ref, float(N) ** 2, rtol=1e-6)     # the oracle's own Bragg pin at these positions
    assert_pixels(I[peak], ref, N, f"{kind}{n_cells} shift={shift} peaks")
    assert np.max(I[~peak]) < 1e-3 * N


def test_i8_config2_full_size_sampled():
    """Config 2 in the bench's launch configuration on the i8 engine (both frame batches of its plan): all 100
    frames x 1024 seeded pixels (1.0e5 pixel-frames, 1.6 % of the run) vs the oracle."""
    cfg = xi.CONFIGS["c2"]
    pos = xi.positions(cfg)
    g = xp.lattice_plane(cfg.L, cfg.n_plane)
    I = xp.xpcs_intensity_grid(_t(pos), None, g, engine=I8).cpu().numpy()
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(cfg.n_plane))
    pix = xi.pixel_subset(q.shape[0], 1024, 11, include=[128 * 256 + 128])
    ref = oracle.intensity(pos, None, q[pix], cfg.L)
    ratio, worst, _ = pixel_gate(I[:, pix], ref, cfg.N)
    print(f"c2 i8 sampled: worst err/allowed {ratio:.3f}, max |dI|/N {worst:.2e}")
    assert ratio <= 1.0


@pytest.mark.parametrize("N", [1, 2, 31, 33, 1025])
@pytest.mark.parametrize("shape", [(1, 1), (3, 200), (257, 129)])
def test_i8_edge_sizes(N, shape):
    """Degenerate and ragged sizes: a single atom (I = f^2 = 1 everywhere), N around the 32-atom stage, 1 x 1 and
    ragged planes beyond one 256 x 128 tile, far-from-origin indices (large phase turns)."""
    L = 11.0
    pos = xi.uniform_frame(3 + N, N, L, "f32")[None]
    n_h, n_k = shape
    g = xp.qgrid(L, -1000, n_h, 417, n_k, m0=(0, 0, -5))
    I = xp.xpcs_intensity_grid(_t(pos), None, g, engine=I8).cpu().numpy()
    ref = oracle.intensity(pos, None, _grid_q(g), L)
    assert_pixels(I, ref, N, f"i8 N={N} shape={shape}")
    if N == 1:
        np.testing.assert_allclose(I, 1.0, atol=3e-4)    # limb representation: |dp| <= ~1e-4 per real part


def test_i8_many_frames_batched():
    """More virtual frames than one 1-GiB scratch batch holds (the call splits them into several engine launches):
    sampled frames from the first, a middle and the last batch against the oracle, and the batches agree with a
    per-frame call on the same frames."""
    cfg = xi.scaled(xi.CONFIGS["c2"], N=1500, T=700)
    pos = xi.positions(cfg)
    g = xp.lattice_plane(cfg.L, 256)
    d = _t(pos)
    I = xp.xpcs_intensity_grid(d, None, g, engine=I8).cpu().numpy()
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(256))
    pix = xi.pixel_subset(q.shape[0], 256, 8)
    frames = [0, 350, 699]
    ref = oracle.intensity(pos[frames], None, q[pix], cfg.L)
    assert_pixels(I[frames][:, pix], ref, cfg.N, "i8 batched frames")
    one = xp.xpcs_intensity_grid(d[699:700], None, g, engine=I8).cpu().numpy()
    assert_pixels(one[0][pix], ref[2], cfg.N, "i8 single frame")


@pytest.mark.parametrize("shape", [(256, 256), (257, 129)])
@pytest.mark.parametrize("what", ["I32", "I64", "A32"])
def test_i8_direct_drain_equals_partial_fold(monkeypatch, shape, what):
    """With one atom chunk the integer engine writes the result from its drain; the partial-plane path (forced with
    XPCS_I8_DIRECT=0) folds the same fp32 amplitude in FP64 with k_amp_reduce: the two must agree bit for bit
    (intensity in fp32 and fp64, amplitude), including odd n_k (unaligned pixel pairs) and ragged tiles."""
    L = 17.0
    N = 3000
    pos = _t(xi.uniform_frame(91, N, L, "f32")[None].repeat(3, axis=0))
    n_h, n_k = shape
    g = xp.qgrid(L, -n_h // 2, n_h, -n_k // 2, n_k)

    def run():
        if what == "A32":
            return xp.xpcs_amplitude_grid(pos, None, g, engine=I8).cpu().numpy()
        return xp.xpcs_intensity_grid(pos, None, g, engine=I8,
                                      out_dtype=xp.F64 if what == "I64" else xp.F32).cpu().numpy()

    direct = run()
    monkeypatch.setenv("XPCS_I8_DIRECT", "0")
    folded = run()
    assert np.array_equal(direct, folded)


def test_i8_frame_split_plan_parity(monkeypatch):
    """Enough (tile, frame) units that the last wave of clusters is partial: the call splits the frames into two
    batches with their own atom chunking.  Both batches against the oracle, and against the unsplit plan
    (XPCS_I8_TAILSPLIT=0) within the limb-rounding difference of their chunk folds."""
    cfg = xi.scaled(xi.CONFIGS["c2"], N=6000, T=100)
    pos = xi.positions(cfg)
    g = xp.lattice_plane(cfg.L, 256)
    d = _t(pos)
    split = xp.xpcs_intensity_grid(d, None, g, engine=I8).cpu().numpy()
    monkeypatch.setenv("XPCS_I8_TAILSPLIT", "0")
    plain = xp.xpcs_intensity_grid(d, None, g, engine=I8).cpu().numpy()
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(256))
    pix = xi.pixel_subset(q.shape[0], 128, 5)
    frames = [0, 40, 99]
    ref = oracle.intensity(pos[frames], None, q[pix], cfg.L)
    assert_pixels(split[frames][:, pix], ref, cfg.N, "i8 split plan")
    assert_pixels(plain[frames][:, pix], ref, cfg.N, "i8 unsplit plan")
    assert np.max(np.abs(split - plain)) / cfg.N < 1e-5
