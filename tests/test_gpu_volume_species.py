"""GPU parity of SURVEY 8(f) rank 3: 3-D reciprocal-lattice blocks (Algorithm 1 step 1 on a q volume, Table 1's
81^3 grid) and q-dependent atomic form factors f_s(q) (Eq. 2), through the C ABI,
against the FP64 oracle on the same seeded inputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402
from _gates import assert_pixels  # noqa: E402

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


def _vol_q(v):
    p = v.plane
    return oracle.lattice_volume_q(p.L, p.h0, p.n_h, p.k0, p.n_k, v.l0, v.n_l, tuple(p.m0), tuple(p.ma), tuple(p.mb),
                                   tuple(v.mc))


def _fq(q, S, dtype):
    coef = xi.gaussian_form_factor_coefficients(S)
    return np.stack([oracle.form_factor_gaussian(q, *coef[s]) for s in range(S)]).astype(dtype)


def _species_gate(I_gpu, I_or, sp, fq, what):
    """Per-pixel gate of DESIGN.md R11 with the atom count generalised to sum_j f_{s(j)}(q)^2 per q (the errors of
    the per-kind amplitudes scale with f_s)."""
    counts = np.bincount(sp, minlength=fq.shape[0]).astype(np.float64)
    S2 = (counts[:, None] * fq.astype(np.float64) ** 2).sum(0)
    err = np.abs(np.asarray(I_gpu, np.float64) - I_or)
    ratio = np.max(err / (1e-3 * S2 + 1e-5 * np.abs(I_or)))
    assert np.all(np.isfinite(I_gpu)) and ratio <= 1.0, (what, ratio)
    return ratio


@pytest.mark.parametrize("engine", [xp.ENGINE_TENSOR, xp.ENGINE_SIMT])
def test_volume_f32_parity(engine):
    """Ragged 3-D block (n_h, n_k not tile multiples, tilted plane step mc), two species, 3 frames."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=5001, T=3)
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg)
    v = xp.qvolume(cfg.L, -20, 41, -35, 70, -3, 5, mc=(0, 1, 1))
    I = xp.xpcs_intensity_volume(_t(pos), _t(f), v, engine=engine).cpu().numpy()
    assert I.shape == (3, 5 * 41 * 70)
    ref = oracle.intensity(pos, f.astype(np.float64), _vol_q(v), cfg.L)
    assert_pixels(I, ref, cfg.N, "volume f32")


def test_volume_fp64_and_amplitude():
    N, L = 1500, 9.0
    pos = np.stack([xi.uniform_frame(90 + s, N, L) for s in range(2)])
    v = xp.qvolume(L, -6, 13, -5, 10, -4, 9)
    I = xp.xpcs_intensity_volume(_t(pos), None, v).cpu().numpy()
    q = _vol_q(v)
    np.testing.assert_allclose(I, oracle.intensity(pos, None, q, L), rtol=1e-9, atol=1e-9 * N)
    A = xp.xpcs_intensity_volume(_t(pos), None, v, amplitude=True).cpu().numpy()
    ref = oracle.amplitudes(pos, None, q, L)
    np.testing.assert_allclose(A[..., 0] + 1j * A[..., 1], ref, rtol=1e-9, atol=1e-9 * N)


def test_volume_bragg_peaks_gpu():
    """SC crystal of 8^3 atoms: I = N^2 at h, k, l in 8Z of a 3-D block, ~0 elsewhere (tensor engine)."""
    n_c, L = 8, 8.0
    pos = xi.crystal("sc", n_c, L, "f32")
    N = pos.shape[0]
    v = xp.qvolume(L, -12, 25, -12, 25, -9, 19)
    I = xp.xpcs_intensity_volume(_t(pos[None]), None, v).cpu().numpy()[0].reshape(19, 25, 25)
    l, h, k = np.meshgrid(np.arange(-9, 10), np.arange(-12, 13), np.arange(-12, 13), indexing="ij")
    peak = (h % n_c == 0) & (k % n_c == 0) & (l % n_c == 0)
    np.testing.assert_allclose(I[peak], float(N) ** 2, rtol=1e-5)
    assert np.max(I[~peak]) < 1e-3 * N


@pytest.mark.parametrize("engine", [xp.ENGINE_TENSOR, xp.ENGINE_SIMT])
def test_species_volume_parity(engine):
    """Three kinds with Gaussian-sum f_s(q) on a 3-D block: I and p (tensor engine partials hold conj(p))."""
    cfg = xi.scaled(xi.CONFIGS["c2"], N=4003, T=2)
    pos = xi.positions(cfg)
    sp = xi.species_labels(cfg.N, 3, 5)
    v = xp.qvolume(cfg.L, -30, 60, -17, 130, -1, 3)
    q = _vol_q(v)
    fq = _fq(q, 3, np.float32)
    I = xp.xpcs_intensity_volume(_t(pos), None, v, species=sp, f_q=_t(fq), engine=engine).cpu().numpy()
    ref = oracle.species_intensity(pos, sp, fq.astype(np.float64), q, cfg.L)
    _species_gate(I, ref, sp, fq, "species volume")
    A = xp.xpcs_intensity_volume(_t(pos), None, v, species=sp, f_q=_t(fq), engine=engine, amplitude=True)
    A = A.cpu().numpy().astype(np.float64)
    Aref = oracle.species_intensity(pos, sp, fq.astype(np.float64), q, cfg.L, amp=True)
    counts = np.bincount(sp, minlength=3).astype(np.float64)
    S2 = (counts[:, None] * fq.astype(np.float64) ** 2).sum(0)
    err = np.abs(A[..., 0] + 1j * A[..., 1] - Aref)
    assert np.max(err / (1e-3 * np.sqrt(S2) + 1e-5 * np.abs(Aref))) <= 1.0


def test_species_fp64_grid_and_empty_kind():
    """FP64 lattice path with species; kind 1 has no atoms (its f_q row must not matter)."""
    N, L = 1200, 8.5
    pos = xi.uniform_frame(5, N, L)[None]
    sp = np.where(np.arange(N) % 3 == 0, 2, 0).astype(np.int32)
    v = xp.qvolume(L, -8, 16, -8, 16, 0, 1)
    q = _vol_q(v)
    fq = _fq(q, 3, np.float64)
    fq[1] = 1e6
    I = xp.xpcs_intensity_volume(_t(pos), None, v, species=sp, f_q=_t(fq)).cpu().numpy()
    np.testing.assert_allclose(I, oracle.species_intensity(pos, sp, fq, q, L), rtol=1e-9, atol=1e-9 * N)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_species_explicit_q(dtype):
    """Off-lattice q list (generic SFU kernel / FP64 kernel) with two kinds."""
    N, L = 3001, 14.0
    npdt = np.float32 if dtype == "f32" else np.float64
    pos = np.stack([xi.uniform_frame(60 + s, N, L, dtype) for s in range(2)])
    sp = xi.species_labels(N, 2, 9)
    q = np.random.default_rng(4).uniform(-7, 7, (900, 3)).astype(npdt)
    fq = _fq(q.astype(np.float64), 2, npdt)
    I = xp.xpcs_intensity_species(_t(pos), sp, _t(fq), _t(q), L).cpu().numpy()
    ref = oracle.species_intensity(pos, sp, fq.astype(np.float64), q.astype(np.float64), L)
    if dtype == "f64":
        np.testing.assert_allclose(I, ref, rtol=1e-9, atol=1e-9 * N)
    else:
        _species_gate(I, ref, sp, fq, "species explicit q")


def test_form_factor_gaussian_kernel():
    L = 20.0
    v = xp.qvolume(L, -10, 21, -10, 21, -3, 7)
    a, b, c = xi.gaussian_form_factor_coefficients(4)[3]
    f = xp.xpcs_form_factor_gaussian(a, b, c, vol=v, out_dtype=xp.F64).cpu().numpy()
    np.testing.assert_allclose(f, oracle.form_factor_gaussian(_vol_q(v), a, b, c), rtol=1e-13)
    q = np.random.default_rng(1).uniform(-9, 9, (777, 3))
    f = xp.xpcs_form_factor_gaussian(a, b, c, q_vectors=_t(q), out_dtype=xp.F64).cpu().numpy()
    np.testing.assert_allclose(f, oracle.form_factor_gaussian(q, a, b, c), rtol=1e-13)


def test_table1_grid():
    """Table 1's workload: one frame of N = 4000 atoms, L = 59.19, the full 81^3 grid on the GPU;
    the oracle checks 3 seeded l-planes in full plus the forward point I(0) = N^2."""
    t1 = xi.TABLE1
    pos = xi.uniform_frame(t1["seed"], t1["N"], t1["L"], "f32")
    h = t1["n"] // 2
    v = xp.qvolume(t1["L"], -h, t1["n"], -h, t1["n"], -h, t1["n"])
    I = xp.xpcs_intensity_volume(_t(pos[None]), None, v).cpu().numpy()[0].reshape(t1["n"], t1["n"], t1["n"])
    assert abs(I[h, h, h] - t1["N"] ** 2) <= 1e-5 * t1["N"] ** 2
    for il in (0, 17, h + 1):
        qp = oracle.lattice_q(t1["L"], -h, t1["n"], -h, t1["n"], m0=(0, 0, il - h))
        ref = oracle.intensity(pos, None, qp, t1["L"])[0].reshape(t1["n"], t1["n"])
        assert_pixels(I[il], ref, t1["N"], f"table1 l-plane {il}")


@pytest.mark.parametrize("f_heavy", [2.0, 4.0])
def test_species_hybrid_auto_parity(f_heavy):
    """AUTO with f_max hints: f in {1, 2} runs every kind on the integer engine (budget 2.5), f in {1, 4} splits the
    heavy kind between the integer and split-FP16 engines; parity at the gate, and the amplitude of the mixed
    engines (both hold conj(p) partials)."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=7001, T=2)
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg)
    sp = (f > 1.5).astype(np.int32)
    f = np.where(sp == 1, f_heavy, 1.0)
    counts = np.bincount(sp, minlength=2)
    split = xp.species_engines(counts, [1.0, f_heavy])
    assert split[0] == counts[0] and (split[1] == counts[1]) == (f_heavy == 2.0)
    v = xp.qvolume(cfg.L, -60, 120, -40, 150, 0, 1)
    q = _vol_q(v)
    fq = np.stack([np.full(q.shape[0], 1.0), np.full(q.shape[0], f_heavy)]).astype(np.float32)
    I = xp.xpcs_intensity_volume(_t(pos), None, v, species=sp, f_q=_t(fq), f_max=[1.0, f_heavy]).cpu().numpy()
    ref = oracle.intensity(pos, f.astype(np.float64), q, cfg.L)
    assert_pixels(I, ref, cfg.N, f"species hybrid f_heavy {f_heavy}")
    A = xp.xpcs_intensity_volume(_t(pos), None, v, species=sp, f_q=_t(fq), f_max=[1.0, f_heavy], amplitude=True)
    A = A.cpu().numpy().astype(np.float64)
    Aref = oracle.amplitudes(pos, f.astype(np.float64), q, cfg.L)
    err = np.abs(A[..., 0] + 1j * A[..., 1] - Aref)
    assert np.max(err / (1e-3 * np.sqrt(cfg.N) + 1e-5 * np.abs(Aref))) <= 1.0


@pytest.mark.parametrize("case", ["species_hybrid", "per_atom_f", "uniform_i8"])
def test_frame_batches_overlapped(case, monkeypatch):
    """Frames split into many batches (XPCS_BATCH_BYTES) run on two alternating streams with their own buffers
    (a batch's staging and reduction beside the neighbouring batch's tensor engine): the same intensities as one
    batch -- bit-identical where the atom chunking does not change (species calls) -- and the per-pixel gate."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=5003, T=7)
    pos = xi.positions(cfg)
    v = xp.qvolume(cfg.L, -70, 140, -64, 256, 0, 1)
    q = _vol_q(v)
    kw, f64 = {}, None
    if case == "species_hybrid":
        f = xi.form_factors(cfg)
        sp = (f > 1.5).astype(np.int32)
        f64 = np.where(sp == 1, 4.0, 1.0)
        fq = np.stack([np.full(q.shape[0], 1.0), np.full(q.shape[0], 4.0)]).astype(np.float32)
        kw = dict(species=sp, f_q=_t(fq), f_max=[1.0, 4.0])
        ff = None
    elif case == "per_atom_f":
        f64 = 1.0 + np.random.default_rng(3).random(cfg.N)
        ff = _t(f64.astype(np.float32))
    else:
        ff = None
    one = xp.xpcs_intensity_volume(_t(pos), ff, v, **kw).cpu().numpy()
    monkeypatch.setenv("XPCS_BATCH_BYTES", str(16 * cfg.N * 2))    # two frames per batch: 4 batches
    many = xp.xpcs_intensity_volume(_t(pos), ff, v, **kw).cpu().numpy()
    torch.cuda.synchronize()
    if case == "species_hybrid":
        np.testing.assert_array_equal(many, one)
    ref = oracle.intensity(pos, f64, q, cfg.L)
    assert_pixels(many, ref, cfg.N if f64 is None else float((f64 ** 2).sum()), f"batched {case}")
