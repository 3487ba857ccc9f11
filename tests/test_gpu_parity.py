"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on the same seeded inputs.

Small cases span several tiles, atom chunks and ragged tails; full-size cases run in the launch configuration
bench.py times (paper_2204_13241_b200.pipeline) and compare sampled outputs the oracle can afford.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import xpcs_inputs as xi  # noqa: E402
import paper_2204_13241_b200 as xp  # noqa: E402
from paper_2204_13241_b200 import pipeline  # noqa: E402
from _gates import assert_pixels, assert_rel  # noqa: E402

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


def _grid_q(grid):
    return oracle.lattice_q(grid.L, grid.h0, grid.n_h, grid.k0, grid.n_k, tuple(grid.m0), tuple(grid.ma), tuple(grid.mb))


# ----------------------------------------------------------------------------------- lattice planes
@pytest.mark.parametrize("engine", [xp.ENGINE_SIMT, xp.ENGINE_TENSOR, xp.ENGINE_TENSOR_I8])
def test_lattice_f32_ragged(engine):
    """Ragged everything: N not a multiple of the 16-atom sub-block or the 4096-atom chunk, n_h / n_k not
    multiples of the 64 x 128 tile, an l != 0 plane with a tilted direction, two species."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=9001, T=3)
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg)
    g = xp.qgrid(cfg.L, -37, 70, -75, 150, m0=(0, 0, 2), ma=(1, 0, 0), mb=(0, 1, 1))
    I = xp.xpcs_intensity_grid(_t(pos), _t(f), g, engine=engine).cpu().numpy()
    ref = oracle.intensity(pos, f.astype(np.float64), _grid_q(g), cfg.L)
    assert_pixels(I, ref, cfg.N, "lattice f32 ragged")


def test_config1_fp64_full():
    """Config 1 in full: N = 1000, L = 10, fp64, 64 x 64 plane, one frame, I in fp64."""
    cfg = xi.CONFIGS["c1"]
    pos = xi.positions(cfg)
    g = xp.lattice_plane(cfg.L, cfg.n_plane)
    I = xp.xpcs_intensity_grid(_t(pos), None, g).cpu().numpy()
    ref = oracle.intensity(pos, None, _grid_q(g), cfg.L)
    assert I.dtype == np.float64
    assert_pixels(I, ref, cfg.N, "c1")
    np.testing.assert_allclose(I, ref, rtol=1e-9, atol=1e-9 * cfg.N)


@pytest.mark.parametrize("engine", [xp.ENGINE_SIMT, xp.ENGINE_TENSOR, xp.ENGINE_TENSOR_I8])
@pytest.mark.parametrize("kind,n_cells,L,n,dtype", [("sc", 10, 10.0, 64, "f64"), ("sc", 10, 10.0, 64, "f32"),
                                                     ("fcc", 20, xi.CONFIGS["c2"].L, 256, "f32"),
                                                     ("bcc", 16, 40.0, 128, "f32")])
def test_bragg_peaks_gpu(kind, n_cells, L, n, dtype, engine):
    """Perfect crystals: I = N^2 at the crystal's reciprocal lattice, ~0 elsewhere (closed form; the c2-size
    FCC is config 2's own N = 32000)."""
    pos = xi.crystal(kind, n_cells, L, dtype)
    N = pos.shape[0]
    g = xp.lattice_plane(L, n)
    if dtype == "f64" and engine != xp.ENGINE_SIMT:
        with pytest.raises(xp.XpcsError, match="f32"):          # tensor engines are f32-only (EUNSUPPORTED)
            xp.xpcs_intensity_grid(_t(pos), None, g, engine=engine)
        engine = xp.ENGINE_AUTO                                  # -> the FP64 kernel
    I = xp.xpcs_intensity_grid(_t(pos), None, g, engine=engine).cpu().numpy().reshape(n, n).astype(np.float64)
    h = np.arange(-n // 2, n // 2)
    H, K = np.meshgrid(h, h, indexing="ij")
    period = 2 * n_cells if kind == "fcc" else n_cells
    peak = (H % period == 0) & (K % period == 0)
    if kind == "bcc":
        peak &= ((H // period + K // period) % 2 == 0)
    np.testing.assert_allclose(I[peak], float(N) ** 2, rtol=1e-5)
    assert np.max(I[~peak]) <= 1e-3 * N


def test_tensor_engine_available():
    """On a B200 the AUTO engine must resolve to the tcgen05 kernel (no silent SIMT fallback)."""
    assert xp.engine_available(xp.ENGINE_TENSOR)


@pytest.mark.parametrize("N", [16, 1000, 4096, 20000])
def test_tensor_engine_accumulation_length(N):
    """The tcgen05 accumulator truncates; drains every 128 atoms keep the error flat in N."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=N, T=1)
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg)
    g = xp.qgrid(cfg.L, -64, 128, -64, 128)
    I = xp.xpcs_intensity_grid(_t(pos), _t(f), g, engine=xp.ENGINE_TENSOR).cpu().numpy()
    ref = oracle.intensity(pos, f.astype(np.float64), _grid_q(g), cfg.L)
    ratio, worst = assert_pixels(I, ref, N, "tc accumulation")
    assert worst < 2e-4, worst


def test_shift_invariance_gpu():
    """PBC: a rigid shift of every atom leaves lattice-q intensities unchanged."""
    cfg = xi.scaled(xi.CONFIGS["c2"], N=5000, T=2)
    pos = xi.positions(cfg)
    g = xp.lattice_plane(cfg.L, 96)
    I0 = xp.xpcs_intensity_grid(_t(pos), None, g).cpu().numpy()
    I1 = xp.xpcs_intensity_grid(_t((pos + np.float32(7.25)).astype(np.float32)), None, g).cpu().numpy()
    assert_pixels(I1, I0, cfg.N, "shift")


# ----------------------------------------------------------------------------------- explicit q lists
def test_generic_q_off_lattice_and_ewald():
    """Off-lattice q (R3) incl. the Ewald detector q of config 4 at reduced size, two frames."""
    N, L = 7000, 20.0
    pos = np.stack([xi.uniform_frame(5 + s, N, L, "f32") for s in range(2)])
    rng = np.random.default_rng(9)
    q_rand = rng.uniform(-12, 12, (1000, 3))
    q_ew = oracle.ewald_q(xi.EWALD_WAVELENGTH_SIGMA, 48, 40, xi.EWALD_PITCH_RAD * 20)
    q = np.concatenate([q_rand, q_ew, np.zeros((1, 3))]).astype(np.float32)
    f = np.where(np.arange(N) % 3 == 0, 2.0, 1.0).astype(np.float32)
    I = xp.xpcs_intensity(_t(pos), _t(f), _t(q), L).cpu().numpy()
    ref = oracle.intensity(pos, f.astype(np.float64), q.astype(np.float64), L)
    assert_pixels(I, ref, N, "generic f32")
    # forward pixel: I(0) = (sum f)^2
    np.testing.assert_allclose(I[:, -1], f.astype(np.float64).sum() ** 2, rtol=1e-5)


def test_generic_q_fp64():
    N, L = 800, 9.0
    pos = xi.uniform_frame(3, N, L, "f64")[None]
    q = np.random.default_rng(1).uniform(-20, 20, (300, 3))
    I = xp.xpcs_intensity(_t(pos), None, _t(q), L).cpu().numpy()
    ref = oracle.intensity(pos, None, q, L)
    np.testing.assert_allclose(I, ref, rtol=1e-9, atol=1e-9 * N)


def test_generic_few_q_splits_atoms():
    """Few q and one frame: the library splits the atom sum across CTAs (FP64 fold of the chunks)."""
    N, L = 40000, 30.0
    pos = xi.uniform_frame(77, N, L, "f32")[None]
    q = oracle.lattice_q(L, 3, 2, -5, 2, m0=(0, 0, 1)).astype(np.float32)     # 4 q (the paper's single-q case class)
    I = xp.xpcs_intensity(_t(pos), None, _t(q), L).cpu().numpy()
    ref = oracle.intensity(pos, None, q.astype(np.float64), L)
    assert_pixels(I, ref, N, "few q")


def test_edge_cases():
    """N = 1, one q, one frame; f = NULL; a pixel of a 1 x 1 grid."""
    L = 5.0
    pos = np.array([[[1.25, 2.5, 3.75]]], np.float32)
    q = np.array([[0.7, -1.1, 2.3]], np.float32)
    I = xp.xpcs_intensity(_t(pos), None, _t(q), L).cpu().numpy()
    np.testing.assert_allclose(I, 1.0, rtol=1e-6)
    g = xp.qgrid(L, 3, 1, -2, 1)
    I = xp.xpcs_intensity_grid(_t(pos), _t(np.array([2.0], np.float32)), g).cpu().numpy()
    np.testing.assert_allclose(I, 4.0, rtol=1e-6)


# ----------------------------------------------------------------------------------- geometry
def test_geometry_parity():
    q_or = oracle.ewald_q(xi.EWALD_WAVELENGTH_SIGMA, 1024, 1024, xi.EWALD_PITCH_RAD)
    q32 = xp.xpcs_qgrid_ewald(xi.EWALD_WAVELENGTH_SIGMA, 1024, 1024, xi.EWALD_PITCH_RAD).cpu().numpy()
    q64 = xp.xpcs_qgrid_ewald(xi.EWALD_WAVELENGTH_SIGMA, 1024, 1024, xi.EWALD_PITCH_RAD, out_dtype=xp.F64).cpu().numpy()
    np.testing.assert_allclose(q64, q_or, rtol=0, atol=1e-13)
    ulp = np.spacing(np.abs(q_or).astype(np.float32))
    assert np.all(np.abs(q32.astype(np.float64) - q_or.astype(np.float32).astype(np.float64)) <= ulp)
    for n in (64, 256, 512):
        g = xp.lattice_plane(10.0, n)
        b = xp.xpcs_lattice_bins(g, 32, n // 64).cpu().numpy()
        np.testing.assert_array_equal(b, oracle.lattice_bins(n))
    qf = q_or.astype(np.float32)
    b = xp.xpcs_radial_bins(_t(qf), xi.EWALD_QMAX, 32).cpu().numpy()
    np.testing.assert_array_equal(b, oracle.radial_bins(qf, xi.EWALD_QMAX))


# ----------------------------------------------------------------------------------- statistics (reduction parity)
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_g2_reduction_parity(dt):
    rng = np.random.default_rng(4)
    T, n_q = 157, 3000
    I = rng.exponential(1.0, (T, n_q)).astype(np.float32 if dt == "f32" else np.float64)
    I[:, 7] = 0.0
    lags = [0, 1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 144, 156] + list(range(30, 60))
    G = xp.xpcs_g2(_t(I), lags).cpu().numpy()
    ref = oracle.g2(I, lags)
    assert_rel(G, ref, 1e-10, "g2")


@pytest.mark.parametrize("lags", [list(range(1, 201)),                       # config 3's list: 7 warps x 24 + 32
                                  list(range(0, 301)),                       # two block rows (> 256 lags)
                                  list(range(1, 51)),                        # config 2's list: 7 warps x 8 (ragged)
                                  [3, 9, 10, 11, 40] + list(range(60, 101)) + [150, 151, 203]])  # mixed runs
def test_g2_reduction_parity_long_lag_lists(lags):
    rng = np.random.default_rng(41)
    T, n_q = 419, 70                                     # ragged: 3 chunks + a tail, 3 pixel blocks (the last partial)
    I = rng.exponential(1.0, (T, n_q)).astype(np.float32)
    G = xp.xpcs_g2(_t(I), lags).cpu().numpy()
    assert_rel(G, oracle.g2(I, lags), 1e-10, "g2")


def test_rings_and_structure_factor_parity():
    rng = np.random.default_rng(5)
    T, n = 11, 256
    I = rng.exponential(3.0, (T, n * n)).astype(np.float32)
    bins = oracle.lattice_bins(n)
    bins_d = _t(bins)
    out = xp.xpcs_shell_mean(_t(I), bins_d, 33).cpu().numpy()          # ring 32 is empty -> NaN
    assert_rel(out, oracle.shell_mean(I, bins, 33), 1e-10, "rings")
    f = np.where(np.arange(5000) % 2 == 1, 2.0, 1.0).astype(np.float32)
    S = xp.xpcs_structure_factor_shells(_t(I), _t(f), 5000, bins_d, 32).cpu().numpy()
    assert_rel(S, oracle.structure_factor_shells(I, f, 5000, bins, 32), 1e-10, "S rings")
    S1 = xp.xpcs_structure_factor_shells(_t(I), None, 5000, bins_d, 32).cpu().numpy()
    assert_rel(S1, oracle.structure_factor_shells(I, None, 5000, bins, 32), 1e-10, "S rings f=1")


@pytest.mark.parametrize("T,windows", [(200, [1, 2, 4, 8, 16, 32, 64, 128]), (37, [1, 3, 5, 36, 37]),
                                       (64, list(range(1, 21)))])
def test_xsvs_reduction_parity(T, windows):
    rng = np.random.default_rng(T)
    n = 128
    I = rng.exponential(2.0, (T, n * n)).astype(np.float32)
    bins = oracle.lattice_bins(n, n_bins=16)
    bins[:50] = 15    # a scattered ring
    beta = xp.xsvs_contrast(_t(I), _t(bins), 17, windows).cpu().numpy()    # ring 16 empty
    assert_rel(beta, oracle.xsvs_beta(I, bins, 17, windows), 1e-10, "xsvs")


@pytest.mark.parametrize("case", ["wide", "wide_f64", "long"])
def test_xsvs_kernel_paths(case):
    """The three XSVS gather paths (k_stats.cu launch_xsvs): four pixels per lane when the detector fills the GPU
    (65536 pixels), one per lane below that (the test above), and the one-warp-per-window kernel for series longer
    than the shared-memory close mask (17000 frames)."""
    rng = np.random.default_rng(11)
    if case == "long":
        T, n, windows = 17000, 32, [1, 7, 1000, 16999]
    else:
        T, n, windows = 130, 256, [1, 2, 3, 4, 8, 16, 64, 129]
    I = rng.exponential(2.0, (T, n * n)).astype(np.float64 if case == "wide_f64" else np.float32)
    nb = n // 16 if case == "long" else 16          # ring width n / (2 nb) pixels
    bins = oracle.lattice_bins(n, n_bins=nb)
    bins[:37] = nb - 1  # a scattered ring with a ragged pixel count
    beta = xp.xsvs_contrast(_t(I), _t(bins), nb + 1, windows).cpu().numpy()    # ring nb empty
    assert_rel(beta, oracle.xsvs_beta(I, bins, nb + 1, windows), 1e-10, f"xsvs {case}")


# ----------------------------------------------------------------------------------- config-size cases
def test_config2_simt_engine_sampled():
    """The SIMT engine on config 2's size (first 10 frames) against the oracle."""
    cfg = xi.scaled(xi.CONFIGS["c2"], T=10)
    pos = xi.positions(cfg)
    g = xp.lattice_plane(cfg.L, cfg.n_plane)
    I = xp.xpcs_intensity_grid(_t(pos), None, g, engine=xp.ENGINE_SIMT).cpu().numpy()
    q = oracle.lattice_q(cfg.L, **oracle.plane_grid(cfg.n_plane))
    pix = xi.pixel_subset(q.shape[0], 256, 7)
    ref = oracle.intensity(pos[[0, 9]], None, q[pix], cfg.L)
    assert_pixels(I[[0, 9]][:, pix], ref, cfg.N, "c2 simt")


def test_end_to_end_host_path_matches_device_path():
    """pipeline.run_host (xpcs_step_host: pinned H2D in frame batches on internal copy streams, D2H of every result)
    == pipeline.run.  The
    integer engine sizes its atom chunks by the frames of each call, so the host path's smaller batches fold the
    same exact per-chunk sums in different fp32 partials: results agree to fp32 rounding, not bit for bit; the
    second run_host of the same batches is bit-identical to the first (determinism)."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=5000, T=37, lags=(1, 2, 5, 9), windows=(1, 2, 4, 8))
    cfg = xi.Config(**{**cfg.__dict__, "n_plane": 128})
    pos = xi.positions(cfg)
    f = xi.form_factors(cfg)
    wl = pipeline.workload_from_config(cfg)
    P = pipeline.Pipeline(wl)
    dev = P.run(_t(pos), _t(f))
    ref = {k: v.cpu().numpy().copy() for k, v in dev.items()}
    P.alloc_host_io(pos, f, batches=5)
    first = None
    for _ in range(2):
        host = P.run_host()
        torch.cuda.synchronize()
        for k in ref:
            a = host[k].numpy().astype(np.float64)
            b = ref[k].astype(np.float64)
            ok = np.isfinite(b)
            assert np.array_equal(np.isfinite(a), ok), k
            np.testing.assert_allclose(a[ok], b[ok], rtol=2e-5, atol=2e-5 * np.abs(b[ok]).max(), err_msg=k)
        if first is None:
            first = {k: v.numpy().copy() for k, v in host.items()}
        else:
            for k in first:
                np.testing.assert_array_equal(host[k].numpy(), first[k], err_msg=k)
    h2d, d2h = P.io_bytes()
    assert h2d == pos.nbytes + f.nbytes and d2h > pos.shape[0] * 128 * 128 * 4


@pytest.mark.parametrize("out_dtype", [xp.F32, xp.F64])
def test_step_host_mixed_dtypes_and_host_kinds(out_dtype):
    """xpcs_step_host straight through the C ABI with f32 inputs, f32 or f64 outputs and per-atom HOST form factors
    f in {1, 2} (no species): the library runs the two values as atom kinds (integer engine for the light kind) and
    normalises S(q,t) by sum f^2 read at the INPUT dtype (it was read at the output dtype).  I against
    the oracle at the per-pixel gate; S rings, g2 and beta against the oracle's reductions of the returned I."""
    cfg = xi.scaled(xi.CONFIGS["c3"], N=6000, T=12)
    pos = np.ascontiguousarray(xi.positions(cfg))
    f = xi.form_factors(cfg).astype(np.float32)
    n = 96
    g = xp.lattice_plane(cfg.L, n)
    bins_h = oracle.lattice_bins(n, 32 if n % 64 == 0 else 16)
    nb = int(bins_h.max()) + 1
    bins = _t(bins_h)
    T, n_q = cfg.T, n * n
    od = np.float64 if out_dtype == xp.F64 else np.float32
    pos_p = torch.from_numpy(pos).pin_memory()
    f_p = torch.from_numpy(f).pin_memory()
    I = torch.empty((T, n_q), dtype=torch.float64 if out_dtype == xp.F64 else torch.float32).pin_memory()
    S = torch.empty((T, nb), dtype=torch.float64).pin_memory()
    g2 = torch.empty((3, n_q), dtype=I.dtype).pin_memory()
    beta = torch.empty((3, nb), dtype=torch.float64).pin_memory()
    keep = xp.xpcs_step_host(pos_p, f_p, g, bins, nb, lags=(1, 2, 5), windows=(1, 2, 4), I_out=I, g2_out=g2,
                             S_rings=S, beta=beta, batches=3, out_dtype=out_dtype)
    torch.cuda.synchronize()
    del keep
    Ih = I.numpy()
    assert Ih.dtype == od
    ref = oracle.intensity(pos, f.astype(np.float64), _grid_q(g), cfg.L)
    assert_pixels(Ih, ref, cfg.N, "step_host host kinds")
    assert_rel(S.numpy(), oracle.structure_factor_shells(Ih, f, cfg.N, bins_h, nb), 1e-10, "S rings (sum f^2 norm)")
    assert_rel(g2.numpy(), oracle.g2(Ih, (1, 2, 5)).astype(od), 1e-6 if od == np.float32 else 1e-10, "g2")
    assert_rel(beta.numpy(), oracle.xsvs_beta(Ih, bins_h, nb, (1, 2, 4)), 1e-10, "beta")
