"""CPU-side checks of the boundary: the library builds for sm_100a, loads, exports every symbol that
include/xpcs.h declares, and its host-only / validation paths behave as documented (no compute calls)."""
import ctypes
import os
import re

import pytest

import paper_2204_13241_b200 as xp
from paper_2204_13241_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "xpcs.h")).read()
    return sorted(set(re.findall(r"^XPCS_API\s+(?:const\s+)?\w+\*?\s+(\w+)\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2204_13241_b200 import build
    build.build()
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    decl = _declared()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED) == decl


def test_sass_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_lattice_plane_host_helper(lib):
    g = xp.lattice_plane(34.2, 256, 0)
    assert (g.h0, g.n_h, g.k0, g.n_k) == (-128, 256, -128, 256)
    assert list(g.ma) == [1, 0, 0] and list(g.mb) == [0, 1, 0] and list(g.m0) == [0, 0, 0]
    g = _lib.QGrid()
    rc = lib.xpcs_qgrid_lattice_plane(-1.0, 4, 0, ctypes.byref(g))
    assert rc == _lib.XPCS_EINVAL and b"L must" in lib.xpcs_last_error()


def test_validation_rejects_before_any_launch(lib):
    """EINVAL paths never touch the device (they run in this GPU-less container)."""
    n0 = lib.xpcs_launch_count()
    o = _lib.Opts(0, 0, None, 0, 0)
    rc = lib.xpcs_intensity(None, 10, None, None, 5, 1, 1.0, None, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"must not be NULL" in lib.xpcs_last_error()
    dummy = ctypes.c_void_p(16)
    rc = lib.xpcs_intensity(dummy, 0, None, dummy, 5, 1, 1.0, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"N must be > 0" in lib.xpcs_last_error()
    rc = lib.xpcs_intensity(dummy, 10, None, dummy, 5, 1, -2.0, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL
    bad = _lib.Opts(7, 0, None, 0, 0)
    rc = lib.xpcs_intensity(dummy, 10, None, dummy, 5, 1, 1.0, dummy, ctypes.byref(bad))
    assert rc == _lib.XPCS_EINVAL and b"dtype" in lib.xpcs_last_error()
    lags, lp = _lib._i32_array([1, 5, 9])
    rc = lib.xpcs_g2(dummy, 9, 4, lp, 3, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"lag 9" in lib.xpcs_last_error()
    w, wp = _lib._i32_array([1, 0])
    rc = lib.xsvs_contrast(dummy, 9, 4, dummy, 3, wp, 2, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"window 0" in lib.xpcs_last_error()
    g = xp.lattice_plane(10.0, 8)
    g.n_h = 0
    rc = lib.xpcs_intensity_grid(dummy, 10, None, ctypes.byref(g), 1, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL
    rc = lib.xpcs_profile_query(99, None, None, None)
    assert rc == _lib.XPCS_EINVAL
    # block-streamed g2: the ring must hold the largest lag; t0 >= 0; finalize checks lags against the frame count
    rc = lib.xpcs_g2_accumulate(dummy, 4, 0, 4, lp, 3, dummy, 8, dummy, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"ring" in lib.xpcs_last_error()
    rc = lib.xpcs_g2_accumulate(dummy, 4, -1, 4, lp, 3, dummy, 9, dummy, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"t0" in lib.xpcs_last_error()
    rc = lib.xpcs_g2_accumulate(dummy, 4, 0, 4, lp, 3, None, 9, dummy, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"ring" in lib.xpcs_last_error()
    big, bp = _lib._i32_array([1, 700])
    rc = lib.xpcs_g2_accumulate(dummy, 4, 0, 4, bp, 2, dummy, 700, dummy, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EUNSUPPORTED
    rc = lib.xpcs_g2_finalize(dummy, dummy, 9, 4, lp, 3, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"lag 9" in lib.xpcs_last_error()
    rc = lib.xpcs_g2_finalize(dummy, None, 10, 4, lp, 3, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"must not be NULL" in lib.xpcs_last_error()
    assert lib.xpcs_launch_count() == n0


def test_binding_refuses_host_tensors(lib):
    torch = pytest.importorskip("torch")
    with pytest.raises(ValueError, match="device memory"):
        _lib._ptr(torch.zeros(3))


def test_volume_species_validation_before_launch(lib):
    """3-D blocks / q-dependent form factors: host-side validation rejects before any launch."""
    n0 = lib.xpcs_launch_count()
    o = _lib.Opts(0, 0, None, 0, 0)
    dummy = ctypes.c_void_p(16)
    vol = xp.qvolume(10.0, -4, 8, -4, 8, -2, 5)
    assert vol.n_q == 320
    vol.n_l = 0
    rc = lib.xpcs_intensity_volume(dummy, 4, None, None, ctypes.byref(vol), 1, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"n_l" in lib.xpcs_last_error()
    vol = xp.qvolume(10.0, -4, 8, -4, 8, -2, 5, mc=(0, 0, 1 << 30))
    rc = lib.xpcs_intensity_volume(dummy, 4, None, None, ctypes.byref(vol), 1, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"out of range" in lib.xpcs_last_error()
    vol = xp.qvolume(10.0, -4, 8, -4, 8, -2, 5)
    sp = _lib.Species()
    arr, ap = _lib._i32_array([0, 1, 2, 1])
    sp.species, sp.f_q, sp.n_species = ap, dummy, 2
    rc = lib.xpcs_intensity_volume(dummy, 4, None, ctypes.byref(sp), ctypes.byref(vol), 1, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"species[2] = 2" in lib.xpcs_last_error()
    sp.n_species = 17
    rc = lib.xpcs_intensity_species(dummy, 4, ctypes.byref(sp), dummy, 5, 1, 1.0, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"n_species" in lib.xpcs_last_error()
    sp.n_species = 3
    rc = lib.xpcs_intensity_volume(dummy, 4, dummy, ctypes.byref(sp), ctypes.byref(vol), 1, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"exclusive" in lib.xpcs_last_error()
    sp.f_q = None
    rc = lib.xpcs_intensity_species(dummy, 4, ctypes.byref(sp), dummy, 5, 1, 1.0, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"f_q" in lib.xpcs_last_error()
    rc = lib.xpcs_intensity_species(dummy, 4, None, dummy, 5, 1, 1.0, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL
    a = (ctypes.c_double * 7)()
    rc = lib.xpcs_form_factor_gaussian(dummy, 5, None, 7, a, a, 0.0, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"n_gauss" in lib.xpcs_last_error()
    rc = lib.xpcs_form_factor_gaussian(None, 5, None, 1, a, a, 0.0, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL
    assert lib.xpcs_launch_count() == n0


def test_fft_method_validation(lib):
    n0 = lib.xpcs_launch_count()
    o = _lib.Opts(0, 0, None, 0, 0)
    dummy = ctypes.c_void_p(16)
    ok = xp.qvolume(10.0, -4, 8, -4, 8, -2, 5)
    tilted = xp.qvolume(10.0, -4, 8, -4, 8, -2, 5, mb=(0, 1, 1))
    rc = lib.xpcs_intensity_fft(dummy, 10, 1, ctypes.byref(tilted), 32, 0.3, 0, None, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"axis-aligned" in lib.xpcs_last_error()
    rc = lib.xpcs_intensity_fft(dummy, 10, 1, ctypes.byref(ok), 33, 0.3, 0, None, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"n_grid" in lib.xpcs_last_error()
    rc = lib.xpcs_intensity_fft(dummy, 10, 1, ctypes.byref(ok), 32, 0.3, 10, None, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"odd" in lib.xpcs_last_error()
    wide = xp.qvolume(10.0, -5, 8, -4, 8, -2, 5)
    rc = lib.xpcs_intensity_fft(dummy, 10, 1, ctypes.byref(wide), 8, 0.3, 0, None, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"block indices" in lib.xpcs_last_error()
    rc = lib.xpcs_intensity_fft(dummy, 10, 1, ctypes.byref(ok), 32, -1.0, 0, None, dummy, ctypes.byref(o))
    assert rc == _lib.XPCS_EINVAL and b"eta" in lib.xpcs_last_error()
    assert lib.xpcs_launch_count() == n0


def test_binding_argument_checks():
    """The binding refuses mixed dtypes and mis-shaped arrays before calling the library (the C ABI takes one
    in_dtype for every float array of a call)."""
    torch = pytest.importorskip("torch")
    from paper_2204_13241_b200._lib import _positions3
    pos = torch.zeros(2, 5, 3)
    assert _positions3(pos[0]).shape == (1, 5, 3)
    with pytest.raises(ValueError, match=r"\[T\]\[N\]\[3\]"):
        _positions3(torch.zeros(2, 5, 2))
    with pytest.raises(TypeError, match="dtype"):
        _positions3(pos, form_factors=torch.zeros(5, dtype=torch.float64))
    with pytest.raises(ValueError, match="form_factors"):
        _positions3(pos, form_factors=torch.zeros(4))
    with pytest.raises(ValueError, match="q_vectors"):
        _positions3(pos, q_vectors=torch.zeros(7, 2))


def test_species_engine_rule():
    """AUTO's per-kind engine split (mirror of api.cu): kinds in increasing f_max on the integer engine while
    sum (f_max / f_min)^2 N_s / N <= 1, the crossing kind split at the budget."""
    se = lambda c, f: xp.species_engines(c, f, budget=1.0)
    assert se([1000], [1.0]) == [1000]
    assert se([500, 500], [1.0, 2.0]) == [500, 125]            # budget 1: f = 1 half + a quarter of the f = 2 half
    assert se([300, 700], [2.0, 1.0]) == [75, 700]
    assert se([400, 400, 200], [1.0, 1.0, 1.0]) == [400, 400, 200]
    assert se([10, 10], None) == [0, 0]                        # no hints: every kind on split-FP16
    assert se([0, 100], [0.5, 1.0])[1] == 100                  # an empty kind does not set the reference weight
    # the default budget (2.5, api.cu kI8BudgetDefault; tools/i8_budget_probe.py): an f in {1, 2} half-half mix runs
    # entirely on the integer engine, a heavier kind only in part
    assert xp.species_engines([500, 500], [1.0, 2.0]) == [500, 500]
    assert xp.species_engines([500, 500], [1.0, 8.0]) == [500, 31]


def test_step_host_validation_before_launch(lib):
    """xpcs_step_host (the host-buffer end-to-end entry) rejects bad arguments before any copy or launch."""
    n0 = lib.xpcs_launch_count()
    o = _lib.Opts(0, 0, None, 0, 0)
    assert lib.xpcs_step_host(None, ctypes.byref(o)) == _lib.XPCS_EINVAL
    st = _lib.Step()
    st.positions = 16
    st.bin_of_q = 32
    st.N, st.frames, st.n_bins, st.batches = 100, 10, 4, 2
    st.grid = xp.lattice_plane(10.0, 8)
    lags, lp = _lib._i32_array([1, 10])
    st.lags, st.n_lags = lp, 2
    assert lib.xpcs_step_host(ctypes.byref(st), ctypes.byref(o)) == _lib.XPCS_EINVAL
    assert b"lag 10" in lib.xpcs_last_error()
    st.n_lags = 1
    w, wp = _lib._i32_array([0])
    st.windows, st.n_windows = wp, 1
    assert lib.xpcs_step_host(ctypes.byref(st), ctypes.byref(o)) == _lib.XPCS_EINVAL
    assert b"window 0" in lib.xpcs_last_error()
    st.n_windows = 0
    st.batches = 0
    assert lib.xpcs_step_host(ctypes.byref(st), ctypes.byref(o)) == _lib.XPCS_EINVAL
    st.batches = 2
    # the limits of the calls inside the step are checked up front too (an error after the stream fork
    # left the copy streams unjoined): a lag beyond the g2 kernel's 640, too many rings
    st.frames = 1000
    big, bp = _lib._i32_array([700])
    st.lags, st.n_lags = bp, 1
    assert lib.xpcs_step_host(ctypes.byref(st), ctypes.byref(o)) == _lib.XPCS_EUNSUPPORTED
    st.n_lags = 0
    st.n_bins = 20000
    assert lib.xpcs_step_host(ctypes.byref(st), ctypes.byref(o)) == _lib.XPCS_EINVAL
    st.n_bins = 4
    st.frames = 10
    st.positions = None
    assert lib.xpcs_step_host(ctypes.byref(st), ctypes.byref(o)) == _lib.XPCS_EINVAL
    assert lib.xpcs_launch_count() == n0
