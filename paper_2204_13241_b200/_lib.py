"""ctypes binding of libxpcs.so (include/xpcs.h).  Argument marshalling only: every step runs in the CUDA
library; there is no CPU fallback -- if the shared library or a CUDA device is missing, calls raise.

Names follow the C ABI.  Tensor arguments are torch CUDA tensors (device memory + the current stream are the
only things PyTorch provides); host-side integer lists (lags, windows) are plain Python sequences.
"""
from __future__ import annotations

import ctypes
import itertools
import threading
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XPCS_LIB", os.path.join(_HERE, "lib", "libxpcs.so"))   # XPCS_LIB: experiments only

XPCS_OK, XPCS_EINVAL, XPCS_ECUDA, XPCS_ENOMEM, XPCS_EUNSUPPORTED = 0, 1, 2, 3, 4
F32, F64 = 0, 1
ENGINE_AUTO, ENGINE_SIMT, ENGINE_TENSOR, ENGINE_TENSOR_I8 = 0, 1, 2, 3
KERNEL_CLASSES = ("intensity_main", "stage", "amplitude_reduce", "g2", "xsvs", "rings", "fixup", "intensity_i8",
                  "intensity_tc")

EXPORTED = (
    "xpcs_intensity", "xpcs_intensity_grid", "xpcs_g2", "xsvs_contrast", "xpcs_shell_mean",
    "xpcs_structure_factor_shells", "xpcs_qgrid_lattice_plane", "xpcs_qgrid_ewald", "xpcs_lattice_bins",
    "xpcs_radial_bins", "xpcs_last_error", "xpcs_release", "xpcs_launch_count", "xpcs_profile_reset",
    "xpcs_profile_query", "xpcs_device_info", "xpcs_version", "xpcs_engine_available",
    "xpcs_amplitude", "xpcs_amplitude_grid", "xpcs_isf",
    "xpcs_intensity_volume", "xpcs_amplitude_volume", "xpcs_intensity_species", "xpcs_amplitude_species",
    "xpcs_form_factor_gaussian", "xpcs_speckle_histogram", "xpcs_intensity_fft", "xpcs_rings_register",
    "xpcs_rings_unregister", "xpcs_step_host", "xpcs_ring_moments", "xpcs_ring_means_from_moments", "xsvs_moments",
    "xsvs_contrast_from_moments", "xpcs_g2_accumulate", "xpcs_g2_finalize",
)


class XpcsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"xpcs status {status}: {msg}")
        self.status = status


class Opts(ctypes.Structure):
    _fields_ = [("in_dtype", ctypes.c_int32), ("out_dtype", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("engine", ctypes.c_int32), ("profile", ctypes.c_int32), ("workspace", ctypes.c_int32),
                ("pad_", ctypes.c_int32)]


class QGrid(ctypes.Structure):
    _fields_ = [("L", ctypes.c_double), ("m0", ctypes.c_int32 * 3), ("ma", ctypes.c_int32 * 3),
                ("mb", ctypes.c_int32 * 3), ("pad_", ctypes.c_int32), ("h0", ctypes.c_int64),
                ("n_h", ctypes.c_int64), ("k0", ctypes.c_int64), ("n_k", ctypes.c_int64)]

    @property
    def n_q(self):
        return int(self.n_h * self.n_k)


class QVolume(ctypes.Structure):
    _fields_ = [("plane", QGrid), ("mc", ctypes.c_int32 * 3), ("pad_", ctypes.c_int32), ("l0", ctypes.c_int64),
                ("n_l", ctypes.c_int64)]

    @property
    def n_q(self):
        return int(self.plane.n_h * self.plane.n_k * self.n_l)


class Step(ctypes.Structure):
    """xpcs_step (include/xpcs.h): one host-buffer pass of the whole hot path."""
    _fields_ = [("positions", ctypes.c_void_p), ("form_factors", ctypes.c_void_p), ("species", ctypes.c_void_p),
                ("N", ctypes.c_int64), ("frames", ctypes.c_int64), ("grid", QGrid), ("q_vectors", ctypes.c_void_p),
                ("n_q", ctypes.c_int64), ("box_L", ctypes.c_double), ("bin_of_q", ctypes.c_void_p),
                ("n_bins", ctypes.c_int32), ("batches", ctypes.c_int32), ("lags", ctypes.POINTER(ctypes.c_int32)),
                ("n_lags", ctypes.c_int64), ("windows", ctypes.POINTER(ctypes.c_int32)), ("n_windows", ctypes.c_int64),
                ("I_out", ctypes.c_void_p), ("g2_out", ctypes.c_void_p), ("S_rings", ctypes.c_void_p),
                ("g2_rings", ctypes.c_void_p), ("beta", ctypes.c_void_p)]


class Species(ctypes.Structure):
    _fields_ = [("n_species", ctypes.c_int32), ("pad_", ctypes.c_int32), ("species", ctypes.POINTER(ctypes.c_int32)),
                ("f_q", ctypes.c_void_p), ("f_max", ctypes.POINTER(ctypes.c_double))]


_lib = None


def load():
    """Load libxpcs.so (raises if it has not been built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} not built (run `python -c 'import __graft_entry__ as g; g.build()'`)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    op = ctypes.POINTER(Opts)
    gp = ctypes.POINTER(QGrid)
    ip32 = ctypes.POINTER(ctypes.c_int32)
    sig = {
        "xpcs_intensity": [vp, i64, vp, vp, i64, i64, dbl, vp, op],
        "xpcs_intensity_grid": [vp, i64, vp, gp, i64, vp, op],
        "xpcs_g2": [vp, i64, i64, ip32, i64, vp, op],
        "xpcs_g2_accumulate": [vp, i64, i64, i64, ip32, i64, vp, i64, vp, vp, op],
        "xpcs_g2_finalize": [vp, vp, i64, i64, ip32, i64, vp, op],
        "xsvs_contrast": [vp, i64, i64, vp, i32, ip32, i64, vp, op],
        "xpcs_shell_mean": [vp, i64, i64, vp, i32, dbl, vp, op],
        "xpcs_structure_factor_shells": [vp, i64, i64, vp, i64, vp, i32, vp, op],
        "xpcs_qgrid_lattice_plane": [dbl, i64, i32, gp],
        "xpcs_qgrid_ewald": [dbl, i64, i64, dbl, vp, op],
        "xpcs_lattice_bins": [gp, i32, i32, vp, op],
        "xpcs_radial_bins": [vp, i64, dbl, i32, vp, op],
        "xpcs_last_error": [],
        "xpcs_release": [],
        "xpcs_launch_count": [],
        "xpcs_profile_reset": [],
        "xpcs_profile_query": [i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_int64)],
        "xpcs_device_info": [ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)],
        "xpcs_version": [],
        "xpcs_engine_available": [i32],
        "xpcs_amplitude": [vp, i64, vp, vp, i64, i64, dbl, vp, op],
        "xpcs_amplitude_grid": [vp, i64, vp, gp, i64, vp, op],
        "xpcs_isf": [vp, i64, i64, ip32, i64, vp, i64, vp, op],
        "xpcs_intensity_volume": [vp, i64, vp, ctypes.POINTER(Species), ctypes.POINTER(QVolume), i64, vp, op],
        "xpcs_amplitude_volume": [vp, i64, vp, ctypes.POINTER(Species), ctypes.POINTER(QVolume), i64, vp, op],
        "xpcs_intensity_species": [vp, i64, ctypes.POINTER(Species), vp, i64, i64, dbl, vp, op],
        "xpcs_amplitude_species": [vp, i64, ctypes.POINTER(Species), vp, i64, i64, dbl, vp, op],
        "xpcs_rings_register": [vp, i64, i32, op],
        "xpcs_rings_unregister": [vp],
        "xpcs_intensity_fft": [vp, i64, i64, ctypes.POINTER(QVolume), i32, dbl, i32, vp, vp, op],
        "xpcs_speckle_histogram": [vp, i64, i64, vp, i32, i32, i32, dbl, vp, op],
        "xpcs_form_factor_gaussian": [vp, i64, ctypes.POINTER(QVolume), i32, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double), dbl, vp, op],
        "xpcs_step_host": [ctypes.POINTER(Step), op],
        "xpcs_ring_moments": [vp, i64, i64, vp, i32, vp, op],
        "xpcs_ring_means_from_moments": [vp, i64, i32, dbl, vp, i64, vp, op],
        "xsvs_moments": [vp, i64, i64, vp, i32, ip32, i64, vp, op],
        "xsvs_contrast_from_moments": [vp, i64, ip32, i64, i32, vp, op],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.xpcs_last_error.restype = ctypes.c_char_p
    L.xpcs_launch_count.restype = ctypes.c_int64
    _lib = L
    return L


def _check(rc):
    if rc != XPCS_OK:
        raise XpcsError(rc, load().xpcs_last_error().decode())


def _dtype_code(t):
    import torch
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise TypeError(f"unsupported dtype {t.dtype}")


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("xpcs: tensors must live in device memory (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("xpcs: tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


_WORKSPACE = threading.local()


def make_opts(in_dtype=F32, out_dtype=F32, stream=None, engine=ENGINE_AUTO, profile=False):
    return Opts(in_dtype, out_dtype, _stream(stream), engine, 1 if profile else 0, getattr(_WORKSPACE, "id", 0), 0)


_ws_counter = itertools.count(1)


def new_workspace() -> int:
    """A fresh scratch workspace id (xpcs_opts.workspace) for one user of the library, e.g. one Pipeline."""
    return next(_ws_counter)


class workspace:
    """Context manager: library calls made inside use scratch workspace `ws_id` (0 = per-stream default)."""

    def __init__(self, ws_id: int):
        self.ws_id = int(ws_id)

    def __enter__(self):
        self.prev = getattr(_WORKSPACE, "id", 0)
        _WORKSPACE.id = self.ws_id
        return self

    def __exit__(self, *a):
        _WORKSPACE.id = self.prev


def _i32_array(seq):
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.int32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


# --------------------------------------------------------------------------------------------- API
def lattice_plane(L, n, l=0) -> QGrid:
    g = QGrid()
    _check(load().xpcs_qgrid_lattice_plane(float(L), int(n), int(l), ctypes.byref(g)))
    return g


def qgrid(L, h0, n_h, k0, n_k, m0=(0, 0, 0), ma=(1, 0, 0), mb=(0, 1, 0)) -> QGrid:
    g = QGrid()
    g.L = float(L)
    g.m0[:], g.ma[:], g.mb[:] = list(m0), list(ma), list(mb)
    g.h0, g.n_h, g.k0, g.n_k = int(h0), int(n_h), int(k0), int(n_k)
    return g


def qvolume(L, h0, n_h, k0, n_k, l0, n_l, m0=(0, 0, 0), ma=(1, 0, 0), mb=(0, 1, 0), mc=(0, 0, 1)) -> QVolume:
    """3-D reciprocal-lattice block q = (2 pi / L)(m0 + h ma + k mb + l mc), output order (l, h, k)."""
    v = QVolume()
    v.plane = qgrid(L, h0, n_h, k0, n_k, m0, ma, mb)
    v.mc[:] = list(mc)
    v.l0, v.n_l = int(l0), int(n_l)
    return v


def _host_ptr(t):
    if t is None:
        return None
    if t.is_cuda:
        raise ValueError("xpcs: this argument is a HOST buffer")
    if not t.is_contiguous():
        raise ValueError("xpcs: tensors must be contiguous")
    return t.data_ptr()


def xpcs_step_host(positions, form_factors, grid, bins, n_bins, lags=(), windows=(), I_out=None, g2_out=None,
                   S_rings=None, g2_rings=None, beta=None, species=None, batches=8, engine=ENGINE_AUTO, stream=None,
                   profile=False, out_dtype=None, q_vectors=None, box_L=0.0):
    """xpcs_step_host: the whole hot path from HOST buffers (positions [T][N][3], optional form factors [N]; pinned
    for overlap) into HOST outputs (any may be None).  `bins` is the DEVICE ring index [n_q]; `species` an optional
    (host species [N], device f_q [S][n_q], f_max) triple.  Enqueued on `stream`; outputs valid after it syncs."""
    import torch
    T, N = positions.shape[0], positions.shape[1]
    ind = F64 if positions.dtype == torch.float64 else F32
    outd = ind if out_dtype is None else out_dtype
    st = Step()
    st.positions = _host_ptr(positions)
    st.form_factors = _host_ptr(form_factors)
    keep = []
    if species is not None:
        sp, keep = species_desc(*species)
        keep = (sp, keep)
        st.species = ctypes.addressof(sp)
    st.N, st.frames = N, T
    if q_vectors is not None:
        st.q_vectors, st.n_q, st.box_L = _ptr(q_vectors).value, q_vectors.shape[0], float(box_L)
    else:
        st.grid = grid
    st.bin_of_q = _ptr(bins).value
    st.n_bins, st.batches = int(n_bins), int(batches)
    l_arr, l_p = _i32_array(lags) if len(lags) else (None, None)
    w_arr, w_p = _i32_array(windows) if len(windows) else (None, None)
    st.lags, st.n_lags = l_p, len(lags)
    st.windows, st.n_windows = w_p, len(windows)
    st.I_out, st.g2_out = _host_ptr(I_out), _host_ptr(g2_out)
    st.S_rings, st.g2_rings, st.beta = _host_ptr(S_rings), _host_ptr(g2_rings), _host_ptr(beta)
    o = make_opts(ind, outd, stream, engine, profile)
    _check(load().xpcs_step_host(ctypes.byref(st), ctypes.byref(o)))
    return keep, l_arr, w_arr


def species_desc(species, f_q, f_max=None):
    """xpcs_species from a host int array species [N], a device table f_q [n_species][n_q] and optional host
    per-kind max |f_s| hints (kept alive by the returned tuple's second element)."""
    sp = np.ascontiguousarray(np.asarray(species, dtype=np.int32))
    d = Species()
    d.n_species = int(f_q.shape[0])
    d.species = sp.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    d.f_q = _ptr(f_q)
    fm = None
    if f_max is not None:
        fm = np.ascontiguousarray(np.asarray(f_max, dtype=np.float64))
        assert fm.shape == (d.n_species,)
        d.f_max = fm.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    return d, (sp, f_q, fm)


def _positions3(positions, *same_dtype, form_factors=None, q_vectors=None):
    """[T][N][3] view of positions ([N][3] accepted) and argument checks the C ABI cannot make: every float
    array of the call shares the positions' dtype (one in_dtype), form_factors has N entries, q has 3 columns."""
    if positions.dim() == 2:
        positions = positions.unsqueeze(0)
    if positions.dim() != 3 or positions.shape[2] != 3:
        raise ValueError(f"xpcs: positions must be [T][N][3] (got {tuple(positions.shape)})")
    for t in (form_factors, q_vectors) + tuple(same_dtype):
        if t is not None and t.dtype != positions.dtype:
            raise TypeError(f"xpcs: all float arrays of a call share the positions' dtype ({positions.dtype}, got {t.dtype})")
    if form_factors is not None and form_factors.numel() != positions.shape[1]:
        raise ValueError(f"xpcs: form_factors has {form_factors.numel()} entries for N = {positions.shape[1]} atoms")
    if q_vectors is not None and (q_vectors.dim() != 2 or q_vectors.shape[1] != 3):
        raise ValueError(f"xpcs: q_vectors must be [n_q][3] (got {tuple(q_vectors.shape)})")
    return positions


def xpcs_intensity_volume(positions, form_factors, vol: QVolume, species=None, f_q=None, out=None, out_dtype=None,
                          engine=ENGINE_AUTO, stream=None, profile=False, amplitude=False, f_max=None):
    """Eq.(7)-(8) on a 3-D lattice block (species/f_q: q-dependent form factors) -> I [T][n_l * n_h * n_k]
    (amplitude=True: p as [..][2])."""
    import torch
    positions = _positions3(positions, f_q, form_factors=form_factors)
    T, N = positions.shape[0], positions.shape[1]
    ind = _dtype_code(positions)
    outd = ind if out_dtype is None else out_dtype
    shape = (T, vol.n_q, 2) if amplitude else (T, vol.n_q)
    if out is None:
        out = torch.empty(shape, dtype=torch.float64 if outd == F64 else torch.float32, device=positions.device)
    o = make_opts(ind, outd, stream, engine, profile)
    sp, keep = (species_desc(species, f_q, f_max) if species is not None else (None, None))
    fn = load().xpcs_amplitude_volume if amplitude else load().xpcs_intensity_volume
    _check(fn(_ptr(positions), N, _ptr(form_factors), ctypes.byref(sp) if sp is not None else None,
              ctypes.byref(vol), T, _ptr(out), ctypes.byref(o)))
    del keep
    return out


def xpcs_intensity_species(positions, species, f_q, q_vectors, box_L, out=None, out_dtype=None, stream=None,
                           profile=False, amplitude=False, f_max=None):
    """Eq.(7)-(8) at an explicit q list with q-dependent form factors f_q [n_species][n_q] -> I [T][n_q]."""
    import torch
    positions = _positions3(positions, f_q, q_vectors=q_vectors)
    T, N = positions.shape[0], positions.shape[1]
    n_q = q_vectors.shape[0]
    ind = _dtype_code(positions)
    outd = ind if out_dtype is None else out_dtype
    shape = (T, n_q, 2) if amplitude else (T, n_q)
    if out is None:
        out = torch.empty(shape, dtype=torch.float64 if outd == F64 else torch.float32, device=positions.device)
    o = make_opts(ind, outd, stream, ENGINE_AUTO, profile)
    sp, keep = species_desc(species, f_q, f_max)
    fn = load().xpcs_amplitude_species if amplitude else load().xpcs_intensity_species
    _check(fn(_ptr(positions), N, ctypes.byref(sp), _ptr(q_vectors), n_q, T, float(box_L), _ptr(out),
              ctypes.byref(o)))
    del keep
    return out


def xpcs_form_factor_gaussian(a, b, c, q_vectors=None, vol: QVolume = None, out_dtype=F32, in_dtype=F32,
                              device="cuda", stream=None):
    """f(q) = c + sum_i a_i exp(-b_i (|q|/4 pi)^2) at a q list or every q of a volume -> [n_q]."""
    import torch
    n_q = q_vectors.shape[0] if q_vectors is not None else vol.n_q
    out = torch.empty(n_q, dtype=torch.float64 if out_dtype == F64 else torch.float32,
                      device=q_vectors.device if q_vectors is not None else device)
    ad = (ctypes.c_double * max(1, len(a)))(*[float(x) for x in a])
    bd = (ctypes.c_double * max(1, len(b)))(*[float(x) for x in b])
    o = make_opts(_dtype_code(q_vectors) if q_vectors is not None else in_dtype, out_dtype, stream)
    _check(load().xpcs_form_factor_gaussian(_ptr(q_vectors), n_q, ctypes.byref(vol) if vol is not None else None,
                                            len(a), ad, bd, float(c), _ptr(out), ctypes.byref(o)))
    return out


def xpcs_intensity(positions, form_factors, q_vectors, box_L, out=None, out_dtype=None, stream=None, profile=False):
    """Eq.(7)-(8) at an explicit q list.  positions [T][N][3], q [n_q][3] (same dtype), -> I [T][n_q]."""
    import torch
    positions = _positions3(positions, form_factors=form_factors, q_vectors=q_vectors)
    T, N = positions.shape[0], positions.shape[1]
    n_q = q_vectors.shape[0]
    ind = _dtype_code(positions)
    outd = ind if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty((T, n_q), dtype=torch.float64 if outd == F64 else torch.float32, device=positions.device)
    o = make_opts(ind, outd, stream, ENGINE_AUTO, profile)
    _check(load().xpcs_intensity(_ptr(positions), N, _ptr(form_factors), _ptr(q_vectors), n_q, T, float(box_L),
                                 _ptr(out), ctypes.byref(o)))
    return out


def xpcs_intensity_grid(positions, form_factors, grid: QGrid, out=None, out_dtype=None, engine=ENGINE_AUTO,
                        stream=None, profile=False):
    """Eq.(7)-(8) on a reciprocal-lattice plane (exact integer phases).  -> I [T][n_h * n_k]."""
    import torch
    positions = _positions3(positions, form_factors=form_factors)
    T, N = positions.shape[0], positions.shape[1]
    ind = _dtype_code(positions)
    outd = ind if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty((T, grid.n_q), dtype=torch.float64 if outd == F64 else torch.float32,
                          device=positions.device)
    o = make_opts(ind, outd, stream, engine, profile)
    _check(load().xpcs_intensity_grid(_ptr(positions), N, _ptr(form_factors), ctypes.byref(grid), T, _ptr(out),
                                      ctypes.byref(o)))
    return out


def xpcs_amplitude(positions, form_factors, q_vectors, box_L, out=None, out_dtype=None, stream=None):
    """Eq.(7) complex amplitude at an explicit q list -> [T][n_q][2] (Re, Im)."""
    import torch
    positions = _positions3(positions, form_factors=form_factors, q_vectors=q_vectors)
    T, N = positions.shape[0], positions.shape[1]
    n_q = q_vectors.shape[0]
    ind = _dtype_code(positions)
    outd = ind if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty((T, n_q, 2), dtype=torch.float64 if outd == F64 else torch.float32, device=positions.device)
    o = make_opts(ind, outd, stream)
    _check(load().xpcs_amplitude(_ptr(positions), N, _ptr(form_factors), _ptr(q_vectors), n_q, T, float(box_L),
                                 _ptr(out), ctypes.byref(o)))
    return out


def xpcs_amplitude_grid(positions, form_factors, grid: QGrid, out=None, out_dtype=None, engine=ENGINE_AUTO,
                        stream=None):
    """Eq.(7) complex amplitude on a lattice plane -> [T][n_h * n_k][2] (Re, Im)."""
    import torch
    positions = _positions3(positions, form_factors=form_factors)
    T, N = positions.shape[0], positions.shape[1]
    ind = _dtype_code(positions)
    outd = ind if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty((T, grid.n_q, 2), dtype=torch.float64 if outd == F64 else torch.float32,
                          device=positions.device)
    o = make_opts(ind, outd, stream, engine)
    _check(load().xpcs_amplitude_grid(_ptr(positions), N, _ptr(form_factors), ctypes.byref(grid), T, _ptr(out),
                                      ctypes.byref(o)))
    return out


def xpcs_isf(A, lags, form_factors=None, N=None, out=None, stream=None):
    """Eq.(22) intermediate scattering function from an amplitude series A [T][n_q][2] -> F [n_lags][n_q][2]."""
    import torch
    T, n_q = A.shape[0], A.shape[1]
    lag_arr, lag_p = _i32_array(lags)
    if N is None:
        N = form_factors.shape[0] if form_factors is not None else 1
    if out is None:
        out = torch.empty((len(lag_arr), n_q, 2), dtype=torch.float64, device=A.device)
    o = make_opts(_dtype_code(A), F64, stream)
    _check(load().xpcs_isf(_ptr(A), T, n_q, lag_p, len(lag_arr), _ptr(form_factors), int(N), _ptr(out),
                           ctypes.byref(o)))
    return out


def xpcs_g2(I, lags, out=None, out_dtype=F64, stream=None, profile=False):
    """Eq.(14) per pixel. I [T][n_q] -> g2 [n_lags][n_q]."""
    import torch
    T, n_q = I.shape
    lag_arr, lag_p = _i32_array(lags)
    if out is None:
        out = torch.empty((len(lag_arr), n_q), dtype=torch.float64 if out_dtype == F64 else torch.float32,
                          device=I.device)
    o = make_opts(_dtype_code(I), out_dtype, stream, ENGINE_AUTO, profile)
    _check(load().xpcs_g2(_ptr(I), T, n_q, lag_p, len(lag_arr), _ptr(out), ctypes.byref(o)))
    return out


def xpcs_g2_accumulate(I_block, t0, lags, ring, acc, sum_, stream=None, profile=False):
    """Block-streamed g2 (include/xpcs.h): add the pairs whose later frame is in I_block [B][n_q] (global frames
    t0 .. t0+B-1) to acc [n_lags][n_q] and the block's frames to sum_ [n_q] (float64); ring [R][n_q] (R >= max lag,
    I_block's dtype) holds the last frames and is updated by the library."""
    B, n_q = I_block.shape
    lag_arr, lag_p = _i32_array(lags)
    o = make_opts(_dtype_code(I_block), F64, stream, ENGINE_AUTO, profile)
    _check(load().xpcs_g2_accumulate(_ptr(I_block), B, int(t0), n_q, lag_p, len(lag_arr), _ptr(ring),
                                     ring.shape[0] if ring is not None else 0, _ptr(acc), _ptr(sum_), ctypes.byref(o)))


def xpcs_g2_finalize(acc, sum_, frames, lags, out=None, out_dtype=F64, stream=None):
    """g2 [n_lags][n_q] of the streamed series of `frames` frames from the accumulated state."""
    import torch
    n_q = sum_.shape[0]
    lag_arr, lag_p = _i32_array(lags)
    if out is None:
        out = torch.empty((len(lag_arr), n_q), dtype=torch.float64 if out_dtype == F64 else torch.float32,
                          device=acc.device)
    o = make_opts(F64, out_dtype, stream)
    _check(load().xpcs_g2_finalize(_ptr(acc), _ptr(sum_), int(frames), n_q, lag_p, len(lag_arr), _ptr(out),
                                   ctypes.byref(o)))
    return out


class G2Stream:
    """Owns the block-streamed g2 state (acc, sum, frame ring) for one detector: push(I_block) per block of frames in
    order, result() = xpcs_g2 of everything pushed.  Buffers only; the arithmetic is in the library."""

    def __init__(self, n_q, lags, dtype=None, device="cuda", stream=None):
        import torch
        self.lags = tuple(int(t) for t in lags)
        self.n_q, self.t, self.stream = int(n_q), 0, stream
        dtype = dtype or torch.float32
        self.acc = torch.zeros((len(self.lags), self.n_q), dtype=torch.float64, device=device)
        self.sum = torch.zeros((self.n_q,), dtype=torch.float64, device=device)
        R = max(self.lags) if self.lags else 0
        self.ring = torch.empty((R, self.n_q), dtype=dtype, device=device) if R > 0 else None

    def push(self, I_block):
        xpcs_g2_accumulate(I_block, self.t, self.lags, self.ring, self.acc, self.sum, stream=self.stream)
        self.t += I_block.shape[0]

    def result(self, out=None, out_dtype=F64):
        return xpcs_g2_finalize(self.acc, self.sum, self.t, self.lags, out=out, out_dtype=out_dtype,
                                stream=self.stream)


def xsvs_contrast(I, bins, n_bins, windows, out=None, stream=None, profile=False):
    """Eq.(15)+(17): beta [n_windows][n_bins] (float64)."""
    import torch
    T, n_q = I.shape
    w_arr, w_p = _i32_array(windows)
    if out is None:
        out = torch.empty((len(w_arr), n_bins), dtype=torch.float64, device=I.device)
    o = make_opts(_dtype_code(I), F64, stream, ENGINE_AUTO, profile)
    _check(load().xsvs_contrast(_ptr(I), T, n_q, _ptr(bins), int(n_bins), w_p, len(w_arr), _ptr(out),
                                ctypes.byref(o)))
    return out


def xpcs_intensity_fft(positions, block: QVolume, n_grid, eta, k_cut=0, f_q=None, out=None, out_dtype=None,
                       stream=None, profile=False):
    """Algorithm 2 (FFT method): I on an axis-aligned block of the n_grid^3 FFT grid -> [T][n_l * n_h * n_k]."""
    import torch
    positions = _positions3(positions, f_q)
    T, N = positions.shape[0], positions.shape[1]
    ind = _dtype_code(positions)
    outd = ind if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty((T, block.n_q), dtype=torch.float64 if outd == F64 else torch.float32,
                          device=positions.device)
    o = make_opts(ind, outd, stream, ENGINE_AUTO, profile)
    _check(load().xpcs_intensity_fft(_ptr(positions), N, T, ctypes.byref(block), int(n_grid), float(eta), int(k_cut),
                                     _ptr(f_q), _ptr(out), ctypes.byref(o)))
    return out


def xpcs_rings_register(bins, n_bins, stream=None):
    """Build and keep the ring plan of a device bin array (reused by every ring reduction given the same tensor)."""
    o = make_opts(stream=stream)
    _check(load().xpcs_rings_register(_ptr(bins), bins.shape[0], int(n_bins), ctypes.byref(o)))


def xpcs_rings_unregister(bins):
    _check(load().xpcs_rings_unregister(_ptr(bins)))


def xpcs_speckle_histogram(I, bins, n_bins, M, n_hist, kappa_max, out=None, stream=None, profile=False):
    """Eq.(37)-(38) statistics: counts of kappa = I_M / <I_M>_ring -> int64 [n_bins][n_hist]."""
    import torch
    T, n_q = I.shape
    if out is None:
        out = torch.empty((n_bins, n_hist), dtype=torch.int64, device=I.device)
    o = make_opts(_dtype_code(I), F64, stream, ENGINE_AUTO, profile)
    _check(load().xpcs_speckle_histogram(_ptr(I), T, n_q, _ptr(bins), int(n_bins), int(M), int(n_hist),
                                         float(kappa_max), _ptr(out), ctypes.byref(o)))
    return out


def xpcs_ring_moments(values, bins, n_bins, out=None, stream=None, profile=False):
    """Additive ring moments [rows][n_bins][2] = (count of finite values, sum) (float64, device)."""
    import torch
    if values.dim() == 1:
        values = values.unsqueeze(0)
    rows, n_q = values.shape
    if out is None:
        out = torch.empty((rows, n_bins, 2), dtype=torch.float64, device=values.device)
    o = make_opts(_dtype_code(values), F64, stream, ENGINE_AUTO, profile)
    _check(load().xpcs_ring_moments(_ptr(values), rows, n_q, _ptr(bins), int(n_bins), _ptr(out), ctypes.byref(o)))
    return out


def xpcs_ring_means_from_moments(moments, scale=1.0, form_factors=None, N=0, out=None, stream=None):
    """scale * sum / count per (row, ring) from [rows][n_bins][2] moments, / sum f^2 when form_factors is given."""
    import torch
    rows, n_bins = moments.shape[0], moments.shape[1]
    if out is None:
        out = torch.empty((rows, n_bins), dtype=torch.float64, device=moments.device)
    ind = _dtype_code(form_factors) if form_factors is not None else F32
    o = make_opts(ind, F64, stream)
    _check(load().xpcs_ring_means_from_moments(_ptr(moments), rows, int(n_bins), float(scale), _ptr(form_factors),
                                               int(N), _ptr(out), ctypes.byref(o)))
    return out


def xsvs_n_slots(frames, windows):
    return int(sum(int(frames) // int(w) for w in windows))


def xsvs_moments(I, bins, n_bins, windows, out=None, stream=None, profile=False):
    """XSVS moments [n_slots][n_bins][3] = (ring pixel count, sum I_W, sum I_W^2) (float64, device)."""
    import torch
    T, n_q = I.shape
    w_arr, w_p = _i32_array(windows)
    if out is None:
        out = torch.empty((xsvs_n_slots(T, windows), n_bins, 3), dtype=torch.float64, device=I.device)
    o = make_opts(_dtype_code(I), F64, stream, ENGINE_AUTO, profile)
    _check(load().xsvs_moments(_ptr(I), T, n_q, _ptr(bins), int(n_bins), w_p, len(w_arr), _ptr(out), ctypes.byref(o)))
    return out


def xsvs_contrast_from_moments(moments, frames, windows, out=None, stream=None):
    import torch
    n_bins = moments.shape[1]
    w_arr, w_p = _i32_array(windows)
    if out is None:
        out = torch.empty((len(w_arr), n_bins), dtype=torch.float64, device=moments.device)
    o = make_opts(F32, F64, stream)
    _check(load().xsvs_contrast_from_moments(_ptr(moments), int(frames), w_p, len(w_arr), int(n_bins), _ptr(out),
                                             ctypes.byref(o)))
    return out


def xpcs_shell_mean(values, bins, n_bins, scale=1.0, out=None, stream=None, profile=False):
    import torch
    if values.dim() == 1:
        values = values.unsqueeze(0)
    rows, n_q = values.shape
    if out is None:
        out = torch.empty((rows, n_bins), dtype=torch.float64, device=values.device)
    o = make_opts(_dtype_code(values), F64, stream, ENGINE_AUTO, profile)
    _check(load().xpcs_shell_mean(_ptr(values), rows, n_q, _ptr(bins), int(n_bins), float(scale), _ptr(out),
                                  ctypes.byref(o)))
    return out


def xpcs_structure_factor_shells(I, form_factors, N, bins, n_bins, out=None, stream=None, profile=False):
    import torch
    rows, n_q = I.shape
    if out is None:
        out = torch.empty((rows, n_bins), dtype=torch.float64, device=I.device)
    o = make_opts(_dtype_code(I), F64, stream, ENGINE_AUTO, profile)
    _check(load().xpcs_structure_factor_shells(_ptr(I), rows, n_q, _ptr(form_factors), int(N), _ptr(bins),
                                               int(n_bins), _ptr(out), ctypes.byref(o)))
    return out


def xpcs_qgrid_ewald(wavelength, npx, npy, pitch, out_dtype=F32, device="cuda", stream=None):
    import torch
    out = torch.empty((npx * npy, 3), dtype=torch.float64 if out_dtype == F64 else torch.float32, device=device)
    o = make_opts(F32, out_dtype, stream)
    _check(load().xpcs_qgrid_ewald(float(wavelength), int(npx), int(npy), float(pitch), _ptr(out), ctypes.byref(o)))
    return out


def xpcs_lattice_bins(grid: QGrid, n_bins, w, device="cuda", stream=None):
    import torch
    out = torch.empty(grid.n_q, dtype=torch.int32, device=device)
    o = make_opts(stream=stream)
    _check(load().xpcs_lattice_bins(ctypes.byref(grid), int(n_bins), int(w), _ptr(out), ctypes.byref(o)))
    return out


def xpcs_radial_bins(q, q_max, n_bins, stream=None):
    import torch
    out = torch.empty(q.shape[0], dtype=torch.int32, device=q.device)
    o = make_opts(_dtype_code(q), F32, stream)
    _check(load().xpcs_radial_bins(_ptr(q), q.shape[0], float(q_max), int(n_bins), _ptr(out), ctypes.byref(o)))
    return out


def engine_resolved(engine, uniform_f=True) -> int:
    """The engine a lattice f32 call with this opts.engine runs (mirrors api.cu): AUTO -> the integer tensor engine
    for uniform form factors, the split-FP16 tensor engine otherwise; SIMT when tcgen05 is unavailable."""
    if engine == ENGINE_SIMT or not engine_available(ENGINE_TENSOR):
        return ENGINE_SIMT
    if engine == ENGINE_AUTO:
        return ENGINE_TENSOR_I8 if (uniform_f and AUTO_I8) else ENGINE_TENSOR
    return engine


AUTO_I8 = True    # AUTO routes uniform-f lattice calls to the integer engine (mirrors api.cu)


I8_BUDGET = float(os.environ.get("XPCS_I8_BUDGET", "2.5"))   # mirror of api.cu's kI8BudgetDefault (env: experiments)


def species_engines(counts, f_max=None, budget=None):
    """Mirror of api.cu's AUTO rule for species calls: kinds in increasing |f_max| go to the integer engine while
    sum (f_max / f_min)^2 N_s / N <= budget (default I8_BUDGET = 2.5); the kind that crosses the budget is split (its first atoms on the integer
    engine up to the budget), the rest run on split-FP16.  Without f_max hints every kind runs on split-FP16.
    Returns the number of atoms of each kind on the integer engine."""
    counts = [int(c) for c in counts]
    n = len(counts)
    if f_max is None:
        return [0] * n
    order = sorted(range(n), key=lambda k: abs(f_max[k]))
    fref = next((abs(f_max[k]) for k in order if counts[k] > 0 and abs(f_max[k]) > 0), 0.0)
    total = max(1, sum(counts))
    cap = I8_BUDGET if budget is None else float(budget)
    out, budget = [0] * n, 0.0
    for k in order:
        w2 = (f_max[k] / fref) ** 2 if fref > 0 else 1.0
        room = cap + 1e-12 - budget
        take = counts[k]
        if room <= 0:
            take = 0
        elif w2 * counts[k] / total > room:
            take = int(math.floor(room * total / w2))
        take = min(take, counts[k])
        out[k] = take
        budget += w2 * take / total
    return out


def launch_count() -> int:
    return int(load().xpcs_launch_count())


def profile_reset():
    _check(load().xpcs_profile_reset())


def profile_query():
    """{class name: (total ms, launches)} for every kernel class (synchronises on the recorded events)."""
    out = {}
    for i in range(len(KERNEL_CLASSES)):
        name = ctypes.c_char_p()
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        _check(load().xpcs_profile_query(i, ctypes.byref(name), ctypes.byref(ms), ctypes.byref(n)))
        out[name.value.decode()] = (ms.value, n.value)
    return out


def release():
    _check(load().xpcs_release())


def engine_available(engine) -> bool:
    return bool(load().xpcs_engine_available(int(engine)))


def device_info():
    sm = ctypes.c_int32()
    clk = ctypes.c_int32()
    _check(load().xpcs_device_info(ctypes.byref(sm), ctypes.byref(clk)))
    return sm.value, clk.value
