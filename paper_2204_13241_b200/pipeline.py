"""One pass of the whole hot path for a workload, through the C ABI.

    I(q,t)      xpcs_intensity_grid (lattice plane) | xpcs_intensity (explicit q, e.g. Ewald detector)
    g2(q,tau)   xpcs_g2                               Eq.(14)
    S_b(t)      xpcs_structure_factor_shells          Eq.(12)-(13), ring average PAPER.md:192
    g2_b(tau)   xpcs_shell_mean(g2)                   ring-averaged g2
    beta_{W,b}  xsvs_contrast                         Eq.(15)+(17)

This module is orchestration only (which ABI call, with which buffers); it contains no arithmetic of the method.
``run_host`` is the end-to-end entry a user calls with host arrays: pinned host -> device copy of the step's
inputs, the device pass, and the device -> host copy of its results.
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np
import torch

from . import _lib as X


@dataclasses.dataclass
class Workload:
    name: str
    N: int
    L: float
    T: int
    n_plane: int = 0            # lattice plane n x n (0 = explicit q list)
    q: torch.Tensor | None = None   # explicit q [n_q][3] (device) when n_plane == 0
    q_max: float = 0.0          # ring range for explicit q
    lags: tuple = ()
    windows: tuple = ()
    n_bins: int = 32
    in_dtype: int = X.F32
    engine: int = X.ENGINE_AUTO
    # optional atom kinds for per-atom form factors with few distinct values (f_j = kind_f[kinds[j]]): the intensity
    # then goes through the species path, which lets AUTO put the light kinds on the integer engine
    kinds: np.ndarray | None = None
    kind_f: tuple = ()


class Pipeline:
    def __init__(self, wl: Workload, device="cuda", stream=None):
        self.wl = wl
        self.device = torch.device(device)
        self.stream = stream
        if wl.n_plane:
            self.grid = X.lattice_plane(wl.L, wl.n_plane, 0)
            self.n_q = self.grid.n_q
            # ring unit w = n / (2 n_bins) pixels: rings cover the inscribed disk |h|,|k| < n/2 (R8)
            self.bins = X.xpcs_lattice_bins(self.grid, wl.n_bins, wl.n_plane // (2 * wl.n_bins), self.device, stream)
        else:
            assert wl.q is not None
            self.grid = None
            self.n_q = wl.q.shape[0]
            self.bins = X.xpcs_radial_bins(wl.q, wl.q_max, wl.n_bins, stream)
        # the detector geometry is fixed for the workload: build its ring plan once (reused by every reduction)
        X.xpcs_rings_register(self.bins, wl.n_bins, stream)
        self._registered = True
        odt = torch.float64 if wl.in_dtype == X.F64 else torch.float32
        self.kind_fq = None
        if wl.kinds is not None and self.grid is not None:
            # constant rows f_s(q) = kind_f[s] on the plane, as the 3-D block of one l-plane
            self.vol = X.qvolume(wl.L, self.grid.h0, self.grid.n_h, self.grid.k0, self.grid.n_k, 0, 1,
                                 m0=tuple(self.grid.m0), ma=tuple(self.grid.ma), mb=tuple(self.grid.mb))
            kf = torch.tensor(list(wl.kind_f), dtype=odt, device=self.device)
            self.kind_fq = kf[:, None].expand(len(wl.kind_f), self.n_q).contiguous()
        self.I = torch.empty((wl.T, self.n_q), dtype=odt, device=self.device)
        self.g2 = torch.empty((len(wl.lags), self.n_q), dtype=torch.float32, device=self.device) if wl.lags else None
        # the reductions of I are independent (g2 -> g2 rings | XSVS | S rings) and each is too small to fill the
        # GPU alone: they run concurrently on two side streams and the caller's stream, joined before returning
        self.s_red = [torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)] if self.device.type == "cuda" else None
        self.serial_reductions = False      # True: all reductions on the caller's stream (per-kernel timing)
        # own library scratch (xpcs_opts.workspace): pipelines replayed concurrently never share buffers, even when
        # torch hands out recycled pool streams
        self.ws = X.new_workspace()

    def close(self):
        """Free the registered ring plan (the bins tensor dies with the pipeline; a stale plan must not outlive it)."""
        if getattr(self, "bins", None) is not None and getattr(self, "_registered", False):
            try:
                X.xpcs_rings_unregister(self.bins)
            except Exception:
                pass
            self._registered = False

    def __del__(self):
        self.close()

    @property
    def pairs_per_step(self) -> int:
        return int(self.wl.N) * int(self.n_q) * int(self.wl.T)

    def run(self, positions: torch.Tensor, form_factors: torch.Tensor | None, profile=False) -> dict:
        with X.workspace(self.ws):
            return self._run(positions, form_factors, profile)

    def _run(self, positions, form_factors, profile):
        wl, s = self.wl, self.stream
        if self.kind_fq is not None:
            X.xpcs_intensity_volume(positions, None, self.vol, species=wl.kinds, f_q=self.kind_fq, out=self.I,
                                    engine=wl.engine, stream=s, profile=profile, f_max=wl.kind_f)
        elif self.grid is not None:
            X.xpcs_intensity_grid(positions, form_factors, self.grid, out=self.I, engine=wl.engine, stream=s,
                                  profile=profile)
        else:
            X.xpcs_intensity(positions, form_factors, wl.q, wl.L, out=self.I, stream=s, profile=profile)
        out = {"I": self.I}
        self._reductions(out, self.I, form_factors, s, profile)
        return out

    def _reductions(self, out, I, form_factors, s, profile=False, after_g2=None):
        """g2 + g2 rings on side stream 0, XSVS on side stream 1, S rings on the caller's stream s; joined into s.
        after_g2(stream): optional hook enqueued on side stream 0 right after g2 (e.g. its D2H copy)."""
        wl = self.wl
        main = s if s is not None else torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(main)
        r0, r1 = self.s_red
        if self.serial_reductions or os.environ.get("XPCS_SERIAL_REDUCTIONS") == "1":   # isolated kernel timings
            r0 = r1 = main
        r0.wait_event(ev)
        r1.wait_event(ev)
        skip = os.environ.get("XPCS_SKIP_REDUCTIONS", "").split(",")   # experiments: critical-path attribution
        if wl.lags and "g2" not in skip:
            X.xpcs_g2(I, wl.lags, out=self.g2, out_dtype=X.F32, stream=r0, profile=profile)
            out["g2"] = self.g2
            if after_g2 is not None:
                after_g2(r0)
            out["g2_rings"] = X.xpcs_shell_mean(self.g2, self.bins, wl.n_bins, stream=r0, profile=profile)
        if wl.windows and "xsvs" not in skip:
            out["beta"] = X.xsvs_contrast(I, self.bins, wl.n_bins, wl.windows, stream=r1, profile=profile)
        if "rings" not in skip:
            out["S_rings"] = X.xpcs_structure_factor_shells(I, form_factors, wl.N, self.bins, wl.n_bins, stream=main,
                                                            profile=profile)
        main.wait_stream(r0)
        main.wait_stream(r1)

    # ---------------------------------------------------------------- CUDA graphs of a step
    def _capture(self, fn, warmup=2, warm_fn=None):
        """Capture fn() (one whole step, all streams forked from and joined into the capture stream) into a CUDA
        graph.  The library's scratch, lag tables and ring plan are sized by `warmup` eager calls on the capture
        stream first (nothing is allocated inside the capture).  Returns (graph, fn's result); graph.replay() reruns
        the step on the same buffers."""
        cur = torch.cuda.current_stream(self.device)
        cs = torch.cuda.Stream(self.device)
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            for _ in range(warmup):
                (warm_fn or fn)()
        cur.wait_stream(cs)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        n0 = X.launch_count()
        with torch.cuda.graph(g, stream=cs):
            res = fn()
        self.capture_launches = X.launch_count() - n0     # library kernels per replay
        torch.cuda.synchronize(self.device)
        return g, res

    def capture(self, positions: torch.Tensor, form_factors: torch.Tensor | None, profile=False):
        """CUDA graph of run(positions, form_factors): replay() recomputes I, g2, rings and XSVS from the current
        contents of `positions` (same tensor).  With profile=True the library's kernel-class events are external
        event-record nodes (xpcs_profile_query() after a replay reads that replay's times)."""
        return self._capture(lambda: self.run(positions, form_factors, profile=profile),
                             warm_fn=lambda: self.run(positions, form_factors))

    def capture_host(self):
        """CUDA graph of run_host() (needs alloc_host_io): H2D of the pinned inputs, the step, D2H of every result."""
        return self._capture(self.run_host)

    # ---------------------------------------------------------------- end to end from host memory
    def alloc_host_io(self, pos_host: np.ndarray, f_host: np.ndarray | None, batches: int = 4):
        """Pinned host copies of the inputs (allocated once, reused per step); the pinned result buffers are made by
        the first run_host.  `batches`: frame batches of the copy / compute overlap inside xpcs_step_host."""
        self.h_pos = torch.from_numpy(np.ascontiguousarray(pos_host)).pin_memory()
        self.h_f = torch.from_numpy(np.ascontiguousarray(f_host)).pin_memory() if f_host is not None else None
        self.h_out = {}
        self.n_batches = max(1, min(int(batches), self.wl.T))

    def run_host(self) -> dict:
        """End to end from pinned host memory: one `xpcs_step_host` call (the C ABI's host-buffer entry: frame-batched
        H2D / intensity / D2H overlap on internal copy streams, then g2, rings and XSVS and their D2H), enqueued on
        the current stream (lattice planes and explicit q lists)."""
        with X.workspace(self.ws):
            return self._run_host()

    def _run_host(self):
        wl = self.wl
        main = torch.cuda.current_stream(self.device)
        h = self.h_out
        T, nl, nw, nb = wl.T, len(wl.lags), len(wl.windows), wl.n_bins
        if "I" not in h:
            pin = dict(pin_memory=True)
            h["I"] = torch.empty(self.I.shape, dtype=self.I.dtype, **pin)
            h["S_rings"] = torch.empty((T, nb), dtype=torch.float64, **pin)
            if nl:
                h["g2"] = torch.empty((nl, self.n_q), dtype=torch.float32, **pin)
                h["g2_rings"] = torch.empty((nl, nb), dtype=torch.float64, **pin)
            if nw:
                h["beta"] = torch.empty((nw, nb), dtype=torch.float64, **pin)
        sp = (wl.kinds, self.kind_fq, wl.kind_f) if self.kind_fq is not None else None
        self._keep = X.xpcs_step_host(self.h_pos, self.h_f, self.grid, self.bins, nb, lags=wl.lags, windows=wl.windows,
                                      I_out=h["I"], g2_out=h.get("g2"), S_rings=h["S_rings"],
                                      g2_rings=h.get("g2_rings"), beta=h.get("beta"), species=sp,
                                      batches=self.n_batches, engine=wl.engine, stream=main,
                                      out_dtype=X.F64 if self.I.dtype == torch.float64 else X.F32,
                                      q_vectors=wl.q if self.grid is None else None, box_L=wl.L)
        return h

    def io_bytes(self):
        h2d = self.h_pos.numel() * self.h_pos.element_size()
        if self.h_f is not None:
            h2d += self.h_f.numel() * self.h_f.element_size()
        d2h = sum(v.numel() * v.element_size() for v in self.h_out.values())
        return h2d, d2h


def workload_from_config(cfg, device="cuda", stream=None) -> Workload:
    """Map an xpcs_inputs.Config onto the pipeline (geometry computed on the device for explicit-q configs)."""
    import xpcs_inputs as xi
    in_dtype = X.F64 if cfg.dtype == "f64" else X.F32
    if cfg.n_plane:
        kinds, kind_f = None, ()
        if cfg.two_species and in_dtype == X.F32:
            f = xi.form_factors(cfg)
            kind_f = tuple(float(v) for v in np.unique(f))
            kinds = np.searchsorted(np.asarray(kind_f, dtype=f.dtype), f).astype(np.int32)
        return Workload(cfg.name, cfg.N, cfg.L, cfg.T, n_plane=cfg.n_plane, lags=tuple(cfg.lags),
                        windows=tuple(cfg.windows), n_bins=cfg.n_bins, in_dtype=in_dtype, kinds=kinds, kind_f=kind_f)
    q = X.xpcs_qgrid_ewald(xi.EWALD_WAVELENGTH_SIGMA, cfg.detector, cfg.detector, xi.EWALD_PITCH_RAD,
                           out_dtype=in_dtype, device=device, stream=stream)
    return Workload(cfg.name, cfg.N, cfg.L, cfg.T, n_plane=0, q=q, q_max=xi.EWALD_QMAX, lags=tuple(cfg.lags),
                    windows=tuple(cfg.windows), n_bins=cfg.n_bins, in_dtype=in_dtype)


class MomentLayout:
    """The q-sharded step's single FP64 all-reduce buffer: [S moments T x n_bins x 2 | g2 moments n_lags x n_bins x 2 |
    XSVS moments n_slots x n_bins x 3] (the layouts of xpcs_ring_moments and xsvs_moments, include/xpcs.h).  Pure
    indexing: the arithmetic is in the library."""

    def __init__(self, T, n_lags, n_slots, n_bins):
        self.T, self.n_lags, self.n_slots, self.n_bins = int(T), int(n_lags), int(n_slots), int(n_bins)
        self.sizes = [self.T * self.n_bins * 2, self.n_lags * self.n_bins * 2, self.n_slots * self.n_bins * 3]
        self.offsets = [0, self.sizes[0], self.sizes[0] + self.sizes[1]]
        self.total = sum(self.sizes)

    def views(self, m):
        """(S [T][nb][2], g2 [n_lags][nb][2] or None, XSVS [n_slots][nb][3] or None) views of a flat buffer m."""
        o, nb = self.offsets, self.n_bins
        mS = m[o[0]:o[1]].view(self.T, nb, 2)
        mG = m[o[1]:o[2]].view(self.n_lags, nb, 2) if self.n_lags else None
        mX = m[o[2]:].view(self.n_slots, nb, 3) if self.n_slots else None
        return mS, mG, mX


class QShardPipeline:
    """One trajectory on a detector split across ranks ("partition by q ... each GPU then owns complete
    time series, so g2 stays local; shell sums need one small all-reduce"; the q vectors are
    independent).  Lattice planes are split into 2-D blocks aligned to the tensor engines' 256 (h) x 128 (k) pair
    tiles (dist.qblocks); explicit q lists (config 4's Ewald detector) into contiguous pixel ranges.  Rank r computes
    I and g2 on its block (atom kinds included: the kinds' f_q rows cover the block), the additive ring moments of I
    (S rings), of g2 (g2 rings) and the XSVS moments on its pixels, all-reduces the moments once (one flat FP64
    buffer, MomentLayout: NCCL on GPUs), and forms S_b(t), g2_b(tau) and beta_{W,b} from the sums -- equal to the
    single-device reductions up to summation order.  Orchestration only: every step is an ABI call; `allreduce(t)`
    sums a device tensor in place over the ranks (torch.distributed.all_reduce when a process group exists)."""

    def __init__(self, wl: Workload, rank: int, world: int, device="cuda", allreduce=None):
        from . import dist as xd
        self.wl, self.rank, self.world = wl, rank, world
        self.device = torch.device(device)
        self.ws = X.new_workspace()
        odt = torch.float64 if wl.in_dtype == X.F64 else torch.float32
        self.kind_fq = None
        if wl.n_plane:
            full = X.lattice_plane(wl.L, wl.n_plane, 0)
            (h0, n_h, k0, n_k), self.block = xd.qblocks(full.n_h, full.n_k, full.h0, full.k0, rank, world)
            self.full = full
            self.grid = X.qgrid(wl.L, h0, n_h, k0, n_k, tuple(full.m0), tuple(full.ma), tuple(full.mb))
            self.n_q = self.grid.n_q
            self.q = None
            self.bins = X.xpcs_lattice_bins(self.grid, wl.n_bins, wl.n_plane // (2 * wl.n_bins), self.device)
            if wl.kinds is not None:
                self.vol = X.qvolume(wl.L, h0, n_h, k0, n_k, 0, 1, m0=tuple(full.m0), ma=tuple(full.ma),
                                     mb=tuple(full.mb))
                kf = torch.tensor(list(wl.kind_f), dtype=odt, device=self.device)
                self.kind_fq = kf[:, None].expand(len(wl.kind_f), self.n_q).contiguous()
        else:
            lo, hi = xd.shard(wl.q.shape[0], rank, world)
            self.block = (lo, hi)
            self.grid = None
            self.q = wl.q[lo:hi].contiguous()
            self.n_q = hi - lo
            self.bins = X.xpcs_radial_bins(self.q, wl.q_max, wl.n_bins)
        X.xpcs_rings_register(self.bins, wl.n_bins)
        self.I = torch.empty((wl.T, self.n_q), dtype=odt, device=self.device)
        self.g2 = torch.empty((len(wl.lags), self.n_q), dtype=torch.float32, device=self.device) if wl.lags else None
        self.n_slots = X.xsvs_n_slots(wl.T, wl.windows) if wl.windows else 0
        self.layout = MomentLayout(wl.T, len(wl.lags), self.n_slots, wl.n_bins)
        self.mom = torch.zeros(self.layout.total, dtype=torch.float64, device=self.device)
        self.mS, self.mG, self.mX = self.layout.views(self.mom)
        self._allreduce = allreduce if allreduce is not None else self._default_allreduce

    @staticmethod
    def _default_allreduce(t):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

    @property
    def pairs_per_step(self) -> int:
        return int(self.wl.N) * int(self.n_q) * int(self.wl.T)

    def local(self, positions, form_factors, profile=False):
        """This rank's block: I, g2 and the ring / XSVS moments (before the all-reduce)."""
        wl = self.wl
        with X.workspace(self.ws):
            if self.kind_fq is not None:
                X.xpcs_intensity_volume(positions, None, self.vol, species=wl.kinds, f_q=self.kind_fq, out=self.I,
                                        engine=wl.engine, profile=profile, f_max=wl.kind_f)
            elif self.grid is not None:
                X.xpcs_intensity_grid(positions, form_factors, self.grid, out=self.I, engine=wl.engine, profile=profile)
            else:
                X.xpcs_intensity(positions, form_factors, self.q, wl.L, out=self.I, profile=profile)
            X.xpcs_ring_moments(self.I, self.bins, wl.n_bins, out=self.mS, profile=profile)
            if wl.lags:
                X.xpcs_g2(self.I, wl.lags, out=self.g2, out_dtype=X.F32, profile=profile)
                X.xpcs_ring_moments(self.g2, self.bins, wl.n_bins, out=self.mG, profile=profile)
            if self.n_slots:
                X.xsvs_moments(self.I, self.bins, wl.n_bins, wl.windows, out=self.mX, profile=profile)
        return self.mom

    def finish(self, form_factors, moments=None):
        """Ring results from (summed) moments."""
        wl = self.wl
        mS, mG, mX = self.layout.views(self.mom if moments is None else moments)
        out = {"I": self.I}
        with X.workspace(self.ws):
            if form_factors is not None:
                out["S_rings"] = X.xpcs_ring_means_from_moments(mS, 1.0, form_factors, wl.N)
            else:
                out["S_rings"] = X.xpcs_ring_means_from_moments(mS, 1.0 / wl.N)
            if wl.lags:
                out["g2"] = self.g2
                out["g2_rings"] = X.xpcs_ring_means_from_moments(mG)
            if self.n_slots:
                out["beta"] = X.xsvs_contrast_from_moments(mX, wl.T, wl.windows)
        return out

    def run(self, positions, form_factors, profile=False):
        self.local(positions, form_factors, profile)
        self._allreduce(self.mom)
        return self.finish(form_factors)

    def close(self):
        try:
            X.xpcs_rings_unregister(self.bins)
        except Exception:
            pass


QSlabPipeline = QShardPipeline   # round-1 name
