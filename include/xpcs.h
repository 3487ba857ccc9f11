/*
 * xpcs.h -- C ABI of libxpcs.so, the B200 (sm_100a) implementation of the direct method of
 * S. Mohanty, C. B. Cooper, H. Wang, M. Liang, W. Cai, "Computational Approaches to Model X-ray Photon
 * Correlation Spectroscopy from Molecular Dynamics", arXiv 2204.13241 (cited as PAPER.md:<line>).
 *
 * Conventions shared by every entry point
 *  - Array pointers are DEVICE pointers owned by the caller unless marked HOST; arrays are contiguous
 *    and row-major.  Structs passed by pointer (xpcs_opts, xpcs_qgrid) live in HOST memory.
 *  - All work is enqueued on opts->stream (a cudaStream_t; NULL = the legacy default stream).  Calls
 *    return as soon as the work is enqueued; outputs are valid after that stream is synchronised.
 *  - Return value: 0 (XPCS_OK) or a positive xpcs_status.  A human-readable message for the most recent
 *    failure of the calling thread is returned by xpcs_last_error().  No C++ exception crosses the ABI.
 *    An asynchronous CUDA fault from earlier work is reported as XPCS_ECUDA by the next call.
 *  - Argument validation happens before any work is enqueued: on XPCS_EINVAL nothing was launched.
 *  - The library owns only internal scratch (cached per device, grown on demand); xpcs_release() frees it.
 *  - There is no CPU fallback: every step runs in this library's CUDA kernels.
 */
#ifndef XPCS_H_
#define XPCS_H_

#include <stdint.h>

#if defined(__GNUC__)
#define XPCS_API __attribute__((visibility("default")))
#else
#define XPCS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    XPCS_OK = 0,
    XPCS_EINVAL = 1,       /* bad argument (null pointer, size <= 0, lag >= frames, window out of range, ...) */
    XPCS_ECUDA = 2,        /* CUDA runtime error (launch failure or an earlier asynchronous fault)        */
    XPCS_ENOMEM = 3,       /* device scratch allocation failed                                            */
    XPCS_EUNSUPPORTED = 4  /* valid request this build does not implement (e.g. engine not available)     */
} xpcs_status;

typedef enum { XPCS_F32 = 0, XPCS_F64 = 1 } xpcs_dtype;

/* Which kernel family evaluates a lattice-grid contraction (xpcs_intensity_grid / _volume, f32 only).
 * AUTO picks the fastest available engine that meets the north_star tolerance for the call: TENSOR_I8 when
 * form_factors is NULL (f = 1, and every kind of a species call), TENSOR for per-atom form factors, SIMT without
 * tcgen05 (XPCS_DISABLE_TC=1); SIMT = FP32 CUDA-core
 * factorised kernel; TENSOR = tcgen05 split-FP16 kernel (FP32-class products, per-pixel |dI| ~ 1e-4 N at most);
 * TENSOR_I8 = tcgen05 integer kernel (two int8 limbs per phasor component, exact int32 accumulation; per-pixel
 * rms |dI| ~ 3e-5 N (f = 1), W scaled by max |f_j| for per-atom form factors).  The generic q-list path ignores
 * this field. */
typedef enum { XPCS_ENGINE_AUTO = 0, XPCS_ENGINE_SIMT = 1, XPCS_ENGINE_TENSOR = 2, XPCS_ENGINE_TENSOR_I8 = 3 } xpcs_engine;

typedef struct {
    int32_t in_dtype;   /* xpcs_dtype of positions / form factors / q vectors, or of the intensity series fed to
                           xpcs_g2, xsvs_contrast, xpcs_shell_mean                                              */
    int32_t out_dtype;  /* xpcs_dtype of I_out (xpcs_intensity*) and g2_out (xpcs_g2)                          */
    void*   stream;     /* cudaStream_t; NULL = legacy default stream                                           */
    int32_t engine;     /* xpcs_engine (lattice grids only)                                                     */
    int32_t profile;    /* nonzero: time the dominant kernels with CUDA events (see xpcs_profile_query)        */
    int32_t workspace;  /* 0: library scratch cached per (device, stream); k > 0: per (device, k, stream), so that
                           callers replaying CUDA graphs concurrently (one workspace id each) never share scratch
                           even if their streams are recycled.  A scratch buffer that a graph capture has used is
                           never freed before xpcs_release (a later, larger call gets a new buffer).          */
    int32_t pad_;
} xpcs_opts;

/* A plane of the reciprocal lattice of a cubic periodic box of edge L (Algorithm 1 step 1,
 * PAPER.md:295): pixel (ih, ik), 0 <= ih < n_h, 0 <= ik < n_k, has integer indices h = h0 + ih, k = k0 + ik and
 *     q = (2 pi / L) (m0 + h * ma + k * mb),
 * with integer 3-vectors m0, ma, mb.  Pixel index = ih * n_k + ik.  The configs' detector plane is
 * m0 = 0, ma = (1,0,0), mb = (0,1,0), h0 = k0 = -n/2, n_h = n_k = n (xpcs_qgrid_lattice_plane). */
typedef struct {
    double  L;
    int32_t m0[3];
    int32_t ma[3];
    int32_t mb[3];
    int32_t pad_;
    int64_t h0, n_h, k0, n_k;
} xpcs_qgrid;

/* ------------------------------------------------------------------------------------------------
 * Speckle intensity by the direct method.
 * Eq.(7):  p^e(q,t) = sum_j f_j exp(-i q . r_j(t));  Eq.(8), PAPER.md:134-138:
 * I(q,t) = |p^e(q,t)|^2;  Algorithm 1, evaluated for every q and every frame.
 *
 * xpcs_intensity: an explicit list of q vectors (any q, e.g. Ewald-sphere detector pixels).
 *   positions    [frames][N][3] in_dtype  atom positions r_j(t); wrapped into [0, box_L)^3 before use
 *                                          (reading R3: off-lattice q sees this image choice)
 *   N            atoms per frame (> 0)
 *   form_factors [N] in_dtype or NULL      q-independent f_j (NULL: f_j = 1)  (R2)
 *   q_vectors    [n_q][3] in_dtype         diffraction vectors q = k_f - k_i (Eq. 1)
 *   n_q, frames  > 0
 *   box_L        > 0, periodic box edge (same length unit as 1/|q|)
 *   I_out        [frames][n_q] out_dtype
 * Errors: EINVAL for null positions / q_vectors / I_out, N, n_q, frames <= 0, box_L <= 0 or non-finite,
 *         unknown dtype.  Positions are read as given: NaN/Inf inputs propagate into I_out. */
XPCS_API int xpcs_intensity(const void* positions, int64_t N, const void* form_factors,
                   const void* q_vectors, int64_t n_q, int64_t frames, double box_L,
                   void* I_out, const xpcs_opts* opts);

/* xpcs_intensity_grid: q on a reciprocal-lattice plane (host struct *grid).  Same output as xpcs_intensity
 * with the q list of the grid, but the library forms every phase from the exact integers (h, k, m0, ma, mb)
 * and L (R9: q is never rounded to fp32) and evaluates the per-axis factorisation
 *     p^e(h,k) = sum_j X_h(j) W_k(j),  X_h = e^{-2 pi i h (ma . r_j)/L},  W_k = f_j e^{-2 pi i (m0 + k mb) . r_j / L}
 * on the engine selected by opts->engine.
 *   I_out [frames][n_h * n_k] out_dtype.
 * Errors: as xpcs_intensity, plus EINVAL for n_h, n_k <= 0 or |indices| too large for 32-bit turns,
 *         EUNSUPPORTED if opts->engine = TENSOR is requested for f64 inputs. */
XPCS_API int xpcs_intensity_grid(const void* positions, int64_t N, const void* form_factors,
                        const xpcs_qgrid* grid, int64_t frames, void* I_out, const xpcs_opts* opts);

/* Complex amplitude p^e(q,t) = sum_j f_j exp(-i q . r_j(t)) itself (Eq. 7, the paper's sign),
 * for the intermediate scattering function (Eq. 22) and any analysis that needs phases.  Same arguments and
 * engines as xpcs_intensity / xpcs_intensity_grid; A_out [frames][n_q][2] out_dtype = (Re p, Im p). */
XPCS_API int xpcs_amplitude(const void* positions, int64_t N, const void* form_factors,
                   const void* q_vectors, int64_t n_q, int64_t frames, double box_L,
                   void* A_out, const xpcs_opts* opts);
XPCS_API int xpcs_amplitude_grid(const void* positions, int64_t N, const void* form_factors,
                        const xpcs_qgrid* grid, int64_t frames, void* A_out, const xpcs_opts* opts);

/* ------------------------------------------------------------------------------------------------
 * 3-D blocks of the reciprocal lattice and q-dependent atomic form factors.
 *
 * xpcs_qvolume: n_l stacked lattice planes (Algorithm 1 step 1; the 81 x 81 x 81 grid of Table 1,
 * PAPER.md:459): plane il (0 <= il < n_l) is `plane` with m0 replaced by m0 + (l0 + il) mc, i.e.
 *     q = (2 pi / L) (m0 + h ma + k mb + l mc),   l = l0 + il,
 * output index (il * n_h + ih) * n_k + ik.  A plane is the n_l = 1 case. */
typedef struct {
    xpcs_qgrid plane;
    int32_t mc[3];
    int32_t pad_;
    int64_t l0, n_l;
} xpcs_qvolume;

/* Atom kinds with q-dependent form factors (Eq.(2): f_i(q); f is the Fourier
 * transform of the atom's electron density, e.g. a sum of Gaussians, see xpcs_form_factor_gaussian):
 *     p(q,t) = sum_j f_{species[j]}(q) exp(-i q . r_j(t)).
 *   n_species  1 .. 16
 *   species    HOST [N] int32, each in [0, n_species): atoms are gathered per kind on the device (the permutation is
 *              built on the host and uploaded once per call; the array may be freed when the call returns)
 *   f_q        DEVICE [n_species][n_q_total] in_dtype: f_s at every output q (n_q_total = n_q for a q list,
 *              n_l * n_h * n_k for a volume, same q order as the output) */
typedef struct {
    int32_t n_species;
    int32_t pad_;
    const int32_t* species;
    const void* f_q;
    const double* f_max;   /* HOST [n_species] or NULL: max_q |f_s(q)| per kind, a hint for AUTO's engine choice
                              (lightest kinds on the integer engine while sum f_max^2 N_s / (f_min^2 N) <= 2.5, the kind
                              crossing the budget split at it, the rest on the split-FP16 engine; NULL: AUTO runs
                              every kind on the split-FP16 engine, XPCS_ENGINE_TENSOR_I8 every kind on the integer
                              engine) */
} xpcs_species;

/* xpcs_intensity_volume / xpcs_amplitude_volume: I (or p, as (re, im) pairs) on a 3-D lattice block for every
 * frame, by the same exact-turn factorised engines as xpcs_intensity_grid (each (frame, l-plane) pair is one
 * plane contraction).  species == NULL: per-atom q-independent form_factors [N] (NULL => 1) as in
 * xpcs_intensity_grid; species != NULL: q-dependent f_s(q) (form_factors must then be NULL).
 *   I_out [frames][n_l][n_h][n_k] out_dtype (amplitude: [..][2]).
 * Errors: as xpcs_intensity_grid, plus EINVAL for vol NULL, n_l <= 0, |l| too large, form_factors together with
 *         species, n_species outside [1, 16], a species index out of range, f_q NULL. */
XPCS_API int xpcs_intensity_volume(const void* positions, int64_t N, const void* form_factors,
                                   const xpcs_species* species, const xpcs_qvolume* vol, int64_t frames,
                                   void* I_out, const xpcs_opts* opts);
XPCS_API int xpcs_amplitude_volume(const void* positions, int64_t N, const void* form_factors,
                                   const xpcs_species* species, const xpcs_qvolume* vol, int64_t frames,
                                   void* A_out, const xpcs_opts* opts);
/* xpcs_intensity_species / xpcs_amplitude_species: explicit q list (as xpcs_intensity) with q-dependent
 * form factors; species must not be NULL.  Errors: as xpcs_intensity plus the species errors above. */
XPCS_API int xpcs_intensity_species(const void* positions, int64_t N, const xpcs_species* species,
                                    const void* q_vectors, int64_t n_q, int64_t frames, double box_L,
                                    void* I_out, const xpcs_opts* opts);
XPCS_API int xpcs_amplitude_species(const void* positions, int64_t N, const xpcs_species* species,
                                    const void* q_vectors, int64_t n_q, int64_t frames, double box_L,
                                    void* A_out, const xpcs_opts* opts);
/* Algorithm 2, the FFT-based method (a cross-check / second workload beside the direct method):
 * rho^eta = sum_i of normalised Gaussians of width eta (Eq. 30) on an n_grid^3 grid of the periodic box, each evaluated
 * on the k x k x k grid points nearest the atom (k = k_cut, or for k_cut <= 0 the paper's "nearest integer greater
 * than 10 eta" in grid spacings, rounded up to odd: DESIGN.md R16); p^eta = FFT(rho^eta) (cuFFT,
 * FP64); f^eta = the DFT of the truncated Gaussian centred at the origin; I = f(q)^2 |p^eta|^2 /
 * f^eta^2 (Eq. 35).  Output: the axis-aligned block `block` of the FFT grid (block->plane.L is the box edge; m0 = 0,
 * ma = x, mb = y, mc = z; every index in [-n_grid/2, n_grid/2 - 1]), order [frames][n_l][n_h][n_k] out_dtype.
 *   positions [frames][N][3] in_dtype (wrapped into the box);  f_q DEVICE [n_l*n_h*n_k] in_dtype or NULL (f = 1).
 * Deposits use FP64 atomics, so the last bits of rho (and of I) may differ between runs.
 * Errors: EINVAL for null pointers, N/frames <= 0, a non-axis-aligned block or indices outside the grid, n_grid odd
 *         or outside [8, 1024], eta <= 0, k even or > 31; ECUDA for CUDA/cuFFT failures. */
XPCS_API int xpcs_intensity_fft(const void* positions, int64_t N, int64_t frames, const xpcs_qvolume* block,
                                int32_t n_grid, double eta, int32_t k_cut, const void* f_q, void* I_out,
                                const xpcs_opts* opts);
/* Gaussian-sum form factor: f(q) = c + sum_{i < n_gauss} a_i exp(-b_i s^2), s = |q| / (4 pi),
 * evaluated in FP64 at an explicit q list (q_vectors DEVICE [n_q][3] in_dtype) or, if q_vectors is NULL, at every
 * q of the volume *vol (n_q ignored).  a, b HOST [n_gauss], 0 <= n_gauss <= 6.  f_out DEVICE [n_q] out_dtype.
 * Errors: EINVAL for f_out NULL, both q_vectors and vol NULL, n_q <= 0 with a q list, n_gauss outside [0, 6],
 *         a/b NULL with n_gauss > 0. */
XPCS_API int xpcs_form_factor_gaussian(const void* q_vectors, int64_t n_q, const xpcs_qvolume* vol, int32_t n_gauss,
                                       const double* a, const double* b, double c, void* f_out,
                                       const xpcs_opts* opts);

/* Intermediate scattering function, Eq.(22), PAPER.md:218-223:
 *   F(q, tau) = (1 / (T - tau)) sum_{t=0}^{T-1-tau} p(q,t) p*(q, t+tau)  /  sum_j f_j^2
 * (time average over the T - tau available pairs; sum_j f_j^2 reduced on the device from form_factors, NULL => N).
 * F(q,0) = S(q) (Eq. 12); the normalised F^ = F(tau)/F(0) of Eq.(23) and the Siegert relation g2 = 1 + beta0 |F^|^2
 * (Eq. 24) are formed from these outputs.
 *   A_series [frames][n_q][2] in_dtype;  lags HOST [n_lags] (0 <= lag < frames, <= 320);
 *   F_out DEVICE [n_lags][n_q][2] double.
 * Errors: EINVAL for null pointers, sizes <= 0, lags out of range; EUNSUPPORTED for lags > 320. */
XPCS_API int xpcs_isf(const void* A_series, int64_t frames, int64_t n_q, const int32_t* lags, int64_t n_lags,
             const void* form_factors, int64_t N, double* F_out, const xpcs_opts* opts);

/* ------------------------------------------------------------------------------------------------
 * Intensity autocorrelation, Eq.(14), PAPER.md:170-174 (literal estimator, R6), per pixel:
 *   num(tau) = 1/(T - tau) sum_{t=0}^{T-1-tau} I_t I_{t+tau},  den = ((1/T) sum_t I_t)^2,  g2 = num / den.
 * tau = 0 gives beta0 + 1 (Eq. 19).  Products and sums in FP64.
 *   I_series [frames][n_q] in_dtype;  lags HOST [n_lags], 0 <= lag < frames;  g2_out [n_lags][n_q] out_dtype.
 * A pixel whose mean intensity is 0 gets g2 = NaN.
 * Errors: EINVAL for null pointers, frames/n_q/n_lags <= 0, any lag outside [0, frames). */
XPCS_API int xpcs_g2(const void* I_series, int64_t frames, int64_t n_q, const int32_t* lags, int64_t n_lags,
            void* g2_out, const xpcs_opts* opts);

/* Block-streamed g2 (SURVEY 8(d) K4 "update in blocks of B frames"; Eq.(14)): for series longer
 * than device memory (PAPER.md:476 uses 5000 frames) the frames arrive in blocks and only the FP64 state and the
 * last max-lag frames stay resident.  Same estimator and FP64 arithmetic as xpcs_g2: after streaming frames
 * 0 .. T-1 in any block sizes, xpcs_g2_finalize gives xpcs_g2 of the whole series (up to summation order).
 * xpcs_g2_accumulate, for the block I_block [block_frames][n_q] in_dtype holding global frames t0 .. t0+B-1:
 *     acc[l][px] += sum of I_t I_{t+tau_l} over the pairs whose LATER frame t + tau_l is in the block and t >= 0,
 *     sum[px]    += sum of the block's frames,
 *   the earlier frames before the block coming from `ring` DEVICE [ring_frames][n_q] in_dtype (frame g in slot
 *   g mod ring_frames, ring_frames >= max lag; the library writes the block's last min(B, ring_frames) frames into it
 *   after reading it: the caller allocates it and never writes it).  acc DEVICE [n_lags][n_q] and sum DEVICE [n_q]
 *   double are zeroed by the caller before the first block (t0 = 0).  Blocks must arrive in order (t0 = frames
 *   already streamed), all with the same lags and ring, on one stream (or ordered streams).
 * xpcs_g2_finalize: g2_out [n_lags][n_q] out_dtype = (acc / (T - tau)) / (sum / T)^2 for the total frame count T
 *   (NaN where the mean intensity is 0).
 * Errors: EINVAL for null pointers, sizes <= 0, t0 < 0, a negative lag, ring_frames < max lag (or a NULL ring with
 * ring_frames > 0), a lag >= frames in finalize; EUNSUPPORTED for lags > 640. */
XPCS_API int xpcs_g2_accumulate(const void* I_block, int64_t block_frames, int64_t t0, int64_t n_q,
                                const int32_t* lags, int64_t n_lags, void* ring, int64_t ring_frames, double* acc,
                                double* sum, const xpcs_opts* opts);
XPCS_API int xpcs_g2_finalize(const double* acc, const double* sum, int64_t frames, int64_t n_q, const int32_t* lags,
                              int64_t n_lags, void* g2_out, const xpcs_opts* opts);

/* ------------------------------------------------------------------------------------------------
 * XSVS optical contrast versus exposure.  Eq.(15), as a discrete unnormalised sum over
 * non-overlapping windows of W frames aligned at t = 0 (remainder dropped):
 *     I_W(q, s) = sum_{t=sW}^{sW+W-1} I(q, t),   s = 0 .. floor(T/W) - 1;
 * Eq.(17), per snapshot and q-ring b (population variance over the ring's pixels):
 *     beta_{W,b,s} = (<I_W^2>_b - <I_W>_b^2) / <I_W>_b^2,
 * then averaged over the snapshots s.  Moments in FP64.
 *   I_series [frames][n_q] in_dtype;  bin_of_q DEVICE [n_q] int32 ring index in [0, n_bins) or -1 (excluded);
 *   windows HOST [n_windows] (1 <= W <= frames);  beta_out DEVICE [n_windows][n_bins] double.
 * An empty ring gives NaN.
 * Errors: EINVAL for null pointers, frames/n_q/n_windows <= 0, n_bins <= 0, any window outside [1, frames]. */
XPCS_API int xsvs_contrast(const void* I_series, int64_t frames, int64_t n_q,
                  const int32_t* bin_of_q, int32_t n_bins,
                  const int32_t* windows, int64_t n_windows,
                  double* beta_out, const xpcs_opts* opts);

/* Speckle intensity statistics (kappa = I / <I>_q over a q ring follows exp(-kappa), Eq.(37), for a
 * coherent beam; the incoherent superposition of M independent patterns follows the Erlang law of
 * Eq.(38) with contrast 1/M).  With I_M(q, s) = sum_{t=sM}^{sM+M-1} I(q, t), s = 0 .. floor(T/M) - 1 (remainder
 * dropped) and kappa = I_M(q, s) / <I_M(., s)>_{ring b} (ring mean over the ring's pixels, FP64), counts kappa over
 * all pixels and snapshots into n_hist bins of width kappa_max / n_hist on [0, kappa_max), bin
 * h = floor((kappa * n_hist) / kappa_max); kappa >= kappa_max is not counted; a ring/snapshot with mean <= 0 is skipped.
 *   I_series [frames][n_q] in_dtype; bin_of_q DEVICE [n_q] (-1 = excluded); counts_out DEVICE [n_bins][n_hist] int64.
 * The counts are exact integers; only a kappa within ~1e-15 relative of a bin edge can land differently from a
 * summation in another order.  Errors: EINVAL for null pointers, sizes <= 0, M outside [1, frames], n_hist outside
 * [1, 2^20], kappa_max <= 0 or non-finite. */
XPCS_API int xpcs_speckle_histogram(const void* I_series, int64_t frames, int64_t n_q, const int32_t* bin_of_q,
                                    int32_t n_bins, int32_t M, int32_t n_hist, double kappa_max, int64_t* counts_out,
                                    const xpcs_opts* opts);

/* Additive ring moments (a detector split into slabs across devices adds these -- e.g. with one
 * NCCL all-reduce -- and then forms the ring means and the XSVS contrast exactly as the single-device calls do).
 * xpcs_ring_moments: moments_out DEVICE [rows][n_bins][2] = (count of finite values, their sum) per ring and row,
 *   for values [rows][n_q] in_dtype (I for S(q,t), g2 for the ring-averaged g2).
 * xpcs_ring_means_from_moments: out DEVICE [rows][n_bins] = scale * sum / count (NaN for count 0), divided by
 *   sum_j f_j^2 reduced on the device from form_factors [N] (in_dtype) when form_factors != NULL (S(q), Eq. 12-13).
 * xsvs_moments: moments_out DEVICE [n_slots][n_bins][3] = (m0 = ring pixel count, m1 = sum I_W, m2 = sum I_W^2) for
 *   every window W (in list order) and snapshot s = 0 .. floor(frames/W) - 1, slot = (windows before W) + s;
 *   n_slots = sum_W floor(frames / W) (Eq. 15 windows, as xsvs_contrast).
 * xsvs_contrast_from_moments: beta_out DEVICE [n_windows][n_bins] from (summed) moments, Eq.(17) per snapshot then
 *   the mean over snapshots; NaN for a ring with m0 = 0.
 * Errors: EINVAL for null pointers, sizes <= 0, windows outside [1, frames]. */
XPCS_API int xpcs_ring_moments(const void* values, int64_t rows, int64_t n_q, const int32_t* bin_of_q, int32_t n_bins,
                               double* moments_out, const xpcs_opts* opts);
XPCS_API int xpcs_ring_means_from_moments(const double* moments, int64_t rows, int32_t n_bins, double scale,
                                          const void* form_factors, int64_t N, double* out, const xpcs_opts* opts);
XPCS_API int xsvs_moments(const void* I_series, int64_t frames, int64_t n_q, const int32_t* bin_of_q, int32_t n_bins,
                          const int32_t* windows, int64_t n_windows, double* moments_out, const xpcs_opts* opts);
XPCS_API int xsvs_contrast_from_moments(const double* moments, int64_t frames, const int32_t* windows,
                                        int64_t n_windows, int32_t n_bins, double* beta_out, const xpcs_opts* opts);

/* Ring plans.  Every ring reduction (xsvs_contrast, xpcs_shell_mean, xpcs_structure_factor_shells,
 * xpcs_speckle_histogram) first groups the detector pixels by ring (a deterministic counting sort of bin_of_q, three
 * small kernels).  xpcs_rings_register builds that plan once for a DEVICE bin_of_q array (n_q entries, n_bins rings)
 * and keeps it (device memory owned by the library); later reductions that pass the same pointer with the same
 * (n_q, n_bins) on the same device reuse it.  The caller must not modify the array while it is registered.
 * xpcs_rings_unregister synchronises the device and frees the plan; xpcs_release frees all plans.
 * Errors: EINVAL for null bin_of_q, n_q <= 0, n_bins outside [1, 12288], an unregistered pointer (unregister);
 *         ENOMEM/ECUDA from the allocation or the build. */
XPCS_API int xpcs_rings_register(const int32_t* bin_of_q, int64_t n_q, int32_t n_bins, const xpcs_opts* opts);
XPCS_API int xpcs_rings_unregister(const int32_t* bin_of_q);

/* Ring average of any per-pixel quantity, per row:
 *   out[r][b] = scale * mean_{q in ring b, values finite} values[r][q]   (NaN if no finite value),
 * e.g. the ring-averaged g2(q, tau) or, with scale = 1 / sum_j f_j^2, the structure factor
 * S(q,t) of Eq.(12)/(13) (see xpcs_structure_factor_shells).
 *   values [rows][n_q] in_dtype; bin_of_q DEVICE [n_q]; out DEVICE [rows][n_bins] double. */
XPCS_API int xpcs_shell_mean(const void* values, int64_t rows, int64_t n_q, const int32_t* bin_of_q, int32_t n_bins,
                    double scale, double* out, const xpcs_opts* opts);

/* Eq.(12)-(13): ring-averaged S(q,t) = <I(q,t)>_ring / sum_j f_j^2, with sum_j f_j^2 reduced
 * on the device from form_factors [N] (in_dtype, NULL => f = 1).  I [rows][n_q] in_dtype -> out [rows][n_bins]. */
XPCS_API int xpcs_structure_factor_shells(const void* I, int64_t rows, int64_t n_q, const void* form_factors, int64_t N,
                                 const int32_t* bin_of_q, int32_t n_bins, double* out, const xpcs_opts* opts);

/* ------------------------------------------------------------------------------------------------
 * One pass of the whole hot path from HOST memory (the end-to-end entry point):
 * I(q,t) on a lattice plane or an explicit q list (Eq. 7-8, Algorithm 1) for every frame, g2 (Eq. 14), the ring
 * averages S(q,t) (Eq. 12-13) and of g2, and the XSVS contrast (Eq. 15+17).
 * The frames are split into `batches`: batch b's positions are copied host -> device on an internal copy stream,
 * its intensities are computed on opts->stream and copied back on a second internal copy stream while batch b+1
 * is computed; the reductions follow on opts->stream and their results are copied back.  The internal streams fork
 * from and join into opts->stream, so all outputs are valid in host memory once opts->stream is synchronised.
 * Host buffers should be page-locked (cudaHostAlloc / cudaHostRegister) for the copies to overlap the kernels;
 * pageable memory is correct but serialises the copies (and cannot be captured in a CUDA graph).  Device buffers
 * are library-owned, cached per (device, opts->stream) and freed by xpcs_release.  After one call outside a
 * capture, the call can be captured in a CUDA graph on the same stream (pinned host buffers).
 *   positions    HOST [frames][N][3] in_dtype
 *   form_factors HOST [N] in_dtype or NULL (f = 1); with species: used only for the S(q) normalisation sum f^2.
 *                Without species, under XPCS_ENGINE_AUTO with f32 inputs, per-atom values with at most 16 distinct
 *                values are run as atom kinds with q-independent f_s (so the light kinds can use the integer
 *                engine; the result is the same Eq.(7) sum)
 *   species      NULL or atom kinds as for xpcs_intensity_volume (species->species HOST, f_q DEVICE
 *                [n_species][n_q]); then form_factors may still be given for the normalisation
 *   bin_of_q     DEVICE [n_q] ring index (-1 excluded), n_bins rings (register it with xpcs_rings_register to
 *                avoid rebuilding the ring plan in every call)
 *   lags HOST [n_lags] (n_lags may be 0);  windows HOST [n_windows] (n_windows may be 0)
 *   I_out HOST [frames][n_q] out_dtype, g2_out HOST [n_lags][n_q] out_dtype, S_rings HOST [frames][n_bins],
 *   g2_rings HOST [n_lags][n_bins], beta HOST [n_windows][n_bins] (double); any output may be NULL (not copied;
 *   g2_rings needs g2 to be computed, which happens whenever n_lags > 0).
 * Errors: EINVAL for a null step/positions/bin_of_q, N/frames/n_bins/batches <= 0, a lag or window out of range,
 *         n_bins > 12288, n_q >= 2^31, invalid species; EUNSUPPORTED for a lag > 640 -- all checked before any work is
 *         enqueued; then the errors of the underlying calls (xpcs_intensity_volume, xpcs_g2, xsvs_contrast, ...), after
 *         which the internal streams are still joined into opts->stream. */
typedef struct {
    const void* positions;
    const void* form_factors;
    const xpcs_species* species;
    int64_t N, frames;
    xpcs_qgrid grid;           /* lattice plane (used when q_vectors == NULL) */
    const void* q_vectors;     /* DEVICE [n_q][3] in_dtype explicit q (e.g. an Ewald detector), or NULL */
    int64_t n_q;               /* with q_vectors */
    double box_L;              /* with q_vectors: box edge (positions are wrapped into [0, L)^3) */
    const int32_t* bin_of_q;
    int32_t n_bins;
    int32_t batches;
    const int32_t* lags;
    int64_t n_lags;
    const int32_t* windows;
    int64_t n_windows;
    void* I_out;
    void* g2_out;
    double* S_rings;
    double* g2_rings;
    double* beta;
} xpcs_step;
XPCS_API int xpcs_step_host(const xpcs_step* step, const xpcs_opts* opts);

/* ------------------------------------------------------------------------------------------------
 * q geometry helpers.
 * xpcs_qgrid_lattice_plane (HOST only, no device work): the configs' plane h, k in [-n/2, n/2 - 1] at height l,
 *   q = (2 pi / L)(h, k, l).  Errors: EINVAL for L <= 0, n <= 0, null out.
 * xpcs_qgrid_ewald: detector pixels on the Ewald sphere (Eq.(1); Fig. 5, PAPER.md:445;
 *   DESIGN.md R4): k = 2 pi / wavelength, k_i = k z, pixel (i, j) at lon-lat angles
 *   psi_x = (i - (npx-1)/2) pitch, psi_y = (j - (npy-1)/2) pitch, u = (sin psi_x cos psi_y, sin psi_y,
 *   cos psi_x cos psi_y), q = k (u - z); computed in FP64, stored as opts->out_dtype into q_out DEVICE
 *   [npx * npy][3] (index i * npy + j).  Errors: EINVAL for wavelength <= 0, npx/npy <= 0, null q_out.
 * xpcs_lattice_bins: ring index of every grid pixel in exact integer arithmetic (R8):
 *   r2 = |m0 + h ma + k mb|^2, b = isqrt(r2) / w; excluded (-1) if r2 == 0 or r2 >= (n_bins w)^2.
 *   bin_out DEVICE [n_h * n_k] int32.  Errors: EINVAL for null pointers, n_bins <= 0, w <= 0.
 * xpcs_radial_bins: ring index of explicit q vectors (in_dtype): b = floor(|q| / q_max * n_bins) in FP64,
 *   -1 for q = 0 or |q| >= q_max.  bin_out DEVICE [n_q]. */
XPCS_API int xpcs_qgrid_lattice_plane(double L, int64_t n, int32_t l, xpcs_qgrid* out);
XPCS_API int xpcs_qgrid_ewald(double wavelength, int64_t npx, int64_t npy, double pitch, void* q_out,
                     const xpcs_opts* opts);
XPCS_API int xpcs_lattice_bins(const xpcs_qgrid* grid, int32_t n_bins, int32_t w, int32_t* bin_out,
                      const xpcs_opts* opts);
XPCS_API int xpcs_radial_bins(const void* q_vectors, int64_t n_q, double q_max, int32_t n_bins, int32_t* bin_out,
                     const xpcs_opts* opts);

/* ------------------------------------------------------------------------------------------------
 * Runtime.
 * xpcs_last_error: message of the calling thread's most recent failure ("" if none); valid until the next call.
 * xpcs_release: synchronise the device and free all cached scratch.
 * xpcs_launch_count: number of CUDA kernels this library has launched since load (monotone).
 * xpcs_profile_reset / xpcs_profile_query: when opts->profile != 0 the library brackets each launch of its
 *   main kernels with CUDA events on opts->stream.  query(i) synchronises and returns, for kernel class i
 *   (0 = intensity main kernel, 1 = staging, 2 = amplitude reduction, 3 = g2, 4 = XSVS, 5 = rings,
 *   6 = the tensor engines' bright-pixel recompute, 7 / 8 = the integer / split-FP16 tensor engine's launches,
 *   which are also counted in class 0),
 *   its name, the summed device time in ms and the number of timed launches; returns EINVAL past the end.
 * xpcs_device_info: SM count and SM clock (kHz) of the current device (HOST outputs). */
XPCS_API const char* xpcs_last_error(void);
XPCS_API int xpcs_release(void);
XPCS_API int64_t xpcs_launch_count(void);
XPCS_API int xpcs_profile_reset(void);
XPCS_API int xpcs_profile_query(int32_t kernel_class, const char** name, double* total_ms, int64_t* launches);
XPCS_API int xpcs_device_info(int32_t* sm_count, int32_t* sm_clock_khz);
/* 1 if xpcs_intensity_grid can run the given xpcs_engine on the current device (AUTO resolves to TENSOR when
 * this returns 1 for TENSOR), else 0.  Set XPCS_DISABLE_TC=1 in the environment to force the SIMT engine. */
XPCS_API int xpcs_engine_available(int32_t engine);
XPCS_API int xpcs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* XPCS_H_ */
