// common.cuh -- internal helpers of libxpcs.so (sm_100a).  Not part of the ABI (see include/xpcs.h).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>

namespace xpcs {

// ------------------------------------------------------------------------------------------------
// host-side runtime services (defined in runtime.cu)
// ------------------------------------------------------------------------------------------------
enum KernelClass { KC_MAIN = 0, KC_STAGE = 1, KC_REDUCE = 2, KC_G2 = 3, KC_XSVS = 4, KC_RINGS = 5, KC_FIXUP = 6, KC_I8 = 7, KC_TC = 8,
                   KC_COUNT = 9 };   // KC_I8 / KC_TC: the tensor engines' launches inside KC_MAIN

void set_error(const char* fmt, ...);
void note_launch(int n = 1);

// Scratch cached per (stream, slot); grown on demand (the grow synchronises the device).
enum ScratchSlot {
    SS_STAGE = 0, SS_PARTIAL, SS_PLAN, SS_PLAN2, SS_XSVS, SS_SMALL, SS_LAGS, SS_TC, SS_IDX, SS_FFT,
    SS_H_POS, SS_H_FF, SS_H_I, SS_H_G2, SS_H_RED, SS_FIX, SS_H_FQ, SS_STAGE2, SS_PARTIAL2, SS_FIX2, SS_COUNT
};
void* scratch(cudaStream_t s, int slot, size_t bytes);   // nullptr on failure (error already set)
// workspace id of the calling thread's current API call (xpcs_opts.workspace): scratch is keyed by (device, workspace,
// stream, slot); set by parse_opts at the start of every call
void set_workspace(int ws);
void release_scratch();

// Profiling: events around launches of one kernel class on a stream (opts->profile).
struct ProfScope {
    ProfScope(bool on, int cls, cudaStream_t s);
    ~ProfScope();
    bool on_;
    int cls_;
    cudaStream_t s_;
    cudaEvent_t a_, b_;
};

int sm_count();
int generic_q_per_block();    // k_generic32 tile: q per CTA
int generic_blocks_per_sm();  // k_generic32: CTAs per SM its registers are sized for
// cached device copy of a host table (by content); pinned if handed out during a capture on s
const void* host_table(const void* data, size_t bytes, cudaStream_t s);
const int32_t* lag_table(const int32_t* lags, int64_t n, cudaStream_t s);   // host_table of a lag list

// ------------------------------------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------------------------------------
// Fixed-point turns: a phase of T * 2^-32 turns (T mod 2^32) -> angle in radians in [-pi, pi).
// Bit trick: (T >> 9) ^ 0x3FC00000 is the float 1.5 + t with t = (int32)T * 2^-32 truncated to 2^-23
// (the truncation is a constant -2^-24-turn mean offset = a global phase, invisible in |p|^2, plus
// a zero-mean error < 2^-23 turns).  Then theta = 2 pi (f - 1.5) in one FFMA.
__device__ __forceinline__ float turns_to_radians(uint32_t T) {
    const float f = __uint_as_float((T >> 9) ^ 0x3FC00000u);
    return fmaf(f, 6.28318530717958647692f, -1.5f * 6.28318530717958647692f);
}

// Accurate conversion for table generation (no truncation): signed turns in [-0.5, 0.5).
__device__ __forceinline__ float turns_signed(uint32_t T) {
    return (float)(int32_t)T * 2.3283064365386963e-10f;   // 2^-32
}

__device__ __forceinline__ double turns_signed64(uint64_t T) {
    return (double)(int64_t)T * 5.421010862427522170037e-20;   // 2^-64
}

// packed FP32x2 FMA (SASS FFMA2): d = a * b + c, element-wise on (lo, hi)
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo2(unsigned long long v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi2(unsigned long long v) { return __uint_as_float((uint32_t)(v >> 32)); }

// Position -> fraction of the box in [0, 1) (periodic wrap) -> 32/64-bit fixed point.
__device__ __forceinline__ double box_fraction(double x, double L) {
    // periodic wrap as the ABI documents it: y = x - L floor(x / L) (a result equal to L maps to 0),
    // then the box fraction u = y / L in [0, 1)
    double y = x - L * floor(x / L);
    if (y >= L || y < 0.0) y = 0.0;
    const double u = y / L;
    return u < 1.0 ? u : 0.0;
}
// Same wrap with a reciprocal multiply (fp32 staging paths): u = x/L - floor(x/L) from x * (1/L); differs from the
// exact quotient by <= 1 ulp, far below the 2^-32-turn resolution of the fixed-point phases it feeds.
__device__ __forceinline__ double box_fraction_fast(double x, double invL) {
    const double v = x * invL;
    double u = v - floor(v);
    if (!(u >= 0.0) || u >= 1.0) u = 0.0;
    return u;
}
__device__ __forceinline__ uint32_t frac_to_fixed32(double u) {
    // round(u * 2^32) mod 2^32 ; u in [0, 1)
    unsigned long long v = (unsigned long long)llrint(u * 4294967296.0);
    return (uint32_t)v;
}
__device__ __forceinline__ uint64_t frac_to_fixed64(double u) {
    // u has <= 53 significant bits, so u * 2^64 is an exact integer-valued real < 2^64
    const double hi = floor(u * 4294967296.0);
    const double lo = (u * 4294967296.0 - hi) * 4294967296.0;   // exact
    return ((uint64_t)hi << 32) + (uint64_t)llrint(lo);
}

}  // namespace xpcs

// ------------------------------------------------------------------------------------------------
// launchers (one per kernel family; defined in the k_*.cu files).  All return cudaError_t of the launch.
// ------------------------------------------------------------------------------------------------
namespace xpcs {

struct LatticeGeom {
    double L;
    int32_t m0[3], ma[3], mb[3];
    int64_t h0, n_h, k0, n_k;
};

// Which source atoms / frames / lattice planes a staging launch reads (see k_stage.cu).
struct StageMap {
    const int32_t* idx;   // device [N staged atoms]: source atom index (species gather); nullptr = identity
    int64_t n_src;        // atoms per source frame
    int64_t v0;           // first virtual frame of the batch
    int64_t n_l, l0;      // virtual frame v = (frame v / n_l, plane l0 + v % n_l); n_l = 1 for a plane / q list
    int32_t mc[3];        // plane step of a 3-D q block: m0(l) = m0 + l mc
};

// staging: positions [T][n_src][3] (f32|f64) + f [n_src] (f32|f64|null) -> per-atom fixed-point turns [frames][N]
cudaError_t launch_stage_lattice32(const void* pos, int pos_f64, const void* f, int f_f64, int64_t N,
                                   int64_t frames, const LatticeGeom& g, const StageMap& m, uint4* out, cudaStream_t s);
cudaError_t launch_stage_lattice64(const void* pos, const void* f, int64_t N, int64_t frames,
                                   const LatticeGeom& g, const StageMap& m, ulonglong4* out, cudaStream_t s);
cudaError_t launch_stage_generic32(const void* pos, int pos_f64, const void* f, int f_f64, int64_t N,
                                   int64_t frames, double L, const StageMap& m, uint4* out, cudaStream_t s);
cudaError_t launch_stage_generic64(const void* pos, const void* f, int64_t N, int64_t frames, double L,
                                   const StageMap& m, ulonglong4* out, cudaStream_t s);

// species superposition (q-dependent form factors): out = |sum_s f_s(q) sum_c part_s[c]|^2 (mode 0) or the
// amplitude (mode 1; mode 2: the partials hold conj(p)).  part_s [C_s][frames][n_q] (float2 | double2);
// fq [n_species][n_l * n_q] (f32|f64), row of virtual frame v: plane (v0 + v) % n_l.
constexpr int kMaxKinds = 16;      // atom kinds a caller may define (xpcs_species.n_species)
constexpr int kMaxSpecies = 32;    // atom groups of a call (a kind may be split between two engines)
struct SpeciesParts {
    const void* part[kMaxSpecies];
    int64_t C[kMaxSpecies];
    int32_t kind[kMaxSpecies];     // f_q row of each group
    int n;
    int part_f64;
};
struct BrightSink;
// rows of constants: out[r][i] = vals[r] (f32 | f64), n_rows <= kMaxKinds (kind form factors of xpcs_step_host)
cudaError_t launch_fill_rows(void* out, int out_f64, int n_rows, int64_t n, const double* vals, cudaStream_t s);
cudaError_t launch_species_combine(const SpeciesParts& sp, int64_t frames, int64_t n_q, const void* fq, int fq_f64,
                                   int64_t v0, int64_t n_l, void* out, int out_f64, int mode, cudaStream_t s,
                                   const BrightSink* bright = nullptr);
// Algorithm 2 (FFT method): spread + cuFFT D2Z + epilogue for `frames` frames; rho [frames][n^3] double, spec
// [frames][n][n][n/2+1] double2 scratch.  Returns 0, 2 (CUDA error) or 3 (cuFFT error); *what names the step.
int launch_fft_intensity(const void* pos, int pos_f64, int64_t N, int64_t frames, double L, int n, double eta, int k,
                         double* rho, double2* spec, int64_t h0, int64_t n_h, int64_t k0, int64_t n_k, int64_t l0,
                         int64_t n_l, const void* fq, int fq_f64, void* out, int out_f64, cudaStream_t s,
                         const char** what);
cudaError_t fft_release_plan();
// f(q) = c + sum_i a_i exp(-b_i (|q| / 4 pi)^2) for an explicit q list (q != nullptr) or a 3-D lattice block
cudaError_t launch_form_factor_gaussian(const void* q, int q_f64, int64_t n_q, const LatticeGeom& g, int64_t l0,
                                        int64_t n_l, const int32_t* mc, int n_gauss, const double* a, const double* b,
                                        double c, void* out, int out_f64, cudaStream_t s);

// lattice contraction, FP32 CUDA cores: partial [C][Tb][n_h*n_k] float2
cudaError_t launch_lattice_simt(const uint4* staged, int64_t N, int64_t frames, const LatticeGeom& g,
                                int64_t chunk_atoms, int64_t n_chunks, float2* partial, cudaStream_t s);
// lattice contraction, tcgen05 split-FP16: partial [C][Tb][n_h*n_k] float2.  Returns cudaErrorNotSupported
// if the geometry does not fit the engine's tiling constraints.
cudaError_t launch_lattice_tc(const uint4* staged, int64_t N, int64_t frames, const LatticeGeom& g,
                              int64_t chunk_atoms, int64_t n_chunks, float2* partial, cudaStream_t s);
bool lattice_tc_supported(const LatticeGeom& g);
// lattice contraction, tcgen05 kind::i8 with two int8 limbs and exact int32 accumulation (k_lattice_i8.cu):
// partial [C][Tb][n_h*n_k] float2 (conj(p), like the split-FP16 engine); chunk_atoms <= kI8MaxChunk.
// uniform_f != 0: all f_j = 1 (no W scale); else F = max |f_j| is reduced into fmax_scratch (1 float) first.
constexpr int64_t kI8MaxChunk = 65536;   // int32 TMEM accumulators: |X| <= 65536 x 2 x 127 x 128 < 2^31
int i8_cluster_slots();   // k_lattice_i8 clusters resident at once (cudaOccupancyMaxActiveClusters)
int i8_stage_atoms();     // k_lattice_i8 atoms per pipeline stage (chunks are multiples of it)
cudaError_t launch_absmax_f(const uint4* staged, int64_t n, float* out, cudaStream_t s);   // max |f| of staged records
// Bright pixels after the integer engine (k_fixup.cu): the epilogue that writes a batch's final I (or p) appends
// every pixel with I > thr * F(q)^2 (F = *fmax or 1; species: max_s |f_s(q)|) to `list` (index v * n_q + pixel of the
// batch); k_fixup.cu then recomputes them exactly.  All pointers null: no detection.
struct BrightSink {
    uint32_t* count;
    uint32_t* list;
    double thr;             // min(64 N, N^2 / 4)
    const float* fmax;      // max |f_j| of per-atom form factors (device), or nullptr (F = 1)
};
__device__ __forceinline__ void bright_append(const BrightSink& b, double I, double F, int64_t e) {
    if (b.count && !(I <= b.thr * F * F)) {          // NaN / inf are recomputed too
        const uint32_t at = atomicAdd(b.count, 1u);
        b.list[at] = (uint32_t)e;
    }
}
__device__ __forceinline__ double bright_F(const BrightSink& b) { return b.fmax ? (double)fmaxf(*b.fmax, 0.0f) : 1.0; }
struct FixGroups {
    const uint4* st[kMaxSpecies];   // staged records of group s: [vb][n[s]]
    int64_t n[kMaxSpecies];
    int32_t kind[kMaxSpecies];      // f_q row of group s (species calls)
    int n_groups;
    const void* fq;                 // species f_q [n_species][n_l * n_q] or nullptr (f inside the records)
    int fq_f64;
    int64_t v0, n_l;                // first virtual frame of the batch, planes per frame (f_q row = (v0 + v) % n_l)
};
size_t fixup_scratch_bytes(int64_t vb, int64_t n_q, int64_t n_atoms);   // count, list, chunk partials
// carve the sink out of the fixup scratch and zero its count (before the batch's epilogue)
cudaError_t fixup_prepare(void* scratch_buf, int64_t n_atoms, const float* fmax, BrightSink& out, cudaStream_t s);
// exact recompute of the listed pixels (after the epilogue): out = the batch's final I [vb][n_q] or p [vb][n_q][2]
cudaError_t launch_fixup(const FixGroups& G, const LatticeGeom& g, int64_t vb, void* out, int out_f64, int amp,
                         void* scratch_buf, cudaStream_t s);
cudaError_t launch_lattice_i8(const uint4* staged, int64_t N, int64_t frames, const LatticeGeom& g, int64_t chunk_atoms,
                              int64_t n_chunks, float* fmax_scratch, int uniform_f, float2* partial, cudaStream_t s,
                              void* direct_out = nullptr, int out_f64 = 0, int mode = 0,
                              const BrightSink* bright = nullptr);
// lattice FP64 (direct per-pixel evaluation with 64-bit turns): writes I directly (double)
cudaError_t launch_lattice_f64(const ulonglong4* staged, int64_t N, int64_t frames, const LatticeGeom& g,
                               void* I_out, int out_f64, int mode, cudaStream_t s,
                               double2* partial = nullptr, int64_t chunk_atoms = 0, int64_t n_chunks = 1);
// generic q list: partial [C][Tb][n_q] double2
cudaError_t launch_generic32(const uint4* staged, int64_t N, int64_t frames, const void* q, int q_f64,
                             int64_t n_q, double L, int64_t chunk_atoms, int64_t n_chunks, double2* partial,
                             cudaStream_t s);
cudaError_t launch_generic64(const ulonglong4* staged, int64_t N, int64_t frames, const void* q,
                             int64_t n_q, double L, double2* partial, cudaStream_t s);
// fold of the atom-chunk partials: mode 0 -> I = |p|^2, 1 -> p (re, im), 2 -> partials hold conj(p), write p
cudaError_t launch_amp_reduce_f(const float2* partial, int64_t C, int64_t frames, int64_t n_q, void* I_out,
                                int out_f64, int mode, cudaStream_t s, const BrightSink* bright = nullptr);
cudaError_t launch_amp_reduce_d(const double2* partial, int64_t C, int64_t frames, int64_t n_q, void* I_out,
                                int out_f64, int mode, cudaStream_t s);
// intermediate scattering function F(q, tau) = <p(t) p*(t + tau)>_t / norm, complex in/out
cudaError_t launch_isf(const void* A, int in_f64, int64_t T, int64_t n_q, const int32_t* lags_dev, int64_t n_lags,
                       int max_lag, const double* norm, double norm_const, double* F_out, cudaStream_t s);

// statistics
cudaError_t launch_g2(const void* I, int in_f64, int64_t T, int64_t n_q, const int32_t* lags_dev,
                      int64_t n_lags, int max_lag, void* out, int out_f64, cudaStream_t s);
// block-streamed g2 (k_stats.cu): acc [n_lags][n_q] / sum [n_q] FP64 state, ring [R][n_q] of the last frames
cudaError_t launch_g2_accumulate(const void* blk, int in_f64, int64_t B, void* ring, int64_t R, int64_t t0,
                                 int64_t n_q, const int32_t* lags_dev, int64_t n_lags, int max_lag, double* acc,
                                 double* sum, cudaStream_t s);
cudaError_t launch_g2_finalize(const double* acc, const double* sum, int64_t T, int64_t n_q, const int32_t* lags_dev,
                               int64_t n_lags, void* out, int out_f64, cudaStream_t s);
#ifndef XPCS_XSVS_PX
#define XPCS_XSVS_PX 4
#endif
constexpr int XSVS_PX = XPCS_XSVS_PX;   // pixels per lane of the XSVS kernel (when the grid still fills the GPU)
struct BinPlan {
    int32_t* perm;        // [n_valid] pixel indices sorted by (bin, pixel)
    int32_t* offsets;     // [n_bins + 1]
    int32_t* warp_off;    // [n_bins + 1] prefix of ceil(count_b / 32)
    int32_t* sw_off;      // [n_bins + 1] prefix of ceil(count_b / (32 XSVS_PX)): the XSVS kernel's warps (XSVS_PX pixels per lane)
    int32_t* bcounts;     // [ceil(n_q / 1024)][n_bins] scratch of the plan build
};
cudaError_t launch_binplan(const int32_t* bins, int64_t n_q, int32_t n_bins, BinPlan plan, cudaStream_t s);
cudaError_t launch_sum_f2(const void* f, int f_f64, int64_t N, double* out, cudaStream_t s);
cudaError_t launch_shell_mean(const void* v, int in_f64, int64_t rows, int64_t n_q, BinPlan plan,
                              int32_t n_bins, double scale, const double* norm, double* out, cudaStream_t s);
cudaError_t launch_speckle_hist(const void* I, int in_f64, int64_t T, int64_t n_q, BinPlan plan, int32_t n_bins,
                                int32_t M, int64_t max_warps, double* warp_moments, double* means, int32_t n_hist,
                                double kappa_max, int64_t* counts, cudaStream_t s);
cudaError_t launch_xsvs(const void* I, int in_f64, int64_t T, int64_t n_q, BinPlan plan, int32_t n_bins,
                        const int32_t* windows_host, int64_t n_windows, int64_t max_warps, double* warp_moments,
                        double* mom_out, cudaStream_t s);   // per (slot, ring) moments; beta: launch_xsvs_beta_from_moments
cudaError_t launch_xsvs_beta_from_moments(const double* mom, int64_t T, const int32_t* windows_host, int64_t n_windows,
                                          int32_t n_bins, double* beta_out, cudaStream_t s);
cudaError_t launch_shell_moments(const void* v, int in_f64, int64_t rows, int64_t n_q, BinPlan plan, int32_t n_bins,
                                 double* out, cudaStream_t s);
cudaError_t launch_ring_means_from_moments(const double* mom, int64_t n, double scale, const double* norm, double* out,
                                           cudaStream_t s);
// geometry
cudaError_t launch_ewald(double wavelength, int64_t npx, int64_t npy, double pitch, void* q, int out_f64,
                         cudaStream_t s);
cudaError_t launch_lattice_bins(const LatticeGeom& g, int32_t n_bins, int32_t w, int32_t* out, cudaStream_t s);
cudaError_t launch_radial_bins(const void* q, int q_f64, int64_t n_q, double q_max, int32_t n_bins,
                               int32_t* out, cudaStream_t s);

}  // namespace xpcs
