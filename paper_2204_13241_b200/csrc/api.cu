// api.cu -- the C ABI of libxpcs.so (include/xpcs.h): validation, frame batching, scratch, orchestration.
// Every computational step is a kernel of this library; this file only validates, sizes and enqueues.
#include "common.cuh"
#include "../../include/xpcs.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace xpcs {
void clear_error();
const char* last_error();
long long launches();
int profile_reset();
int profile_query(int cls, const char** name, double* ms, long long* n);
}  // namespace xpcs

using namespace xpcs;

namespace {

constexpr size_t kBatchBytes = size_t(1) << 30;   // cap for staged atoms / partial amplitudes per frame batch

struct Opts {
    bool in_f64 = false, out_f64 = false, profile = false;
    int engine = XPCS_ENGINE_AUTO;
    cudaStream_t s = nullptr;
};

int parse_opts(const xpcs_opts* o, Opts& out) {
    if (o) {
        if ((o->in_dtype != XPCS_F32 && o->in_dtype != XPCS_F64) || (o->out_dtype != XPCS_F32 && o->out_dtype != XPCS_F64)) {
            set_error("xpcs: unknown dtype (in_dtype=%d, out_dtype=%d)", o->in_dtype, o->out_dtype);
            return XPCS_EINVAL;
        }
        if (o->engine < XPCS_ENGINE_AUTO || o->engine > XPCS_ENGINE_TENSOR) {
            set_error("xpcs: unknown engine %d", o->engine);
            return XPCS_EINVAL;
        }
        out.in_f64 = o->in_dtype == XPCS_F64;
        out.out_f64 = o->out_dtype == XPCS_F64;
        out.s = (cudaStream_t)o->stream;
        out.engine = o->engine;
        out.profile = o->profile != 0;
    }
    return XPCS_OK;
}

int check_sticky() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("xpcs: CUDA error from earlier work: %s", cudaGetErrorString(e));
        return XPCS_ECUDA;
    }
    return XPCS_OK;
}

int cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return XPCS_OK;
    set_error("xpcs: %s failed: %s", what, cudaGetErrorString(e));
    return XPCS_ECUDA;
}

#define TRY(x)                        \
    do {                              \
        const int rc_ = (x);          \
        if (rc_ != XPCS_OK) return rc_; \
    } while (0)

#define NEED(ptr, name)                                                \
    do {                                                               \
        if ((ptr) == nullptr) {                                        \
            set_error("xpcs: %s must not be NULL", name);              \
            return XPCS_EINVAL;                                        \
        }                                                              \
    } while (0)

#define POS(v, name)                                                   \
    do {                                                               \
        if ((v) <= 0) {                                                \
            set_error("xpcs: %s must be > 0 (got %lld)", name, (long long)(v)); \
            return XPCS_EINVAL;                                        \
        }                                                              \
    } while (0)

LatticeGeom to_geom(const xpcs_qgrid& g) {
    LatticeGeom G;
    G.L = g.L;
    for (int c = 0; c < 3; ++c) { G.m0[c] = g.m0[c]; G.ma[c] = g.ma[c]; G.mb[c] = g.mb[c]; }
    G.h0 = g.h0; G.n_h = g.n_h; G.k0 = g.k0; G.n_k = g.n_k;
    return G;
}

int validate_grid(const xpcs_qgrid* grid) {
    NEED(grid, "grid");
    if (!(grid->L > 0.0) || !std::isfinite(grid->L)) {
        set_error("xpcs: grid->L must be finite and > 0");
        return XPCS_EINVAL;
    }
    POS(grid->n_h, "grid->n_h");
    POS(grid->n_k, "grid->n_k");
    const int64_t lim = int64_t(1) << 30;
    if (std::llabs(grid->h0) > lim || std::llabs(grid->k0) > lim || grid->n_h > lim || grid->n_k > lim ||
        grid->n_h * grid->n_k > (int64_t(1) << 31)) {
        set_error("xpcs: grid indices out of range");
        return XPCS_EINVAL;
    }
    return XPCS_OK;
}

size_t out_size(bool f64) { return f64 ? 8 : 4; }

struct PlanBufs {
    BinPlan plan;
    int64_t max_warps;
};

int make_plan(const int32_t* bins, int64_t n_q, int32_t n_bins, cudaStream_t s, PlanBufs& pb) {
    if (n_bins > 12288) {
        set_error("xpcs: n_bins must be <= 12288 (got %d)", n_bins);
        return XPCS_EINVAL;
    }
    const size_t perm_b = ((sizeof(int32_t) * (size_t)n_q + 255) / 256) * 256;
    const size_t off_b = ((sizeof(int32_t) * (size_t)(n_bins + 1) + 255) / 256) * 256;
    const size_t cnt_b = sizeof(int32_t) * (size_t)((n_q + 1023) / 1024) * (size_t)n_bins;
    char* base = (char*)scratch(s, SS_PLAN, perm_b + 2 * off_b + cnt_b + 256);
    if (!base) return XPCS_ENOMEM;
    pb.plan.perm = (int32_t*)base;
    pb.plan.offsets = (int32_t*)(base + perm_b);
    pb.plan.warp_off = (int32_t*)(base + perm_b + off_b);
    pb.plan.bcounts = (int32_t*)(base + perm_b + 2 * off_b);
    pb.max_warps = (n_q + 31) / 32 + n_bins;
    return cuda_fail(launch_binplan(bins, n_q, n_bins, pb.plan, s), "ring plan");
}

}  // namespace

extern "C" {

int xpcs_version(void) { return 100; }

const char* xpcs_last_error(void) { return last_error(); }

int64_t xpcs_launch_count(void) { return (int64_t)launches(); }

int xpcs_release(void) {
    clear_error();
    release_scratch();
    return check_sticky();
}

int xpcs_profile_reset(void) { return profile_reset(); }

int xpcs_profile_query(int32_t kernel_class, const char** name, double* total_ms, int64_t* n) {
    long long nn = 0;
    const int rc = profile_query(kernel_class, name, total_ms, &nn);
    if (n) *n = nn;
    return rc;
}

int xpcs_device_info(int32_t* sm, int32_t* clk) {
    clear_error();
    int dev = 0;
    TRY(cuda_fail(cudaGetDevice(&dev), "cudaGetDevice"));
    int a = 0, b = 0;
    TRY(cuda_fail(cudaDeviceGetAttribute(&a, cudaDevAttrMultiProcessorCount, dev), "attribute"));
    cudaDeviceGetAttribute(&b, cudaDevAttrClockRate, dev);
    if (sm) *sm = a;
    if (clk) *clk = b;
    return XPCS_OK;
}

int xpcs_engine_available(int32_t engine) {
    if (engine == XPCS_ENGINE_SIMT) return 1;
    LatticeGeom g{};
    if (engine == XPCS_ENGINE_TENSOR || engine == XPCS_ENGINE_AUTO) return lattice_tc_supported(g) ? 1 : (engine == XPCS_ENGINE_AUTO);
    return 0;
}

}  // extern "C"

// ------------------------------------------------------------------------------------------- intensity
// amp = 0: I(q,t) = |p|^2 (Eq. 8) -> out [frames][n_q];  amp = 1: p(q,t) (Eq. 7) -> out [frames][n_q][2]
static int run_direct(const void* positions, int64_t N, const void* form_factors, const void* q_vectors, int64_t n_q,
                      int64_t frames, double box_L, void* I_out, const xpcs_opts* opts, int amp) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(positions, "positions");
    NEED(q_vectors, "q_vectors");
    NEED(I_out, "I_out");
    POS(N, "N");
    POS(n_q, "n_q");
    POS(frames, "frames");
    if (!(box_L > 0.0) || !std::isfinite(box_L)) {
        set_error("xpcs: box_L must be finite and > 0");
        return XPCS_EINVAL;
    }
    if (N > (int64_t(1) << 40) || n_q > (int64_t(1) << 40)) {
        set_error("xpcs: N or n_q too large");
        return XPCS_EINVAL;
    }
    TRY(check_sticky());
    const size_t isz = out_size(o.out_f64) * (amp ? 2 : 1);
    const size_t psz = o.in_f64 ? 24 : 12;
    if (o.in_f64) {
        const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(frames, (int64_t)(kBatchBytes / std::max<int64_t>(1, std::max<int64_t>(32 * N, 16 * n_q)))));
        ulonglong4* st = (ulonglong4*)scratch(o.s, SS_STAGE, sizeof(ulonglong4) * (size_t)(N * Tb));
        double2* part = (double2*)scratch(o.s, SS_PARTIAL, sizeof(double2) * (size_t)(n_q * Tb));
        if (!st || !part) return XPCS_ENOMEM;
        for (int64_t t0 = 0; t0 < frames; t0 += Tb) {
            const int64_t tb = std::min(Tb, frames - t0);
            { ProfScope p(o.profile, KC_STAGE, o.s);
              TRY(cuda_fail(launch_stage_generic64((const char*)positions + psz * N * t0, form_factors, N, tb, box_L, st, o.s), "stage")); }
            { ProfScope p(o.profile, KC_MAIN, o.s);
              TRY(cuda_fail(launch_generic64(st, N, tb, q_vectors, n_q, box_L, part, o.s), "generic64")); }
            { ProfScope p(o.profile, KC_REDUCE, o.s);
              TRY(cuda_fail(launch_amp_reduce_d(part, 1, tb, n_q, (char*)I_out + isz * n_q * t0, o.out_f64, amp, o.s), "reduce")); }
        }
        return XPCS_OK;
    }
    // fp32: split atoms only when (q tiles x frames) cannot fill the device
    const int64_t qtiles = (n_q + 1023) / 1024;
    int64_t C = 1;
    const int64_t want = 2LL * sm_count();
    if (qtiles * frames < want) C = std::min<int64_t>((want + qtiles * frames - 1) / (qtiles * frames), (N + 511) / 512);
    int64_t chunk = (N + C - 1) / C;
    chunk = ((chunk + 511) / 512) * 512;
    C = (N + chunk - 1) / chunk;
    const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(frames, (int64_t)(kBatchBytes / std::max<int64_t>(32 * N, 16 * C * n_q))));
    uint4* st = (uint4*)scratch(o.s, SS_STAGE, 2 * sizeof(uint4) * (size_t)(N * Tb));   // 32 B / atom
    double2* part = (double2*)scratch(o.s, SS_PARTIAL, sizeof(double2) * (size_t)(C * n_q * Tb));
    if (!st || !part) return XPCS_ENOMEM;
    for (int64_t t0 = 0; t0 < frames; t0 += Tb) {
        const int64_t tb = std::min(Tb, frames - t0);
        { ProfScope p(o.profile, KC_STAGE, o.s);
          TRY(cuda_fail(launch_stage_generic32((const char*)positions + psz * N * t0, 0, form_factors, 0, N, tb, box_L, st, o.s), "stage")); }
        { ProfScope p(o.profile, KC_MAIN, o.s);
          TRY(cuda_fail(launch_generic32(st, N, tb, q_vectors, 0, n_q, box_L, chunk, C, part, o.s), "generic32")); }
        { ProfScope p(o.profile, KC_REDUCE, o.s);
          TRY(cuda_fail(launch_amp_reduce_d(part, C, tb, n_q, (char*)I_out + isz * n_q * t0, o.out_f64, amp, o.s), "reduce")); }
    }
    return XPCS_OK;
}

static int run_grid(const void* positions, int64_t N, const void* form_factors, const xpcs_qgrid* grid,
                    int64_t frames, void* I_out, const xpcs_opts* opts, int amp) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(positions, "positions");
    NEED(I_out, "I_out");
    POS(N, "N");
    POS(frames, "frames");
    TRY(validate_grid(grid));
    TRY(check_sticky());
    const LatticeGeom g = to_geom(*grid);
    const int64_t n_q = g.n_h * g.n_k;
    const size_t isz = out_size(o.out_f64) * (amp ? 2 : 1);
    if (o.in_f64) {
        if (o.engine == XPCS_ENGINE_TENSOR) {
            set_error("xpcs: the tensor engine needs f32 inputs");
            return XPCS_EUNSUPPORTED;
        }
        const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(frames, (int64_t)(kBatchBytes / (32 * N))));
        ulonglong4* st = (ulonglong4*)scratch(o.s, SS_STAGE, sizeof(ulonglong4) * (size_t)(N * Tb));
        if (!st) return XPCS_ENOMEM;
        for (int64_t t0 = 0; t0 < frames; t0 += Tb) {
            const int64_t tb = std::min(Tb, frames - t0);
            { ProfScope p(o.profile, KC_STAGE, o.s);
              TRY(cuda_fail(launch_stage_lattice64((const char*)positions + 24 * N * t0, form_factors, N, tb, g, st, o.s), "stage")); }
            { ProfScope p(o.profile, KC_MAIN, o.s);
              TRY(cuda_fail(launch_lattice_f64(st, N, tb, g, (char*)I_out + isz * n_q * t0, o.out_f64, amp, o.s), "lattice64")); }
        }
        return XPCS_OK;
    }
    bool tc = false;
    if (o.engine == XPCS_ENGINE_TENSOR || o.engine == XPCS_ENGINE_AUTO) {
        tc = lattice_tc_supported(g);
        if (!tc && o.engine == XPCS_ENGINE_TENSOR) {
            set_error("xpcs: the tensor engine is not available for this grid/build");
            return XPCS_EUNSUPPORTED;
        }
    }
    // atom chunks (split-K over CTAs, folded in FP64 by the reduction): SIMT keeps fp32 register sums short
    // (<= 4096 atoms); the tensor engine drains TMEM every 256 atoms into RN sums, so its chunks only balance
    // the grid (>= ~8 waves of one CTA per SM) and stay >= 1024 atoms.
    int64_t chunk = 4096;
    if (tc) {
        const int64_t tiles = ((g.n_h + 127) / 128) * ((g.n_k + 127) / 128);
        const int64_t units = tiles * std::min<int64_t>(frames, 64);
        int64_t C0 = std::max<int64_t>(1, (8LL * sm_count() + units - 1) / units);
        C0 = std::min<int64_t>(C0, std::max<int64_t>(1, N / 1024));
        chunk = ((N + C0 - 1) / C0 + 15) / 16 * 16;
    }
    if (const char* e = getenv("XPCS_CHUNK_ATOMS")) chunk = std::max<int64_t>(16, atoll(e));   // experiments only
    const int64_t C = (N + chunk - 1) / chunk;
    const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(frames, (int64_t)(kBatchBytes / std::max<int64_t>(16 * N, 8 * C * n_q))));
    uint4* st = (uint4*)scratch(o.s, SS_STAGE, sizeof(uint4) * (size_t)(N * Tb));
    float2* part = (float2*)scratch(o.s, SS_PARTIAL, sizeof(float2) * (size_t)(C * n_q * Tb));
    if (!st || !part) return XPCS_ENOMEM;
    for (int64_t t0 = 0; t0 < frames; t0 += Tb) {
        const int64_t tb = std::min(Tb, frames - t0);
        { ProfScope p(o.profile, KC_STAGE, o.s);
          TRY(cuda_fail(launch_stage_lattice32((const char*)positions + 12 * N * t0, 0, form_factors, 0, N, tb, g, st, o.s), "stage")); }
        { ProfScope p(o.profile, KC_MAIN, o.s);
          if (tc) TRY(cuda_fail(launch_lattice_tc(st, N, tb, g, chunk, C, part, o.s), "lattice tcgen05"));
          else TRY(cuda_fail(launch_lattice_simt(st, N, tb, g, chunk, C, part, o.s), "lattice simt")); }
        { ProfScope p(o.profile, KC_REDUCE, o.s);
          // the tensor engine's partials hold conj(p) (R1)
          TRY(cuda_fail(launch_amp_reduce_f(part, C, tb, n_q, (char*)I_out + isz * n_q * t0, o.out_f64,
                                            amp ? (tc ? 2 : 1) : 0, o.s), "reduce")); }
    }
    return XPCS_OK;
}

extern "C" {

int xpcs_intensity(const void* positions, int64_t N, const void* form_factors, const void* q_vectors, int64_t n_q,
                   int64_t frames, double box_L, void* I_out, const xpcs_opts* opts) {
    return run_direct(positions, N, form_factors, q_vectors, n_q, frames, box_L, I_out, opts, 0);
}
int xpcs_amplitude(const void* positions, int64_t N, const void* form_factors, const void* q_vectors, int64_t n_q,
                   int64_t frames, double box_L, void* A_out, const xpcs_opts* opts) {
    return run_direct(positions, N, form_factors, q_vectors, n_q, frames, box_L, A_out, opts, 1);
}
int xpcs_intensity_grid(const void* positions, int64_t N, const void* form_factors, const xpcs_qgrid* grid,
                        int64_t frames, void* I_out, const xpcs_opts* opts) {
    return run_grid(positions, N, form_factors, grid, frames, I_out, opts, 0);
}
int xpcs_amplitude_grid(const void* positions, int64_t N, const void* form_factors, const xpcs_qgrid* grid,
                        int64_t frames, void* A_out, const xpcs_opts* opts) {
    return run_grid(positions, N, form_factors, grid, frames, A_out, opts, 1);
}

int xpcs_isf(const void* A_series, int64_t frames, int64_t n_q, const int32_t* lags, int64_t n_lags,
             const void* form_factors, int64_t N, double* F_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(A_series, "A_series");
    NEED(lags, "lags");
    NEED(F_out, "F_out");
    POS(frames, "frames");
    POS(n_q, "n_q");
    POS(n_lags, "n_lags");
    POS(N, "N");
    int max_lag = 0;
    for (int64_t i = 0; i < n_lags; ++i) {
        if (lags[i] < 0 || lags[i] >= frames) {
            set_error("xpcs: lag %d out of range [0, %lld)", lags[i], (long long)frames);
            return XPCS_EINVAL;
        }
        max_lag = std::max(max_lag, (int)lags[i]);
    }
    if (max_lag > 320) {
        set_error("xpcs: lags > 320 frames are not supported by xpcs_isf in this build");
        return XPCS_EUNSUPPORTED;
    }
    TRY(check_sticky());
    int32_t* dl = (int32_t*)scratch(o.s, SS_LAGS, sizeof(int32_t) * (size_t)n_lags);
    if (!dl) return XPCS_ENOMEM;
    TRY(cuda_fail(cudaMemcpyAsync(dl, lags, sizeof(int32_t) * (size_t)n_lags, cudaMemcpyHostToDevice, o.s), "lag upload"));
    double* norm = nullptr;
    if (form_factors) {
        norm = (double*)scratch(o.s, SS_SMALL, 64);
        if (!norm) return XPCS_ENOMEM;
        TRY(cuda_fail(launch_sum_f2(form_factors, o.in_f64, N, norm, o.s), "sum f^2"));
    }
    ProfScope p(o.profile, KC_G2, o.s);
    return cuda_fail(launch_isf(A_series, o.in_f64, frames, n_q, dl, n_lags, max_lag, norm, (double)N, F_out, o.s), "isf");
}

// ------------------------------------------------------------------------------------------- statistics
int xpcs_g2(const void* I_series, int64_t frames, int64_t n_q, const int32_t* lags, int64_t n_lags, void* g2_out,
            const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(I_series, "I_series");
    NEED(lags, "lags");
    NEED(g2_out, "g2_out");
    POS(frames, "frames");
    POS(n_q, "n_q");
    POS(n_lags, "n_lags");
    int max_lag = 0;
    for (int64_t i = 0; i < n_lags; ++i) {
        if (lags[i] < 0 || lags[i] >= frames) {
            set_error("xpcs: lag %d out of range [0, %lld)", lags[i], (long long)frames);
            return XPCS_EINVAL;
        }
        max_lag = std::max(max_lag, (int)lags[i]);
    }
    if (max_lag > 640) {
        set_error("xpcs: lags > 640 frames are not supported by this build");
        return XPCS_EUNSUPPORTED;
    }
    TRY(check_sticky());
    int32_t* dl = (int32_t*)scratch(o.s, SS_LAGS, sizeof(int32_t) * (size_t)n_lags);
    if (!dl) return XPCS_ENOMEM;
    TRY(cuda_fail(cudaMemcpyAsync(dl, lags, sizeof(int32_t) * (size_t)n_lags, cudaMemcpyHostToDevice, o.s), "lag upload"));
    ProfScope p(o.profile, KC_G2, o.s);
    return cuda_fail(launch_g2(I_series, o.in_f64, frames, n_q, dl, n_lags, max_lag, g2_out, o.out_f64, o.s), "g2");
}

int xsvs_contrast(const void* I_series, int64_t frames, int64_t n_q, const int32_t* bin_of_q, int32_t n_bins,
                  const int32_t* windows, int64_t n_windows, double* beta_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(I_series, "I_series");
    NEED(bin_of_q, "bin_of_q");
    NEED(windows, "windows");
    NEED(beta_out, "beta_out");
    POS(frames, "frames");
    POS(n_q, "n_q");
    POS(n_bins, "n_bins");
    POS(n_windows, "n_windows");
    if (n_q > (int64_t(1) << 31) - 1) {
        set_error("xpcs: n_q too large for the ring plan");
        return XPCS_EINVAL;
    }
    int64_t max_slots = 0;
    for (int64_t w0 = 0; w0 < n_windows; w0 += 16) {
        int64_t s = 0;
        for (int64_t i = w0; i < std::min(n_windows, w0 + 16); ++i) {
            if (windows[i] < 1 || windows[i] > frames) {
                set_error("xpcs: window %d out of range [1, %lld]", windows[i], (long long)frames);
                return XPCS_EINVAL;
            }
            s += frames / windows[i];
        }
        max_slots = std::max(max_slots, s);
    }
    TRY(check_sticky());
    ProfScope p(o.profile, KC_XSVS, o.s);
    PlanBufs pb;
    TRY(make_plan(bin_of_q, n_q, n_bins, o.s, pb));
    double* mom = (double*)scratch(o.s, SS_XSVS, sizeof(double2) * (size_t)(pb.max_warps * max_slots));
    if (!mom) return XPCS_ENOMEM;
    return cuda_fail(launch_xsvs(I_series, o.in_f64, frames, n_q, pb.plan, n_bins, windows, n_windows, pb.max_warps,
                                 mom, nullptr, beta_out, o.s), "xsvs");
}

int xpcs_shell_mean(const void* values, int64_t rows, int64_t n_q, const int32_t* bin_of_q, int32_t n_bins,
                    double scale, double* out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(values, "values");
    NEED(bin_of_q, "bin_of_q");
    NEED(out, "out");
    POS(rows, "rows");
    POS(n_q, "n_q");
    POS(n_bins, "n_bins");
    TRY(check_sticky());
    ProfScope p(o.profile, KC_RINGS, o.s);
    PlanBufs pb;
    TRY(make_plan(bin_of_q, n_q, n_bins, o.s, pb));
    return cuda_fail(launch_shell_mean(values, o.in_f64, rows, n_q, pb.plan, n_bins, scale, nullptr, out, o.s), "rings");
}

int xpcs_structure_factor_shells(const void* I, int64_t rows, int64_t n_q, const void* form_factors, int64_t N,
                                 const int32_t* bin_of_q, int32_t n_bins, double* out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(I, "I");
    NEED(bin_of_q, "bin_of_q");
    NEED(out, "out");
    POS(rows, "rows");
    POS(n_q, "n_q");
    POS(n_bins, "n_bins");
    POS(N, "N");
    TRY(check_sticky());
    ProfScope p(o.profile, KC_RINGS, o.s);
    PlanBufs pb;
    TRY(make_plan(bin_of_q, n_q, n_bins, o.s, pb));
    double* norm = nullptr;
    double scale = 1.0;
    if (form_factors) {
        norm = (double*)scratch(o.s, SS_SMALL, 64);
        if (!norm) return XPCS_ENOMEM;
        TRY(cuda_fail(launch_sum_f2(form_factors, o.in_f64, N, norm, o.s), "sum f^2"));
    } else {
        scale = 1.0 / (double)N;     // sum_j f_j^2 = N for unit form factors
    }
    return cuda_fail(launch_shell_mean(I, o.in_f64, rows, n_q, pb.plan, n_bins, scale, norm, out, o.s), "rings");
}

// ------------------------------------------------------------------------------------------- geometry
int xpcs_qgrid_lattice_plane(double L, int64_t n, int32_t l, xpcs_qgrid* out) {
    clear_error();
    NEED(out, "out");
    POS(n, "n");
    if (!(L > 0.0) || !std::isfinite(L)) {
        set_error("xpcs: L must be finite and > 0");
        return XPCS_EINVAL;
    }
    std::memset(out, 0, sizeof(*out));
    out->L = L;
    out->m0[2] = l;
    out->ma[0] = 1;
    out->mb[1] = 1;
    out->h0 = -(n / 2);
    out->k0 = -(n / 2);
    out->n_h = n;
    out->n_k = n;
    return XPCS_OK;
}

int xpcs_qgrid_ewald(double wavelength, int64_t npx, int64_t npy, double pitch, void* q_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(q_out, "q_out");
    POS(npx, "npx");
    POS(npy, "npy");
    if (!(wavelength > 0.0) || !std::isfinite(wavelength) || !std::isfinite(pitch)) {
        set_error("xpcs: wavelength must be finite and > 0, pitch finite");
        return XPCS_EINVAL;
    }
    TRY(check_sticky());
    return cuda_fail(launch_ewald(wavelength, npx, npy, pitch, q_out, o.out_f64, o.s), "ewald");
}

int xpcs_lattice_bins(const xpcs_qgrid* grid, int32_t n_bins, int32_t w, int32_t* bin_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    TRY(validate_grid(grid));
    NEED(bin_out, "bin_out");
    POS(n_bins, "n_bins");
    POS(w, "w");
    TRY(check_sticky());
    return cuda_fail(launch_lattice_bins(to_geom(*grid), n_bins, w, bin_out, o.s), "lattice bins");
}

int xpcs_radial_bins(const void* q_vectors, int64_t n_q, double q_max, int32_t n_bins, int32_t* bin_out,
                     const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(q_vectors, "q_vectors");
    NEED(bin_out, "bin_out");
    POS(n_q, "n_q");
    POS(n_bins, "n_bins");
    if (!(q_max > 0.0) || !std::isfinite(q_max)) {
        set_error("xpcs: q_max must be finite and > 0");
        return XPCS_EINVAL;
    }
    TRY(check_sticky());
    return cuda_fail(launch_radial_bins(q_vectors, o.in_f64, n_q, q_max, n_bins, bin_out, o.s), "radial bins");
}

}  // extern "C"
