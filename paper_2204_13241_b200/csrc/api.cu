// api.cu -- the C ABI of libxpcs.so (include/xpcs.h): validation, frame batching, scratch, orchestration.
// Every computational step is a kernel of this library; this file only validates, sizes and enqueues.
#include "common.cuh"
#include <map>
#include <mutex>
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

void release_host_resources();   // xpcs_step_host's copy streams and events (defined below)
void release_overlap_resources();   // the frame-batch overlap's side streams and events (defined below)

namespace {

constexpr size_t kBatchBytes = size_t(1) << 30;   // cap for staged atoms / partial amplitudes per frame batch

struct Opts {
    bool in_f64 = false, out_f64 = false, profile = false;
    int engine = XPCS_ENGINE_AUTO;
    int workspace = 0;
    cudaStream_t s = nullptr;
};

int parse_opts(const xpcs_opts* o, Opts& out) {
    if (o) {
        if ((o->in_dtype != XPCS_F32 && o->in_dtype != XPCS_F64) || (o->out_dtype != XPCS_F32 && o->out_dtype != XPCS_F64)) {
            set_error("xpcs: unknown dtype (in_dtype=%d, out_dtype=%d)", o->in_dtype, o->out_dtype);
            return XPCS_EINVAL;
        }
        if (o->engine < XPCS_ENGINE_AUTO || o->engine > XPCS_ENGINE_TENSOR_I8) {
            set_error("xpcs: unknown engine %d", o->engine);
            return XPCS_EINVAL;
        }
        out.in_f64 = o->in_dtype == XPCS_F64;
        out.out_f64 = o->out_dtype == XPCS_F64;
        out.s = (cudaStream_t)o->stream;
        out.engine = o->engine;
        out.profile = o->profile != 0;
        if (o->workspace < 0) {
            set_error("xpcs: workspace must be >= 0 (got %d)", o->workspace);
            return XPCS_EINVAL;
        }
        out.workspace = o->workspace;
    }
    set_workspace(out.workspace);   // scratch() of this call (and of the calls it makes) keys on it
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

// Ring plans registered by xpcs_rings_register: built once, reused by every ring reduction that passes the same
// bin_of_q pointer with the same (n_q, n_bins), until xpcs_rings_unregister / xpcs_release.
struct RegisteredPlan {
    const int32_t* bins;
    int64_t n_q;
    int32_t n_bins;
    int device;
    char* mem;
    PlanBufs pb;
};
std::vector<RegisteredPlan>& registered() {
    static std::vector<RegisteredPlan> v;
    return v;
}

int build_plan(const int32_t* bins, int64_t n_q, int32_t n_bins, cudaStream_t s, char* base, PlanBufs& pb) {
    const size_t perm_b = ((sizeof(int32_t) * (size_t)n_q + 255) / 256) * 256;
    const size_t off_b = ((sizeof(int32_t) * (size_t)(n_bins + 1) + 255) / 256) * 256;
    pb.plan.perm = (int32_t*)base;
    pb.plan.offsets = (int32_t*)(base + perm_b);
    pb.plan.warp_off = (int32_t*)(base + perm_b + off_b);
    pb.plan.sw_off = (int32_t*)(base + perm_b + 2 * off_b);
    pb.plan.bcounts = (int32_t*)(base + perm_b + 3 * off_b);
    pb.max_warps = (n_q + 31) / 32 + n_bins;
    return cuda_fail(launch_binplan(bins, n_q, n_bins, pb.plan, s), "ring plan");
}

size_t plan_bytes(int64_t n_q, int32_t n_bins) {
    const size_t perm_b = ((sizeof(int32_t) * (size_t)n_q + 255) / 256) * 256;
    const size_t off_b = ((sizeof(int32_t) * (size_t)(n_bins + 1) + 255) / 256) * 256;
    const size_t cnt_b = sizeof(int32_t) * (size_t)((n_q + 1023) / 1024) * (size_t)n_bins;
    return perm_b + 3 * off_b + cnt_b + 256;
}

int make_plan(const int32_t* bins, int64_t n_q, int32_t n_bins, cudaStream_t s, PlanBufs& pb) {
    if (n_bins > 12288) {
        set_error("xpcs: n_bins must be <= 12288 (got %d)", n_bins);
        return XPCS_EINVAL;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    for (const auto& r : registered())
        if (r.bins == bins && r.n_q == n_q && r.n_bins == n_bins && r.device == dev) {
            pb = r.pb;
            return XPCS_OK;
        }
    char* base = (char*)scratch(s, SS_PLAN, plan_bytes(n_q, n_bins));
    if (!base) return XPCS_ENOMEM;
    return build_plan(bins, n_q, n_bins, s, base, pb);
}

}  // namespace

extern "C" {

int xpcs_version(void) { return 100; }

const char* xpcs_last_error(void) { return last_error(); }

int64_t xpcs_launch_count(void) { return (int64_t)launches(); }

int xpcs_release(void) {
    clear_error();
    fft_release_plan();
    release_host_resources();
    release_overlap_resources();
    if (!registered().empty()) {
        cudaDeviceSynchronize();
        for (auto& r : registered()) cudaFree(r.mem);
        registered().clear();
    }
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
    if (engine == XPCS_ENGINE_SIMT || engine == XPCS_ENGINE_AUTO) return 1;
    LatticeGeom g{};
    if (engine == XPCS_ENGINE_TENSOR || engine == XPCS_ENGINE_TENSOR_I8) return lattice_tc_supported(g) ? 1 : 0;
    return 0;
}

}  // extern "C"

// ------------------------------------------------------------------------------------------- intensity
// Atom groups of one call: without species one group (all atoms, identity map); with species one group per kind,
// gathered through a device permutation built here (stable partition of the HOST species array).
struct Groups {
    int n_species = 0;                       // 0: no species
    std::vector<int64_t> off, cnt;           // per group: offset into the permutation, atom count
    std::vector<int32_t> kind;               // per group: species row of f_q (a kind may be split into two groups)
    const int32_t* d_idx = nullptr;          // device permutation (species only)
    std::vector<int32_t> perm;               // host permutation (stable partition by kind)
    const void* fq = nullptr;
    int count() const { return (int)cnt.size(); }
    const int32_t* idx(int g) const { return d_idx ? d_idx + off[g] : nullptr; }
};

// host-side validation and permutation (no device work: runs before any launch, EINVAL launches nothing)
static int prep_groups(const xpcs_species* sp, const void* form_factors, int64_t N, Groups& G) {
    if (!sp) {
        G.off.assign(1, 0);
        G.cnt.assign(1, N);
        G.kind.assign(1, 0);
        return XPCS_OK;
    }
    if (form_factors) {
        set_error("xpcs: form_factors and species are exclusive (fold per-atom weights into f_q)");
        return XPCS_EINVAL;
    }
    if (sp->n_species < 1 || sp->n_species > kMaxKinds) {
        set_error("xpcs: n_species must be in [1, %d] (got %d)", kMaxKinds, sp->n_species);
        return XPCS_EINVAL;
    }
    NEED(sp->species, "species->species");
    NEED(sp->f_q, "species->f_q");
    if (N > (int64_t(1) << 31) - 1) {
        set_error("xpcs: species gather supports N < 2^31");
        return XPCS_EINVAL;
    }
    const int S = sp->n_species;
    G.n_species = S;
    G.fq = sp->f_q;
    G.cnt.assign(S, 0);
    for (int64_t j = 0; j < N; ++j) {
        const int32_t k = sp->species[j];
        if (k < 0 || k >= S) {
            set_error("xpcs: species[%lld] = %d outside [0, %d)", (long long)j, k, S);
            return XPCS_EINVAL;
        }
        ++G.cnt[k];
    }
    G.off.assign(S, 0);
    for (int k = 1; k < S; ++k) G.off[k] = G.off[k - 1] + G.cnt[k - 1];
    G.kind.resize(S);
    for (int k = 0; k < S; ++k) G.kind[k] = k;
    G.perm.resize((size_t)N);
    std::vector<int64_t> fill(G.off);
    for (int64_t j = 0; j < N; ++j) G.perm[(size_t)fill[sp->species[j]]++] = (int32_t)j;
    return XPCS_OK;
}

static int upload_groups(Groups& G, cudaStream_t s) {
    if (!G.n_species) return XPCS_OK;
    // cached device copy keyed by content (graph-capturable after one eager call; see host_table)
    const int32_t* d = (const int32_t*)host_table(G.perm.data(), sizeof(int32_t) * G.perm.size(), s);
    if (!d) return XPCS_ECUDA;
    G.d_idx = d;
    return XPCS_OK;
}

static StageMap stage_map(const Groups& G, int g, int64_t N, int64_t v0, int64_t n_l, int64_t l0, const int32_t* mc) {
    StageMap m;
    m.idx = G.idx(g);
    m.n_src = N;
    m.v0 = v0;
    m.n_l = n_l;
    m.l0 = l0;
    for (int c = 0; c < 3; ++c) m.mc[c] = mc ? mc[c] : 0;
    return m;
}

// amp = 0: I(q,t) = |p|^2 (Eq. 8) -> out [frames][n_q];  amp = 1: p(q,t) (Eq. 7) -> out [frames][n_q][2]
static int run_direct(const void* positions, int64_t N, const void* form_factors, const xpcs_species* species,
                      const void* q_vectors, int64_t n_q, int64_t frames, double box_L, void* I_out,
                      const xpcs_opts* opts, int amp) {
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
    Groups G;
    TRY(prep_groups(species, form_factors, N, G));
    TRY(check_sticky());
    TRY(upload_groups(G, o.s));
    const size_t isz = out_size(o.out_f64) * (amp ? 2 : 1);
    const int ng = G.count();
    SpeciesParts sp{};
    sp.n = G.n_species ? ng : 0;
    for (int k = 0; k < ng && k < kMaxSpecies; ++k) sp.kind[k] = G.kind[k];
    sp.part_f64 = 1;
    if (o.in_f64) {
        const int64_t per_frame = std::max<int64_t>(32 * N, 16 * n_q * ng);
        const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(frames, (int64_t)(kBatchBytes / std::max<int64_t>(1, per_frame))));
        ulonglong4* st = (ulonglong4*)scratch(o.s, SS_STAGE, sizeof(ulonglong4) * (size_t)(N * Tb));
        double2* part = (double2*)scratch(o.s, SS_PARTIAL, sizeof(double2) * (size_t)(n_q * Tb * ng));
        if (!st || !part) return XPCS_ENOMEM;
        for (int64_t t0 = 0; t0 < frames; t0 += Tb) {
            const int64_t tb = std::min(Tb, frames - t0);
            int64_t stoff = 0;
            for (int g = 0; g < ng; ++g) {
                const int64_t Ng = G.cnt[g];
                double2* pg = part + (size_t)g * (size_t)(n_q * tb);
                sp.part[g] = pg;
                sp.C[g] = Ng > 0 ? 1 : 0;
                if (Ng == 0) continue;
                const StageMap m = stage_map(G, g, N, t0, 1, 0, nullptr);
                { ProfScope p(o.profile, KC_STAGE, o.s);
                  TRY(cuda_fail(launch_stage_generic64(positions, form_factors, Ng, tb, box_L, m, st + stoff, o.s), "stage")); }
                { ProfScope p(o.profile, KC_MAIN, o.s);
                  TRY(cuda_fail(launch_generic64(st + stoff, Ng, tb, q_vectors, n_q, box_L, pg, o.s), "generic64")); }
                stoff += Ng * tb;
            }
            void* dst = (char*)I_out + isz * n_q * t0;
            ProfScope p(o.profile, KC_REDUCE, o.s);
            if (G.n_species) TRY(cuda_fail(launch_species_combine(sp, tb, n_q, G.fq, 1, t0, 1, dst, o.out_f64, amp, o.s), "species combine"));
            else TRY(cuda_fail(launch_amp_reduce_d(part, 1, tb, n_q, dst, o.out_f64, amp, o.s), "reduce"));
        }
        return XPCS_OK;
    }
    // fp32: split atoms only when (q tiles x frames) cannot fill the device
    const int64_t qtiles = (n_q + generic_q_per_block() - 1) / generic_q_per_block();
    std::vector<int64_t> chunk(ng, 512), C(ng, 0);
    int64_t sumC = 0;
    for (int g = 0; g < ng; ++g) {
        const int64_t Ng = G.cnt[g];
        if (Ng == 0) continue;
        int64_t c = 1;
        const int64_t want = (int64_t)generic_blocks_per_sm() * sm_count();
        if (qtiles * frames < want) c = std::min<int64_t>((want + qtiles * frames - 1) / (qtiles * frames), (Ng + 511) / 512);
        int64_t ch = (Ng + c - 1) / c;
        ch = ((ch + 511) / 512) * 512;
        chunk[g] = ch;
        C[g] = (Ng + ch - 1) / ch;
        sumC += C[g];
    }
    const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(frames, (int64_t)(kBatchBytes / std::max<int64_t>(32 * N, 16 * sumC * n_q))));
    uint4* st = (uint4*)scratch(o.s, SS_STAGE, 2 * sizeof(uint4) * (size_t)(N * Tb));   // 32 B / atom
    double2* part = (double2*)scratch(o.s, SS_PARTIAL, sizeof(double2) * (size_t)(sumC * n_q * Tb));
    if (!st || !part) return XPCS_ENOMEM;
    for (int64_t t0 = 0; t0 < frames; t0 += Tb) {
        const int64_t tb = std::min(Tb, frames - t0);
        int64_t stoff = 0, poff = 0;
        for (int g = 0; g < ng; ++g) {
            const int64_t Ng = G.cnt[g];
            sp.part[g] = part + poff;
            sp.C[g] = C[g];
            if (Ng == 0) continue;
            const StageMap m = stage_map(G, g, N, t0, 1, 0, nullptr);
            { ProfScope p(o.profile, KC_STAGE, o.s);
              TRY(cuda_fail(launch_stage_generic32(positions, 0, form_factors, 0, Ng, tb, box_L, m, st + 2 * stoff, o.s), "stage")); }
            { ProfScope p(o.profile, KC_MAIN, o.s);
              TRY(cuda_fail(launch_generic32(st + 2 * stoff, Ng, tb, q_vectors, 0, n_q, box_L, chunk[g], C[g], part + poff, o.s), "generic32")); }
            stoff += Ng * tb;
            poff += C[g] * n_q * tb;
        }
        void* dst = (char*)I_out + isz * n_q * t0;
        ProfScope p(o.profile, KC_REDUCE, o.s);
        if (G.n_species) TRY(cuda_fail(launch_species_combine(sp, tb, n_q, G.fq, 0, t0, 1, dst, o.out_f64, amp, o.s), "species combine"));
        else TRY(cuda_fail(launch_amp_reduce_d(part, C[0], tb, n_q, dst, o.out_f64, amp, o.s), "reduce"));
    }
    return XPCS_OK;
}

static int validate_volume(const xpcs_qvolume* vol) {
    NEED(vol, "vol");
    TRY(validate_grid(&vol->plane));
    POS(vol->n_l, "vol->n_l");
    const int64_t lim = int64_t(1) << 30;
    if (std::llabs(vol->l0) > lim || vol->n_l > lim) {
        set_error("xpcs: vol->l0 / n_l out of range");
        return XPCS_EINVAL;
    }
    for (int c = 0; c < 3; ++c) {
        for (const int64_t l : {vol->l0, vol->l0 + vol->n_l - 1}) {
            const int64_t m = (int64_t)vol->plane.m0[c] + l * (int64_t)vol->mc[c];
            if (std::llabs(m) > lim) {
                set_error("xpcs: m0 + l mc out of range for 32-bit turns");
                return XPCS_EINVAL;
            }
        }
    }
    return XPCS_OK;
}

constexpr double kI8BudgetDefault = 2.5;   // tools/i8_budget_probe.py (profiles/r02_i8_budget_probe*.log): f in {1, 2}
                                           // all on the integer engine, worst 0.61 / 0.56 of the gate (c3 3e5 / c5 2e5 samples)
static bool fixup_enabled() {
    static int on = -1;
    if (on < 0) { const char* e = getenv("XPCS_FIXUP"); on = (e && atoi(e) == 0) ? 0 : 1; }   // experiments only
    return on == 1;
}

// AUTO's error budget for the integer engine in species calls: kinds in increasing max |f_s| go to it while
// sum_s (f_max_s / f_ref)^2 N_s / N <= budget (1 = the error level of a single f = 1 species on the engine)
static double i8_budget() {
    const char* e = getenv("XPCS_I8_BUDGET");   // experiments only (read per call: the precision probe varies it)
    return e ? atof(e) : kI8BudgetDefault;
}

// ---- integer-engine grid planning (k_lattice_i8: clusters of 2 CTAs, one CTA per SM, 32-atom stages) ----
constexpr double kI8CtaCostDefault = 40.0;   // per-CTA fixed cost in stage units: prologue, the single drain, teardown
static double i8_cta_cost() {
    static double c = -1.0;
    if (c < 0.0) { const char* e = getenv("XPCS_I8_CTA_COST"); c = e ? atof(e) : kI8CtaCostDefault; }   // experiments
    return c;
}
constexpr double kI8BatchCost = 20.0;   // an extra frame batch: its staging, reduction and launch gaps (stage units)
static int64_t i8_tiles(const LatticeGeom& g) { return ((g.n_h + 255) / 256) * ((g.n_k + 127) / 128); }
// atoms per chunk for `units` (tile, virtual frame) pairs of Ng atoms: chunks only balance the grid (exact int32
// accumulation) and stay <= kI8MaxChunk; cost = waves x (stages per CTA + kI8CtaCost), the smallest C wins ties
static int64_t i8_plan_chunk(int64_t Ng, int64_t units, double* cost_out) {
    const int64_t wave = std::max<int64_t>(1, i8_cluster_slots());
    const int64_t ks = i8_stage_atoms();
    const double cta_cost = i8_cta_cost() * 32.0 / (double)ks;   // the fixed cost is calibrated in 32-atom stages
    const int64_t cmin = std::max<int64_t>(1, (Ng + kI8MaxChunk - 1) / kI8MaxChunk);
    const int64_t cmax = std::max<int64_t>(cmin, std::min<int64_t>((Ng + 1023) / 1024, 64));
    int64_t best = cmin;
    double best_cost = 1e300;
    for (int64_t c = cmin; c <= cmax; ++c) {
        const int64_t ch = std::min<int64_t>(((Ng + c - 1) / c + ks - 1) / ks * ks, kI8MaxChunk);
        const int64_t cc = (Ng + ch - 1) / ch;
        const double waves = std::ceil((double)(units * cc) / (double)wave);
        const double cost = waves * ((double)(ch / ks) + cta_cost);
        if (cost < best_cost * (1.0 - 1e-9)) { best_cost = cost; best = c; }
    }
    if (cost_out) *cost_out = best_cost * (double)ks / 32.0;   // in 32-atom stage units (kI8BatchCost)
    return std::min<int64_t>(((Ng + best - 1) / best + ks - 1) / ks * ks, kI8MaxChunk);
}

// split of V virtual frames into [V1 | V - V1] batches with their own chunking (V1 = 0: no split), memoised: the
// search is O(V x chunk counts) host work that would otherwise sit in front of every launch
static void i8_plan_split(int64_t Ng, int64_t tiles, int64_t V, int64_t& V1, int64_t& ch1, int64_t& ch2) {
    struct Key { int64_t Ng, tiles, V; int slots; };
    struct Entry { Key k; int64_t V1, ch1, ch2; };
    static std::mutex mu;
    static std::vector<Entry> memo;
    const int slots = i8_cluster_slots();
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const Entry& e : memo)
            if (e.k.Ng == Ng && e.k.tiles == tiles && e.k.V == V && e.k.slots == slots) { V1 = e.V1; ch1 = e.ch1; ch2 = e.ch2; return; }
    }
    double whole = 0.0;
    ch1 = ch2 = i8_plan_chunk(Ng, tiles * V, &whole);
    V1 = 0;
    double best = whole;
    for (int64_t v1 = 1; v1 < V; ++v1) {
        double c1 = 0.0, c2 = 0.0;
        const int64_t a = i8_plan_chunk(Ng, tiles * v1, &c1), b = i8_plan_chunk(Ng, tiles * (V - v1), &c2);
        const double cost = c1 + c2 + kI8BatchCost;
        if (cost < best * (1.0 - 1e-9)) { best = cost; V1 = v1; ch1 = a; ch2 = b; }
    }
    std::lock_guard<std::mutex> lk(mu);
    if (memo.size() > 256) memo.clear();
    memo.push_back({{Ng, tiles, V, slots}, V1, ch1, ch2});
}

// Frame-batch overlap (lattice engines): batch b runs on the caller's stream (b even) or on a library side stream
// (b odd) with its own staging / partial / bright-list buffers, so batch b + 1's staging and batch b's reduction and
// bright-pixel recompute (HBM-bound, small CTAs) run beside the tensor engine of the neighbouring batch; the engines
// themselves stay in batch order (each waits for the previous batch's engine).  One side stream and a few events
// per (device, caller stream), created on first use outside a graph capture (inside one without them: serial).
namespace {
struct OverlapRes {
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> ev;
};
std::mutex g_ovl_mu;
std::map<std::pair<int, cudaStream_t>, OverlapRes> g_ovl;   // node-based: references stay valid
OverlapRes* overlap_resources(cudaStream_t s, size_t n_events) {
    std::lock_guard<std::mutex> lk(g_ovl_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    auto it = g_ovl.find({dev, s});
    OverlapRes* r = it == g_ovl.end() ? nullptr : &it->second;
    if (r && r->ev.size() >= n_events) return r;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return nullptr;
    }
    if (!r) {
        r = &g_ovl[{dev, s}];
        if (cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            r->side = nullptr;
            return nullptr;
        }
    }
    if (!r->side) return nullptr;
    while (r->ev.size() < n_events) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        r->ev.push_back(e);
    }
    return r;
}
bool batch_overlap_enabled() {
    static int on = -1;
    if (on < 0) { const char* e = getenv("XPCS_BATCH_OVERLAP"); on = (e && atoi(e) == 0) ? 0 : 1; }
    return on == 1;
}
}  // namespace
void release_overlap_resources() {
    std::lock_guard<std::mutex> lk(g_ovl_mu);
    for (auto& kv : g_ovl) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(kv.first.first);
        if (kv.second.side) { cudaStreamSynchronize(kv.second.side); cudaStreamDestroy(kv.second.side); }
        for (cudaEvent_t e : kv.second.ev) cudaEventDestroy(e);
        cudaSetDevice(cur);
    }
    g_ovl.clear();
}

static int run_volume(const void* positions, int64_t N, const void* form_factors, const xpcs_species* species,
                      const xpcs_qvolume* vol, int64_t frames, void* I_out, const xpcs_opts* opts, int amp) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(positions, "positions");
    NEED(I_out, "I_out");
    POS(N, "N");
    POS(frames, "frames");
    TRY(validate_volume(vol));
    if (frames > (int64_t(1) << 40) / vol->n_l) {
        set_error("xpcs: frames x n_l too large");
        return XPCS_EINVAL;
    }
    Groups G;
    TRY(prep_groups(species, form_factors, N, G));
    TRY(check_sticky());
    const LatticeGeom g = to_geom(vol->plane);
    const int64_t n_q = g.n_h * g.n_k;
    const int64_t n_l = vol->n_l, l0 = vol->l0;
    const int64_t V = frames * n_l;             // virtual frames: (frame, l-plane), row-major = output order
    const size_t isz = out_size(o.out_f64) * (amp ? 2 : 1);
    if (o.in_f64 && (o.engine == XPCS_ENGINE_TENSOR || o.engine == XPCS_ENGINE_TENSOR_I8)) {
        set_error("xpcs: the tensor engines need f32 inputs");
        return XPCS_EUNSUPPORTED;
    }
    bool tc = false, i8 = false;
    if (!o.in_f64 && o.engine != XPCS_ENGINE_SIMT) {
        const bool avail = lattice_tc_supported(g);
        if (!avail && o.engine != XPCS_ENGINE_AUTO) {
            set_error("xpcs: the tensor engine is not available for this grid/build");
            return XPCS_EUNSUPPORTED;
        }
        // AUTO: the integer engine when every atom has f = 1 inside the contraction (form_factors NULL: uniform f, and
        // every kind of a species call); per-atom f keeps the split-FP16 engine (the W scale max|f| costs the small-f
        // atoms limb precision: two-species worst case ~0.8 of the per-pixel gate)
        i8 = avail && (o.engine == XPCS_ENGINE_TENSOR_I8 || (o.engine == XPCS_ENGINE_AUTO && form_factors == nullptr));
        tc = avail && !i8;
    }
    TRY(upload_groups(G, o.s));
    int ng = G.count();
    // engine per atom group.  AUTO with species: the integer engine's limb error grows with the kind's weight, so
    // kinds are taken in increasing max |f_s| (species->f_max, host hints; absent = all equal) while the integer
    // share of the error budget, sum f_max^2 N_s / (f_ref^2 N) with f_ref the smallest weight, stays <= the budget (2.5, i8_budget) -- near the
    // single-species f = 1 level validated against the gate; the heavier kinds run on the split-FP16 engine.
    std::vector<char> gi8((size_t)ng, i8 ? 1 : 0);
    // AUTO species call without f_max hints: the kinds' weights are unknown (f_q lives on the device), so the
    // error budget cannot be applied -- every kind runs on the precise split-FP16 engine (an explicit TENSOR_I8
    // request still puts every kind on the integer engine)
    if (G.n_species && o.engine == XPCS_ENGINE_AUTO && (i8 || tc) && !species->f_max) std::fill(gi8.begin(), gi8.end(), 0);
    if (G.n_species && o.engine == XPCS_ENGINE_AUTO && (i8 || tc) && species->f_max) {
        // kinds in increasing max|f_s|: whole kinds on the integer engine while the budget allows, the kind that
        // crosses it split (its first atoms on the integer engine up to the budget), the rest on split-FP16
        std::vector<int> order((size_t)ng);
        for (int k = 0; k < ng; ++k) order[(size_t)k] = k;
        std::sort(order.begin(), order.end(), [&](int a, int b) { return std::fabs(species->f_max[a]) < std::fabs(species->f_max[b]); });
        double fref = 0.0;
        for (int k : order) if (G.cnt[k] > 0 && std::fabs(species->f_max[k]) > 0.0) { fref = std::fabs(species->f_max[k]); break; }
        std::vector<int64_t> n_int((size_t)ng, 0);
        double budget = 0.0;
        const double cap = i8_budget();
        for (int k : order) {
            const double w2 = fref > 0.0 ? (species->f_max[k] / fref) * (species->f_max[k] / fref) : 1.0;
            const double room = cap + 1e-12 - budget;
            int64_t take = G.cnt[k];
            if (room <= 0.0) take = 0;
            else if (w2 * (double)G.cnt[k] / (double)N > room) take = (int64_t)std::floor(room * (double)N / w2);
            take = std::min<int64_t>(take, G.cnt[k]);
            n_int[(size_t)k] = take;
            budget += w2 * (double)take / (double)N;
        }
        // regroup: [integer part, FP16 part] per kind (empty parts dropped), kind order kept
        std::vector<int64_t> off2, cnt2;
        std::vector<int32_t> kind2;
        std::vector<char> e2;
        for (int k = 0; k < ng; ++k) {
            if (n_int[(size_t)k] > 0) { off2.push_back(G.off[k]); cnt2.push_back(n_int[(size_t)k]); kind2.push_back(G.kind[k]); e2.push_back(1); }
            if (G.cnt[k] > n_int[(size_t)k]) {
                off2.push_back(G.off[k] + n_int[(size_t)k]); cnt2.push_back(G.cnt[k] - n_int[(size_t)k]);
                kind2.push_back(G.kind[k]); e2.push_back(0);
            }
        }
        if ((int)cnt2.size() > kMaxSpecies) {
            set_error("xpcs: too many atom groups after the engine split");
            return XPCS_EUNSUPPORTED;
        }
        G.off = off2; G.cnt = cnt2; G.kind = kind2; gi8 = e2;
    }
    ng = G.count();
    bool any_i8 = false, any_tc = false;
    for (int k = 0; k < ng; ++k) {
        if (G.cnt[k] == 0) continue;
        if (gi8[(size_t)k] && (i8 || tc)) any_i8 = true;
        else if (i8 || tc) any_tc = true;
    }
    if (G.n_species && o.engine == XPCS_ENGINE_AUTO && (i8 || tc)) { i8 = any_i8; tc = any_tc; }
    SpeciesParts sp{};
    sp.n = G.n_species ? ng : 0;
    for (int k = 0; k < ng && k < kMaxSpecies; ++k) sp.kind[k] = G.kind[k];
    if (o.in_f64) {
        // FP64: direct per-pixel evaluation with 64-bit turns; with species each kind's amplitude goes to scratch
        sp.part_f64 = 1;
        const int64_t per_frame = std::max<int64_t>(32 * N, G.n_species ? 16 * n_q * ng : 0);
        const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(V, (int64_t)(kBatchBytes / per_frame)));
        ulonglong4* st = (ulonglong4*)scratch(o.s, SS_STAGE, sizeof(ulonglong4) * (size_t)(N * Tb));
        // split-K over atoms when (pixel blocks x frames) cannot fill ~4 CTAs of 128 threads per SM (config 1: 32
        // blocks); the chunk amplitudes are folded in FP64 in chunk order (k_amp_reduce)
        int64_t C64 = 1, ch64 = N;
        if (!G.n_species) {
            const int64_t blocks = ((n_q + 127) / 128) * std::min(Tb, V);
            const int64_t want = 4LL * sm_count();
            if (blocks < want) {
                C64 = std::min<int64_t>((want + blocks - 1) / blocks, std::max<int64_t>(1, N / 32));
                ch64 = (N + C64 - 1) / C64;
                C64 = (N + ch64 - 1) / ch64;
            }
        }
        double2* part = (G.n_species || C64 > 1)
                            ? (double2*)scratch(o.s, SS_PARTIAL, sizeof(double2) * (size_t)(n_q * Tb * std::max<int64_t>(ng, C64)))
                            : nullptr;
        if (!st || ((G.n_species || C64 > 1) && !part)) return XPCS_ENOMEM;
        for (int64_t v0 = 0; v0 < V; v0 += Tb) {
            const int64_t vb = std::min(Tb, V - v0);
            void* dst = (char*)I_out + isz * n_q * v0;
            int64_t stoff = 0;
            for (int gi = 0; gi < ng; ++gi) {
                const int64_t Ng = G.cnt[gi];
                double2* pg = part ? part + (size_t)gi * (size_t)(n_q * vb) : nullptr;
                sp.part[gi] = pg;
                sp.C[gi] = Ng > 0 ? 1 : 0;
                if (Ng == 0) continue;
                const StageMap m = stage_map(G, gi, N, v0, n_l, l0, vol->mc);
                { ProfScope p(o.profile, KC_STAGE, o.s);
                  TRY(cuda_fail(launch_stage_lattice64(positions, form_factors, Ng, vb, g, m, st + stoff, o.s), "stage")); }
                { ProfScope p(o.profile, KC_MAIN, o.s);
                  if (G.n_species) TRY(cuda_fail(launch_lattice_f64(st + stoff, Ng, vb, g, pg, 1, 1, o.s), "lattice64"));
                  else if (C64 > 1) TRY(cuda_fail(launch_lattice_f64(st + stoff, Ng, vb, g, nullptr, o.out_f64, amp, o.s,
                                                                     part, ch64, C64), "lattice64"));
                  else TRY(cuda_fail(launch_lattice_f64(st + stoff, Ng, vb, g, dst, o.out_f64, amp, o.s), "lattice64")); }
                stoff += Ng * vb;
            }
            if (G.n_species) {
                ProfScope p(o.profile, KC_REDUCE, o.s);
                TRY(cuda_fail(launch_species_combine(sp, vb, n_q, G.fq, 1, v0, n_l, dst, o.out_f64, amp, o.s), "species combine"));
            } else if (C64 > 1) {
                ProfScope p(o.profile, KC_REDUCE, o.s);
                TRY(cuda_fail(launch_amp_reduce_d(part, C64, vb, n_q, dst, o.out_f64, amp, o.s), "reduce"));
            }
        }
        return XPCS_OK;
    }
    // atom chunks (split-K over CTAs, folded in FP64 by the reduction): SIMT keeps fp32 register sums short
    // (<= 4096 atoms) and splits further (>= 512 atoms per chunk) when tiles x frames cannot fill ~2 waves; the
    // tensor engine drains TMEM every 256 atoms into RN sums, so its chunks only balance the grid (>= ~8 waves of
    // one CTA per SM) and stay >= 1024 atoms.  The chunking depends on the frame count of the call only through the
    // grid-fill rule (when the 1024-atom floor binds, splitting the frames over several calls is bit-identical).
    std::vector<int64_t> chunk(ng, 4096), C(ng, 0);
    int64_t sumC = 0;
    for (int gi = 0; gi < ng; ++gi) {
        const int64_t Ng = G.cnt[gi];
        if (Ng == 0) continue;
        int64_t ch = 4096;
        const bool g_i8 = i8 && gi8[(size_t)gi], g_tc = (i8 || tc) && !g_i8;
        if (g_i8) {
            // exact int32 accumulation: chunks only balance the grid (clusters of 2 CTAs, one CTA per SM) and stay
            // <= kI8MaxChunk.  Cost model in 32-atom stage units: waves x (stages per CTA + a fixed per-CTA cost of
            // ~15 stages for the prologue, the single drain and the cluster teardown); the smallest C wins ties.
            ch = i8_plan_chunk(Ng, i8_tiles(g) * V, nullptr);
        } else if (g_tc) {
            const int64_t tiles = ((g.n_h + 255) / 256) * ((g.n_k + 127) / 128);
            const int64_t units = tiles * std::min<int64_t>(V, 64);
            int64_t C0 = std::max<int64_t>(1, (8LL * sm_count() + units - 1) / units);
            C0 = std::min<int64_t>(C0, std::max<int64_t>(1, Ng / 1024));
            ch = ((Ng + C0 - 1) / C0 + 15) / 16 * 16;
        } else {
            const int64_t units = ((g.n_h + 63) / 64) * ((g.n_k + 127) / 128) * V;
            const int64_t want = 2LL * sm_count() * 4;
            if (units * ((Ng + 4095) / 4096) < want) {
                const int64_t C0 = std::min<int64_t>((want + units - 1) / units, std::max<int64_t>(1, Ng / 512));
                ch = std::min<int64_t>(4096, ((Ng + C0 - 1) / C0 + 15) / 16 * 16);
            }
        }
        if (const char* e = getenv("XPCS_CHUNK_ATOMS")) ch = std::max<int64_t>(16, atoll(e));   // experiments only
        chunk[gi] = ch;
        C[gi] = (Ng + ch - 1) / ch;
        sumC += C[gi];
    }
    sp.part_f64 = 0;
    // XPCS_BATCH_BYTES (tests and experiments): a smaller cap forces many frame batches (results do not depend on it)
    const char* bb_env = getenv("XPCS_BATCH_BYTES");
    const int64_t batch_bytes = bb_env ? std::max<int64_t>(1, atoll(bb_env)) : (int64_t)kBatchBytes;
    const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(V, batch_bytes / std::max<int64_t>(16 * N, 8 * sumC * n_q)));
    // frame batches: memory-bounded (Tb).  A single integer-engine group in one batch is split in two when that
    // shortens the last, partly filled wave of clusters: the leading frames fill whole waves with unsplit atom
    // ranges, the remaining frames get their own atom chunking (cost model of i8_plan_chunk), e.g. c2: 100 frames x
    // 2 tiles on 74 cluster slots = 2.7 waves of 1000 stages -> 74 frames (2 waves) + 26 frames in 7 chunks.
    struct FrameBatch { int64_t v0, vb, chunk; };
    std::vector<FrameBatch> batches;
    int64_t part_elems = sumC * n_q * Tb;
    {
        const bool single_i8 = ng == 1 && !G.n_species && i8 && gi8[0] && G.cnt[0] > 0 && V <= Tb &&
                               !getenv("XPCS_CHUNK_ATOMS") && !(getenv("XPCS_I8_TAILSPLIT") && atoi(getenv("XPCS_I8_TAILSPLIT")) == 0);
        int64_t V1 = 0, ch1 = chunk[0], ch2 = chunk[0];
        if (single_i8) i8_plan_split(G.cnt[0], i8_tiles(g), V, V1, ch1, ch2);
        if (V1 > 0) {
            batches.push_back({0, V1, ch1});
            batches.push_back({V1, V - V1, ch2});
            const int64_t C1 = (G.cnt[0] + ch1 - 1) / ch1, C2 = (G.cnt[0] + ch2 - 1) / ch2;
            part_elems = std::max(C1 * V1, C2 * (V - V1)) * n_q;
        } else {
            for (int64_t v0 = 0; v0 < V; v0 += Tb) batches.push_back({v0, std::min(Tb, V - v0), 0});
        }
    }
    // two buffer sets and the side stream when the frames run in several batches (see overlap_resources)
    OverlapRes* ovl = (batches.size() > 1 && batch_overlap_enabled()) ? overlap_resources(o.s, batches.size() + 2) : nullptr;
    uint4* stb[2] = {(uint4*)scratch(o.s, SS_STAGE, sizeof(uint4) * (size_t)(N * Tb)), nullptr};
    float2* partb[2] = {(float2*)scratch(o.s, SS_PARTIAL, sizeof(float2) * (size_t)part_elems), nullptr};
    if (!stb[0] || !partb[0]) return XPCS_ENOMEM;
    if (ovl) {
        stb[1] = (uint4*)scratch(o.s, SS_STAGE2, sizeof(uint4) * (size_t)(N * Tb));
        partb[1] = (float2*)scratch(o.s, SS_PARTIAL2, sizeof(float2) * (size_t)part_elems);
        if (!stb[1] || !partb[1]) return XPCS_ENOMEM;
    }
    float* fmax0 = nullptr;   // max |f| per buffer set (written by the engine launch, read by its batch's fix-up)
    if ((i8 || tc) && form_factors) {
        fmax0 = (float*)scratch(o.s, SS_SMALL, 128);
        if (!fmax0) return XPCS_ENOMEM;
    }
    // the tensor engines' partials hold conj(p) (R1)
    const int mode = amp ? ((tc || i8) ? 2 : 1) : 0;
    void* fbufb[2] = {nullptr, nullptr};
    if ((i8 || tc) && fixup_enabled()) {
        int64_t vb_max = 0;
        for (const FrameBatch& fb : batches) vb_max = std::max(vb_max, fb.vb);
        fbufb[0] = scratch(o.s, SS_FIX, fixup_scratch_bytes(vb_max, n_q, N));
        if (!fbufb[0]) return XPCS_ENOMEM;
        if (ovl) {
            fbufb[1] = scratch(o.s, SS_FIX2, fixup_scratch_bytes(vb_max, n_q, N));
            if (!fbufb[1]) return XPCS_ENOMEM;
        }
    }
    // the side stream joins the caller's stream (fork) and is joined back before returning, also on errors
    cudaEvent_t ev_join = nullptr;
    if (ovl) {
        TRY(cuda_fail(cudaEventRecord(ovl->ev[0], o.s), "fork"));
        TRY(cuda_fail(cudaStreamWaitEvent(ovl->side, ovl->ev[0], 0), "fork"));
        ev_join = ovl->ev[1];
    }
    struct Join {
        OverlapRes* r; cudaEvent_t e; cudaStream_t s;
        ~Join() { if (r) { cudaEventRecord(e, r->side); cudaStreamWaitEvent(s, e, 0); } }
    } join{ovl, ev_join, o.s};
    for (size_t bi = 0; bi < batches.size(); ++bi) {
        const FrameBatch& fb = batches[bi];
        const int64_t v0 = fb.v0, vb = fb.vb;
        const int par = ovl ? (int)(bi & 1) : 0;
        const cudaStream_t sb = par ? ovl->side : o.s;
        uint4* st = stb[par];
        float2* part = partb[par];
        void* fbuf = fbufb[par];
        float* fmax = fmax0 ? fmax0 + 16 * par : nullptr;
        if (fb.chunk > 0) { chunk[0] = fb.chunk; C[0] = (G.cnt[0] + fb.chunk - 1) / fb.chunk; }
        void* dst = (char*)I_out + isz * n_q * v0;
        // one integer-engine group in a single atom chunk: the kernel writes the result itself (no partial planes)
        const bool direct = ng == 1 && !G.n_species && i8 && gi8[0] && G.cnt[0] > 0 && C[0] == 1 &&
                            !(getenv("XPCS_I8_DIRECT") && atoi(getenv("XPCS_I8_DIRECT")) == 0);
        // the tensor engines' errors add coherently where the phasors repeat (q = 0 and the Bragg peaks of perfect
        // crystals: the integer engine's 16-bit limbs, the split-FP16 engine's truncating FP32 accumulator): the
        // epilogue lists the brightest pixels and k_fixup.cu recomputes them exactly
        const bool fix = (i8 || tc) && fbuf;
        BrightSink bs{nullptr, nullptr, 0.0, nullptr};
        if (fix) TRY(cuda_fail(fixup_prepare(fbuf, N, form_factors ? fmax : nullptr, bs, sb), "bright-pixel list"));
        int64_t stoff = 0, poff = 0;
        bool waited = false;
        for (int gi = 0; gi < ng; ++gi) {
            const int64_t Ng = G.cnt[gi];
            sp.part[gi] = part + poff;
            sp.C[gi] = C[gi];
            if (Ng == 0) continue;
            const StageMap m = stage_map(G, gi, N, v0, n_l, l0, vol->mc);
            { ProfScope p(o.profile, KC_STAGE, sb);
              TRY(cuda_fail(launch_stage_lattice32(positions, 0, form_factors, 0, Ng, vb, g, m, st + stoff, sb), "stage")); }
            if (ovl && bi > 0 && !waited) {   // engines in batch order
                TRY(cuda_fail(cudaStreamWaitEvent(sb, ovl->ev[2 + bi - 1], 0), "batch order"));
                waited = true;
            }
            { ProfScope p(o.profile, KC_MAIN, sb);
              const bool g_i8 = i8 && gi8[(size_t)gi], g_tc = (i8 || tc) && !g_i8;
              ProfScope pe(o.profile && (g_i8 || g_tc), g_i8 ? KC_I8 : KC_TC, sb);
              if (g_i8) TRY(cuda_fail(launch_lattice_i8(st + stoff, Ng, vb, g, chunk[gi], C[gi], fmax, form_factors == nullptr,
                                                      part + poff, sb, direct ? dst : nullptr, o.out_f64, mode,
                                                      (fix && direct) ? &bs : nullptr),
                                    "lattice tcgen05 i8"));
              else if (g_tc) {
                  if (fmax) TRY(cuda_fail(launch_absmax_f(st + stoff, Ng, fmax, sb), "max |f|"));   // the fix-up threshold
                  TRY(cuda_fail(launch_lattice_tc(st + stoff, Ng, vb, g, chunk[gi], C[gi], part + poff, sb), "lattice tcgen05"));
              }
              else TRY(cuda_fail(launch_lattice_simt(st + stoff, Ng, vb, g, chunk[gi], C[gi], part + poff, sb), "lattice simt")); }
            stoff += Ng * vb;
            poff += C[gi] * n_q * vb;
        }
        if (ovl) TRY(cuda_fail(cudaEventRecord(ovl->ev[2 + bi], sb), "batch order"));   // this batch's engines done
        if (!direct) {
            ProfScope p(o.profile, KC_REDUCE, sb);
            if (G.n_species) TRY(cuda_fail(launch_species_combine(sp, vb, n_q, G.fq, 0, v0, n_l, dst, o.out_f64, mode, sb,
                                                                  fix ? &bs : nullptr), "species combine"));
            else TRY(cuda_fail(launch_amp_reduce_f(part, C[0], vb, n_q, dst, o.out_f64, mode, sb, fix ? &bs : nullptr), "reduce"));
        }
        if (fix) {
            FixGroups fg{};
            int64_t off = 0;
            for (int gi = 0; gi < ng; ++gi) {
                if (G.cnt[gi] > 0) {
                    fg.st[fg.n_groups] = st + off;
                    fg.n[fg.n_groups] = G.cnt[gi];
                    fg.kind[fg.n_groups] = G.kind[gi];
                    ++fg.n_groups;
                }
                off += G.cnt[gi] * vb;
            }
            fg.fq = G.n_species ? G.fq : nullptr;
            fg.fq_f64 = 0;
            fg.v0 = v0;
            fg.n_l = n_l;
            ProfScope p(o.profile, KC_FIXUP, sb);
            TRY(cuda_fail(launch_fixup(fg, g, vb, dst, o.out_f64, amp ? 1 : 0, fbuf, sb), "bright-pixel recompute"));
        }
    }
    return XPCS_OK;
}

static xpcs_qvolume plane_volume(const xpcs_qgrid* grid) {
    xpcs_qvolume v;
    std::memset(&v, 0, sizeof(v));
    if (grid) v.plane = *grid;
    v.l0 = 0;
    v.n_l = 1;
    return v;
}

extern "C" {

int xpcs_intensity(const void* positions, int64_t N, const void* form_factors, const void* q_vectors, int64_t n_q,
                   int64_t frames, double box_L, void* I_out, const xpcs_opts* opts) {
    return run_direct(positions, N, form_factors, nullptr, q_vectors, n_q, frames, box_L, I_out, opts, 0);
}
int xpcs_amplitude(const void* positions, int64_t N, const void* form_factors, const void* q_vectors, int64_t n_q,
                   int64_t frames, double box_L, void* A_out, const xpcs_opts* opts) {
    return run_direct(positions, N, form_factors, nullptr, q_vectors, n_q, frames, box_L, A_out, opts, 1);
}
int xpcs_intensity_species(const void* positions, int64_t N, const xpcs_species* species, const void* q_vectors,
                           int64_t n_q, int64_t frames, double box_L, void* I_out, const xpcs_opts* opts) {
    if (!species) { clear_error(); set_error("xpcs: species must not be NULL"); return XPCS_EINVAL; }
    return run_direct(positions, N, nullptr, species, q_vectors, n_q, frames, box_L, I_out, opts, 0);
}
int xpcs_amplitude_species(const void* positions, int64_t N, const xpcs_species* species, const void* q_vectors,
                           int64_t n_q, int64_t frames, double box_L, void* A_out, const xpcs_opts* opts) {
    if (!species) { clear_error(); set_error("xpcs: species must not be NULL"); return XPCS_EINVAL; }
    return run_direct(positions, N, nullptr, species, q_vectors, n_q, frames, box_L, A_out, opts, 1);
}
int xpcs_intensity_grid(const void* positions, int64_t N, const void* form_factors, const xpcs_qgrid* grid,
                        int64_t frames, void* I_out, const xpcs_opts* opts) {
    if (!grid) { clear_error(); set_error("xpcs: grid must not be NULL"); return XPCS_EINVAL; }
    const xpcs_qvolume v = plane_volume(grid);
    return run_volume(positions, N, form_factors, nullptr, &v, frames, I_out, opts, 0);
}
int xpcs_amplitude_grid(const void* positions, int64_t N, const void* form_factors, const xpcs_qgrid* grid,
                        int64_t frames, void* A_out, const xpcs_opts* opts) {
    if (!grid) { clear_error(); set_error("xpcs: grid must not be NULL"); return XPCS_EINVAL; }
    const xpcs_qvolume v = plane_volume(grid);
    return run_volume(positions, N, form_factors, nullptr, &v, frames, A_out, opts, 1);
}
int xpcs_intensity_volume(const void* positions, int64_t N, const void* form_factors, const xpcs_species* species,
                          const xpcs_qvolume* vol, int64_t frames, void* I_out, const xpcs_opts* opts) {
    return run_volume(positions, N, form_factors, species, vol, frames, I_out, opts, 0);
}
int xpcs_amplitude_volume(const void* positions, int64_t N, const void* form_factors, const xpcs_species* species,
                          const xpcs_qvolume* vol, int64_t frames, void* A_out, const xpcs_opts* opts) {
    return run_volume(positions, N, form_factors, species, vol, frames, A_out, opts, 1);
}

int xpcs_intensity_fft(const void* positions, int64_t N, int64_t frames, const xpcs_qvolume* block, int32_t n_grid,
                       double eta, int32_t k_cut, const void* f_q, void* I_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(positions, "positions");
    NEED(I_out, "I_out");
    POS(N, "N");
    POS(frames, "frames");
    TRY(validate_volume(block));
    const xpcs_qgrid& pl = block->plane;
    const bool axes = pl.m0[0] == 0 && pl.m0[1] == 0 && pl.m0[2] == 0 && pl.ma[0] == 1 && pl.ma[1] == 0 &&
                      pl.ma[2] == 0 && pl.mb[0] == 0 && pl.mb[1] == 1 && pl.mb[2] == 0 && block->mc[0] == 0 &&
                      block->mc[1] == 0 && block->mc[2] == 1;
    if (!axes) {
        set_error("xpcs: the FFT method returns an axis-aligned block of its grid (m0 = 0, ma = x, mb = y, mc = z)");
        return XPCS_EINVAL;
    }
    if (n_grid < 8 || n_grid > 1024 || (n_grid & 1)) {
        set_error("xpcs: n_grid must be even and in [8, 1024] (got %d)", n_grid);
        return XPCS_EINVAL;
    }
    if (!(eta > 0.0) || !std::isfinite(eta)) {
        set_error("xpcs: eta must be finite and > 0");
        return XPCS_EINVAL;
    }
    const double L = pl.L;
    int k = k_cut;
    if (k <= 0) {   // the paper's rule: the nearest integer greater than 10 eta (grid units), made odd (R16)
        const double kk = std::floor(10.0 * eta / (L / n_grid)) + 1.0;
        k = kk > 64.0 ? 65 : (int)kk;
        if (!(k & 1)) ++k;
    }
    if (!(k & 1) || k > 31 || k > n_grid) {
        set_error("xpcs: the kernel width k must be odd, <= 31 and <= n_grid (got %d)", k);
        return XPCS_EINVAL;
    }
    const int64_t lo = -(int64_t)(n_grid / 2), hi = n_grid / 2 - 1;
    if (pl.h0 < lo || pl.h0 + pl.n_h - 1 > hi || pl.k0 < lo || pl.k0 + pl.n_k - 1 > hi || block->l0 < lo ||
        block->l0 + block->n_l - 1 > hi) {
        set_error("xpcs: block indices must lie in [-n_grid/2, n_grid/2 - 1]");
        return XPCS_EINVAL;
    }
    TRY(check_sticky());
    const int64_t n3 = (int64_t)n_grid * n_grid * n_grid;
    const int64_t per_frame = 8 * n3 + 16 * (int64_t)n_grid * n_grid * (n_grid / 2 + 1);
    const int64_t Tb = std::max<int64_t>(1, std::min<int64_t>(frames, (int64_t)(2 * kBatchBytes) / per_frame));
    char* buf = (char*)scratch(o.s, SS_FFT, (size_t)(per_frame * Tb) + 256);
    if (!buf) return XPCS_ENOMEM;
    double* rho = (double*)buf;
    double2* spec = (double2*)(buf + ((8 * n3 * Tb + 255) / 256) * 256);
    const int64_t blk = block->n_l * pl.n_h * pl.n_k;
    const size_t psz = o.in_f64 ? 24 : 12;
    for (int64_t t0 = 0; t0 < frames; t0 += Tb) {
        const int64_t tb = std::min(Tb, frames - t0);
        const char* what = "";
        ProfScope p(o.profile, KC_MAIN, o.s);
        const int rc = launch_fft_intensity((const char*)positions + psz * N * t0, o.in_f64, N, tb, L, n_grid, eta, k,
                                            rho, spec, pl.h0, pl.n_h, pl.k0, pl.n_k, block->l0, block->n_l, f_q,
                                            o.in_f64, (char*)I_out + out_size(o.out_f64) * blk * t0, o.out_f64, o.s,
                                            &what);
        if (rc == 2) return cuda_fail(cudaGetLastError(), what);
        if (rc == 3) {
            set_error("xpcs: cuFFT %s failed", what);
            return XPCS_ECUDA;
        }
    }
    return XPCS_OK;
}

int xpcs_form_factor_gaussian(const void* q_vectors, int64_t n_q, const xpcs_qvolume* vol, int32_t n_gauss,
                              const double* a, const double* b, double c, void* f_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(f_out, "f_out");
    if (n_gauss < 0 || n_gauss > 6) {
        set_error("xpcs: n_gauss must be in [0, 6] (got %d)", n_gauss);
        return XPCS_EINVAL;
    }
    if (n_gauss > 0) { NEED(a, "a"); NEED(b, "b"); }
    LatticeGeom g{};
    int64_t l0 = 0, n_l = 1;
    const int32_t* mc = nullptr;
    if (q_vectors) {
        POS(n_q, "n_q");
    } else {
        if (!vol) {
            set_error("xpcs: q_vectors and vol must not both be NULL");
            return XPCS_EINVAL;
        }
        TRY(validate_volume(vol));
        g = to_geom(vol->plane);
        l0 = vol->l0;
        n_l = vol->n_l;
        mc = vol->mc;
    }
    TRY(check_sticky());
    return cuda_fail(launch_form_factor_gaussian(q_vectors, o.in_f64, n_q, g, l0, n_l, mc, n_gauss, a, b, c, f_out,
                                                 o.out_f64, o.s), "form factor");
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
    const int32_t* dl = lag_table(lags, n_lags, o.s);
    if (!dl) return XPCS_ECUDA;
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
    const int32_t* dl = lag_table(lags, n_lags, o.s);
    if (!dl) return XPCS_ECUDA;
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
    for (int64_t w0 = 0; w0 < n_windows; w0 += 8) {   // windows per k_xsvs_warp pass (XW in k_stats.cu)
        int64_t s = 0;
        for (int64_t i = w0; i < std::min(n_windows, w0 + 8); ++i) {
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
    // per-warp moments, then the per-(slot, ring) moments (summed over the ring's warps), then beta from those
    int64_t all_slots = 0;
    for (int64_t i = 0; i < n_windows; ++i) all_slots += frames / windows[i];
    const size_t warp_bytes = sizeof(double2) * (size_t)(pb.max_warps * max_slots);
    double* mom = (double*)scratch(o.s, SS_XSVS, warp_bytes + sizeof(double) * 3 * (size_t)(all_slots * n_bins));
    if (!mom) return XPCS_ENOMEM;
    double* ring_mom = (double*)((char*)mom + warp_bytes);
    TRY(cuda_fail(launch_xsvs(I_series, o.in_f64, frames, n_q, pb.plan, n_bins, windows, n_windows, pb.max_warps,
                              mom, ring_mom, o.s), "xsvs"));
    return cuda_fail(launch_xsvs_beta_from_moments(ring_mom, frames, windows, n_windows, n_bins, beta_out, o.s), "xsvs beta");
}

// ------------------------------------------------------------------------------------------- block-streamed g2
static int g2_lag_check(const int32_t* lags, int64_t n_lags, int64_t frames, int& max_lag) {
    max_lag = 0;
    for (int64_t i = 0; i < n_lags; ++i) {
        if (lags[i] < 0 || (frames > 0 && lags[i] >= frames)) {
            set_error("xpcs: lag %d out of range [0, %lld)", lags[i], (long long)frames);
            return XPCS_EINVAL;
        }
        max_lag = std::max(max_lag, (int)lags[i]);
    }
    if (max_lag > 640) {
        set_error("xpcs: lags > 640 frames are not supported by this build");
        return XPCS_EUNSUPPORTED;
    }
    return XPCS_OK;
}

int xpcs_g2_accumulate(const void* I_block, int64_t block_frames, int64_t t0, int64_t n_q, const int32_t* lags,
                       int64_t n_lags, void* ring, int64_t ring_frames, double* acc, double* sum,
                       const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(I_block, "I_block");
    NEED(lags, "lags");
    NEED(acc, "acc");
    NEED(sum, "sum");
    POS(block_frames, "block_frames");
    POS(n_q, "n_q");
    POS(n_lags, "n_lags");
    if (t0 < 0) {
        set_error("xpcs: t0 must be >= 0");
        return XPCS_EINVAL;
    }
    int max_lag = 0;
    for (int64_t i = 0; i < n_lags; ++i)
        if (lags[i] < 0) {
            set_error("xpcs: lag %d out of range (negative)", lags[i]);
            return XPCS_EINVAL;
        }
    TRY(g2_lag_check(lags, n_lags, 0, max_lag));
    if (ring_frames < max_lag || (ring_frames > 0 && !ring)) {
        set_error("xpcs: the frame ring must hold at least the largest lag (%d frames; got %lld)", max_lag,
                  (long long)ring_frames);
        return XPCS_EINVAL;
    }
    TRY(check_sticky());
    const int32_t* dl = lag_table(lags, n_lags, o.s);
    if (!dl) return XPCS_ECUDA;
    ProfScope p(o.profile, KC_G2, o.s);
    return cuda_fail(launch_g2_accumulate(I_block, o.in_f64, block_frames, ring, ring_frames, t0, n_q, dl, n_lags,
                                          max_lag, acc, sum, o.s), "g2 accumulate");
}

int xpcs_g2_finalize(const double* acc, const double* sum, int64_t frames, int64_t n_q, const int32_t* lags,
                     int64_t n_lags, void* g2_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(acc, "acc");
    NEED(sum, "sum");
    NEED(lags, "lags");
    NEED(g2_out, "g2_out");
    POS(frames, "frames");
    POS(n_q, "n_q");
    POS(n_lags, "n_lags");
    int max_lag = 0;
    TRY(g2_lag_check(lags, n_lags, frames, max_lag));
    TRY(check_sticky());
    const int32_t* dl = lag_table(lags, n_lags, o.s);
    if (!dl) return XPCS_ECUDA;
    ProfScope p(o.profile, KC_G2, o.s);
    return cuda_fail(launch_g2_finalize(acc, sum, frames, n_q, dl, n_lags, g2_out, o.out_f64, o.s), "g2 finalize");
}

// ------------------------------------------------------------------------------------------- ring moments
// (the additive form of the ring reductions: a detector split across devices adds these before forming the
// means / beta)
static int window_slots(const int32_t* windows, int64_t n_windows, int64_t frames, int64_t& n_slots, int64_t& max_pass) {
    n_slots = 0;
    max_pass = 0;
    for (int64_t w0 = 0; w0 < n_windows; w0 += 8) {   // windows per XSVS pass (XW in k_stats.cu)
        int64_t sp = 0;
        for (int64_t i = w0; i < std::min(n_windows, w0 + 8); ++i) {
            if (windows[i] < 1 || windows[i] > frames) {
                set_error("xpcs: window %d out of range [1, %lld]", windows[i], (long long)frames);
                return XPCS_EINVAL;
            }
            sp += frames / windows[i];
        }
        n_slots += sp;
        max_pass = std::max(max_pass, sp);
    }
    return XPCS_OK;
}

int xpcs_ring_moments(const void* values, int64_t rows, int64_t n_q, const int32_t* bin_of_q, int32_t n_bins,
                      double* moments_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(values, "values");
    NEED(bin_of_q, "bin_of_q");
    NEED(moments_out, "moments_out");
    POS(rows, "rows");
    POS(n_q, "n_q");
    POS(n_bins, "n_bins");
    TRY(check_sticky());
    ProfScope p(o.profile, KC_RINGS, o.s);
    PlanBufs pb;
    TRY(make_plan(bin_of_q, n_q, n_bins, o.s, pb));
    return cuda_fail(launch_shell_moments(values, o.in_f64, rows, n_q, pb.plan, n_bins, moments_out, o.s), "ring moments");
}

int xpcs_ring_means_from_moments(const double* moments, int64_t rows, int32_t n_bins, double scale,
                                 const void* form_factors, int64_t N, double* out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(moments, "moments");
    NEED(out, "out");
    POS(rows, "rows");
    POS(n_bins, "n_bins");
    if (form_factors) POS(N, "N");
    TRY(check_sticky());
    double* norm = nullptr;
    if (form_factors) {
        norm = (double*)scratch(o.s, SS_SMALL, 64);
        if (!norm) return XPCS_ENOMEM;
        TRY(cuda_fail(launch_sum_f2(form_factors, o.in_f64, N, norm, o.s), "sum f^2"));
    }
    return cuda_fail(launch_ring_means_from_moments(moments, rows * n_bins, scale, norm, out, o.s), "ring means");
}

int xsvs_moments(const void* I_series, int64_t frames, int64_t n_q, const int32_t* bin_of_q, int32_t n_bins,
                 const int32_t* windows, int64_t n_windows, double* moments_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(I_series, "I_series");
    NEED(bin_of_q, "bin_of_q");
    NEED(windows, "windows");
    NEED(moments_out, "moments_out");
    POS(frames, "frames");
    POS(n_q, "n_q");
    POS(n_bins, "n_bins");
    POS(n_windows, "n_windows");
    int64_t n_slots = 0, max_pass = 0;
    TRY(window_slots(windows, n_windows, frames, n_slots, max_pass));
    TRY(check_sticky());
    ProfScope p(o.profile, KC_XSVS, o.s);
    PlanBufs pb;
    TRY(make_plan(bin_of_q, n_q, n_bins, o.s, pb));
    double* mom = (double*)scratch(o.s, SS_XSVS, sizeof(double2) * (size_t)(pb.max_warps * max_pass));
    if (!mom) return XPCS_ENOMEM;
    return cuda_fail(launch_xsvs(I_series, o.in_f64, frames, n_q, pb.plan, n_bins, windows, n_windows, pb.max_warps,
                                 mom, moments_out, o.s), "xsvs moments");
}

int xsvs_contrast_from_moments(const double* moments, int64_t frames, const int32_t* windows, int64_t n_windows,
                               int32_t n_bins, double* beta_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(moments, "moments");
    NEED(windows, "windows");
    NEED(beta_out, "beta_out");
    POS(frames, "frames");
    POS(n_bins, "n_bins");
    POS(n_windows, "n_windows");
    int64_t n_slots = 0, max_pass = 0;
    TRY(window_slots(windows, n_windows, frames, n_slots, max_pass));
    TRY(check_sticky());
    return cuda_fail(launch_xsvs_beta_from_moments(moments, frames, windows, n_windows, n_bins, beta_out, o.s), "beta");
}

int xpcs_rings_register(const int32_t* bin_of_q, int64_t n_q, int32_t n_bins, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(bin_of_q, "bin_of_q");
    POS(n_q, "n_q");
    POS(n_bins, "n_bins");
    if (n_bins > 12288 || n_q > (int64_t(1) << 31) - 1) {
        set_error("xpcs: ring plan limits: n_bins <= 12288, n_q < 2^31");
        return XPCS_EINVAL;
    }
    TRY(check_sticky());
    xpcs_rings_unregister(bin_of_q);
    clear_error();
    RegisteredPlan r{};
    r.bins = bin_of_q;
    r.n_q = n_q;
    r.n_bins = n_bins;
    cudaGetDevice(&r.device);
    TRY(cuda_fail(cudaMalloc(&r.mem, plan_bytes(n_q, n_bins)), "cudaMalloc (ring plan)"));
    const int rc = build_plan(bin_of_q, n_q, n_bins, o.s, r.mem, r.pb);
    if (rc != XPCS_OK) {
        cudaFree(r.mem);
        return rc;
    }
    registered().push_back(r);
    return XPCS_OK;
}

int xpcs_rings_unregister(const int32_t* bin_of_q) {
    clear_error();
    auto& v = registered();
    for (size_t i = 0; i < v.size(); ++i)
        if (v[i].bins == bin_of_q) {
            cudaDeviceSynchronize();   // work enqueued with the plan may still be reading it
            cudaFree(v[i].mem);
            v.erase(v.begin() + (long)i);
            return XPCS_OK;
        }
    set_error("xpcs: bin_of_q %p is not registered", (const void*)bin_of_q);
    return XPCS_EINVAL;
}

int xpcs_speckle_histogram(const void* I_series, int64_t frames, int64_t n_q, const int32_t* bin_of_q, int32_t n_bins,
                           int32_t M, int32_t n_hist, double kappa_max, int64_t* counts_out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(I_series, "I_series");
    NEED(bin_of_q, "bin_of_q");
    NEED(counts_out, "counts_out");
    POS(frames, "frames");
    POS(n_q, "n_q");
    POS(n_bins, "n_bins");
    if (M < 1 || M > frames) {
        set_error("xpcs: M = %d out of range [1, %lld]", M, (long long)frames);
        return XPCS_EINVAL;
    }
    if (n_hist < 1 || n_hist > (1 << 20)) {
        set_error("xpcs: n_hist must be in [1, 2^20] (got %d)", n_hist);
        return XPCS_EINVAL;
    }
    if (!(kappa_max > 0.0) || !std::isfinite(kappa_max)) {
        set_error("xpcs: kappa_max must be finite and > 0");
        return XPCS_EINVAL;
    }
    if (n_q > (int64_t(1) << 31) - 1) {
        set_error("xpcs: n_q too large for the ring plan");
        return XPCS_EINVAL;
    }
    TRY(check_sticky());
    ProfScope p(o.profile, KC_XSVS, o.s);
    PlanBufs pb;
    TRY(make_plan(bin_of_q, n_q, n_bins, o.s, pb));
    const int64_t S = frames / M;
    double* mom = (double*)scratch(o.s, SS_XSVS, sizeof(double2) * (size_t)(pb.max_warps * S) + sizeof(double) * (size_t)(S * n_bins));
    if (!mom) return XPCS_ENOMEM;
    double* means = mom + 2 * (size_t)(pb.max_warps * S);
    return cuda_fail(launch_speckle_hist(I_series, o.in_f64, frames, n_q, pb.plan, n_bins, M, pb.max_warps, mom, means,
                                         n_hist, kappa_max, counts_out, o.s), "speckle histogram");
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

}  // extern "C"
// S(q,t) ring means with the form factors' own dtype (xpcs_step_host: I is out_dtype, f the caller's in_dtype)
static int structure_factor_shells(const void* I, int64_t rows, int64_t n_q, const void* form_factors, int ff_f64,
                                   int64_t N, const int32_t* bin_of_q, int32_t n_bins, double* out, const Opts& o) {
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
        TRY(cuda_fail(launch_sum_f2(form_factors, ff_f64, N, norm, o.s), "sum f^2"));
    } else {
        scale = 1.0 / (double)N;     // sum_j f_j^2 = N for unit form factors
    }
    return cuda_fail(launch_shell_mean(I, o.in_f64, rows, n_q, pb.plan, n_bins, scale, norm, out, o.s), "rings");
}
extern "C" {

int xpcs_structure_factor_shells(const void* I, int64_t rows, int64_t n_q, const void* form_factors, int64_t N,
                                 const int32_t* bin_of_q, int32_t n_bins, double* out, const xpcs_opts* opts) {
    clear_error();
    Opts o;
    TRY(parse_opts(opts, o));
    return structure_factor_shells(I, rows, n_q, form_factors, o.in_f64 ? 1 : 0, N, bin_of_q, n_bins, out, o);
}

// ------------------------------------------------------------------------------------------- host-buffer step
}  // extern "C"
namespace {
// internal copy streams and events of xpcs_step_host, per (device, caller stream); created on first use (outside any
// graph capture) and kept until xpcs_release
struct HostRes {
    cudaStream_t h2d = nullptr, d2h = nullptr, red = nullptr;   // copies in, copies out, a side stream for reductions
    std::vector<cudaEvent_t> ev;
};
std::mutex g_host_mu;
std::map<std::pair<int, cudaStream_t>, HostRes> g_host_res;   // node-based: references stay valid

int host_resources(cudaStream_t s, size_t n_events, HostRes*& out) {
    std::lock_guard<std::mutex> lk(g_host_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    auto it = g_host_res.find({dev, s});
    HostRes* r = it == g_host_res.end() ? nullptr : &it->second;
    if (!r || r->ev.size() < n_events) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
            set_error("xpcs: xpcs_step_host must run once on this stream outside a graph capture first");
            return XPCS_EUNSUPPORTED;
        }
        if (!r) {
            r = &g_host_res[{dev, s}];
            if (cudaStreamCreateWithFlags(&r->h2d, cudaStreamNonBlocking) != cudaSuccess ||
                cudaStreamCreateWithFlags(&r->d2h, cudaStreamNonBlocking) != cudaSuccess ||
                cudaStreamCreateWithFlags(&r->red, cudaStreamNonBlocking) != cudaSuccess) {
                cudaGetLastError();
                set_error("xpcs: cannot create the copy streams");
                return XPCS_ECUDA;
            }
        }
        while (r->ev.size() < n_events) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                set_error("xpcs: cannot create events");
                return XPCS_ECUDA;
            }
            r->ev.push_back(e);
        }
    }
    out = r;
    return XPCS_OK;
}
}  // namespace

void release_host_resources() {
    std::lock_guard<std::mutex> lk(g_host_mu);
    for (auto& kv : g_host_res) {
        for (cudaEvent_t e : kv.second.ev) cudaEventDestroy(e);
        if (kv.second.h2d) cudaStreamDestroy(kv.second.h2d);
        if (kv.second.d2h) cudaStreamDestroy(kv.second.d2h);
        if (kv.second.red) cudaStreamDestroy(kv.second.red);
    }
    g_host_res.clear();
}

extern "C" {

}  // extern "C"

// xpcs_step_host: per-atom HOST form factors with few distinct values (e.g. two species given as f in {1, 2}) are run
// as atom kinds with q-independent f_s, so that AUTO can place the light kinds on the integer engine (per-atom f
// would scale every phasor by max |f| and keep the whole call on the split-FP16 engine).  Returns the kind count
// (0: too many distinct values or none given).
static int host_kinds(const void* ff, int f64, int64_t N, std::vector<int32_t>& kind, std::vector<double>& val) {
    kind.clear();
    val.clear();
    if (!ff) return 0;
    kind.resize((size_t)N);
    for (int64_t j = 0; j < N; ++j) {
        const double f = f64 ? ((const double*)ff)[j] : (double)((const float*)ff)[j];
        size_t k = 0;
        while (k < val.size() && !(val[k] == f)) ++k;     // exact value match (NaN never matches: falls out below)
        if (k == val.size()) {
            if (val.size() == (size_t)kMaxKinds || !std::isfinite(f)) { kind.clear(); val.clear(); return 0; }
            val.push_back(f);
        }
        kind[(size_t)j] = (int32_t)k;
    }
    return (int)val.size();
}

extern "C" {

int xpcs_step_host(const xpcs_step* st, const xpcs_opts* opts) {
    clear_error();
    NEED(st, "step");
    Opts o;
    TRY(parse_opts(opts, o));
    NEED(st->positions, "positions");
    NEED(st->bin_of_q, "bin_of_q");
    POS(st->N, "N");
    POS(st->frames, "frames");
    POS(st->n_bins, "n_bins");
    POS(st->batches, "batches");
    if (!st->q_vectors) TRY(validate_grid(&st->grid));
    else {
        POS(st->n_q, "n_q");
        if (!(st->box_L > 0.0) || !std::isfinite(st->box_L)) {
            set_error("xpcs: box_L must be finite and > 0");
            return XPCS_EINVAL;
        }
    }
    if (st->n_lags < 0 || st->n_windows < 0 || (st->n_lags > 0 && !st->lags) || (st->n_windows > 0 && !st->windows)) {
        set_error("xpcs: lags/windows: negative count or NULL array");
        return XPCS_EINVAL;
    }
    int max_lag = 0;
    for (int64_t i = 0; i < st->n_lags; ++i) {
        if (st->lags[i] < 0 || st->lags[i] >= st->frames) {
            set_error("xpcs: lag %d out of range [0, %lld)", st->lags[i], (long long)st->frames);
            return XPCS_EINVAL;
        }
        max_lag = std::max(max_lag, (int)st->lags[i]);
    }
    for (int64_t i = 0; i < st->n_windows; ++i)
        if (st->windows[i] < 1 || st->windows[i] > st->frames) {
            set_error("xpcs: window %d out of range [1, %lld]", st->windows[i], (long long)st->frames);
            return XPCS_EINVAL;
        }
    // every limit of the calls below is checked here, before any stream is forked (an error after the fork would
    // leave the copy streams unjoined)
    const int64_t n_q = st->q_vectors ? st->n_q : st->grid.n_h * st->grid.n_k;
    if (max_lag > 640) {
        set_error("xpcs: lags > 640 frames are not supported by this build");
        return XPCS_EUNSUPPORTED;
    }
    if (st->n_bins > 12288 || n_q > (int64_t(1) << 31) - 1) {
        set_error("xpcs: ring plan limits: n_bins <= 12288, n_q < 2^31");
        return XPCS_EINVAL;
    }
    if (st->species) {
        Groups Gv;
        TRY(prep_groups(st->species, nullptr, st->N, Gv));      // validates kinds and indices (host only)
    }
    TRY(check_sticky());
    const int64_t N = st->N, T = st->frames, nb = st->n_bins;
    const int64_t n_bat = std::min<int64_t>(st->batches, T);
    const size_t pin = o.in_f64 ? 8 : 4, pout = o.out_f64 ? 8 : 4;
    // few distinct per-atom form factors -> atom kinds (see host_kinds)
    std::vector<int32_t> kinds;
    std::vector<double> kval, kabs;
    const int n_kinds = (!st->species && o.engine == XPCS_ENGINE_AUTO && !o.in_f64)
                            ? host_kinds(st->form_factors, o.in_f64, N, kinds, kval) : 0;
    xpcs_species ksp;
    std::memset(&ksp, 0, sizeof(ksp));
    const xpcs_species* species = st->species;
    void* d_fq = nullptr;
    if (n_kinds > 0) {
        d_fq = scratch(o.s, SS_H_FQ, pin * (size_t)n_kinds * (size_t)n_q);
        if (!d_fq) return XPCS_ENOMEM;
        ksp.n_species = n_kinds;
        ksp.species = kinds.data();
        ksp.f_q = d_fq;
        for (double v : kval) kabs.push_back(std::fabs(v));
        ksp.f_max = kabs.data();
        species = &ksp;
    }
    const size_t pos_bytes = pin * 3 * (size_t)N * (size_t)T, i_bytes = pout * (size_t)n_q * (size_t)T;
    const size_t g2_bytes = pout * (size_t)n_q * (size_t)st->n_lags;
    const size_t red_doubles = (size_t)(T + st->n_lags + st->n_windows) * (size_t)nb;
    char* d_pos = (char*)scratch(o.s, SS_H_POS, pos_bytes);
    char* d_ff = st->form_factors ? (char*)scratch(o.s, SS_H_FF, pin * (size_t)N) : nullptr;
    char* d_I = (char*)scratch(o.s, SS_H_I, i_bytes);
    char* d_g2 = st->n_lags ? (char*)scratch(o.s, SS_H_G2, g2_bytes) : nullptr;
    double* d_red = (double*)scratch(o.s, SS_H_RED, sizeof(double) * red_doubles);
    if (!d_pos || !d_I || !d_red || (st->form_factors && !d_ff) || (st->n_lags && !d_g2)) return XPCS_ENOMEM;
    double* d_sr = d_red;
    double* d_g2r = d_red + (size_t)T * nb;
    double* d_beta = d_g2r + (size_t)st->n_lags * nb;
    HostRes* hr = nullptr;
    TRY(host_resources(o.s, (size_t)(2 * n_bat + 6), hr));
    cudaEvent_t* ev = hr->ev.data();         // [0] fork, [1..n_bat] inputs in, [n_bat+1..2 n_bat] I out, then g2, joins, f
    const cudaEvent_t ev_fork = ev[0], ev_g2 = ev[2 * n_bat + 1], ev_d2h = ev[2 * n_bat + 2], ev_h2d = ev[2 * n_bat + 3],
                      ev_f = ev[2 * n_bat + 4], ev_red = ev[2 * n_bat + 5];
    TRY(cuda_fail(cudaEventRecord(ev_fork, o.s), "fork"));
    TRY(cuda_fail(cudaStreamWaitEvent(hr->h2d, ev_fork, 0), "fork"));
    TRY(cuda_fail(cudaStreamWaitEvent(hr->d2h, ev_fork, 0), "fork"));
    TRY(cuda_fail(cudaStreamWaitEvent(hr->red, ev_fork, 0), "fork"));
    // from here on every exit joins the three side streams back into o.s
    auto body = [&]() -> int {
        if (st->form_factors) {
            TRY(cuda_fail(cudaMemcpyAsync(d_ff, st->form_factors, pin * (size_t)N, cudaMemcpyHostToDevice, hr->h2d), "H2D f"));
            TRY(cuda_fail(cudaEventRecord(ev_f, hr->h2d), "event"));
        }
        if (n_kinds > 0)
            TRY(cuda_fail(launch_fill_rows(d_fq, o.in_f64 ? 1 : 0, n_kinds, n_q, kval.data(), o.s), "kind form factors"));
        const size_t frame_pos = pin * 3 * (size_t)N, frame_i = pout * (size_t)n_q;
        for (int64_t b = 0; b < n_bat; ++b) {
            const int64_t t0 = b * T / n_bat, t1 = (b + 1) * T / n_bat;
            TRY(cuda_fail(cudaMemcpyAsync(d_pos + t0 * frame_pos, (const char*)st->positions + t0 * frame_pos,
                                          (size_t)(t1 - t0) * frame_pos, cudaMemcpyHostToDevice, hr->h2d), "H2D positions"));
            TRY(cuda_fail(cudaEventRecord(ev[1 + b], hr->h2d), "event"));
        }
        xpcs_opts io{};
        io.in_dtype = o.in_f64 ? XPCS_F64 : XPCS_F32;
        io.out_dtype = o.out_f64 ? XPCS_F64 : XPCS_F32;
        io.stream = (void*)o.s;
        io.engine = o.engine;
        io.profile = o.profile ? 1 : 0;
        io.workspace = o.workspace;
        xpcs_qvolume vol;
        std::memset(&vol, 0, sizeof(vol));
        vol.plane = st->grid;
        vol.n_l = 1;
        const void* ff_int = species ? nullptr : d_ff;     // per-atom f inside the contraction (no kinds)
        for (int64_t b = 0; b < n_bat; ++b) {
            const int64_t t0 = b * T / n_bat, t1 = (b + 1) * T / n_bat;
            TRY(cuda_fail(cudaStreamWaitEvent(o.s, ev[1 + b], 0), "wait inputs"));
            if (b == 0 && st->form_factors) TRY(cuda_fail(cudaStreamWaitEvent(o.s, ev_f, 0), "wait f"));
            if (st->q_vectors)
                TRY(run_direct(d_pos + t0 * frame_pos, N, ff_int, species, st->q_vectors, n_q, t1 - t0, st->box_L,
                               d_I + t0 * frame_i, &io, 0));
            else
                TRY(run_volume(d_pos + t0 * frame_pos, N, ff_int, species, &vol, t1 - t0, d_I + t0 * frame_i, &io, 0));
            TRY(cuda_fail(cudaEventRecord(ev[1 + n_bat + b], o.s), "event"));
            if (st->I_out) {
                TRY(cuda_fail(cudaStreamWaitEvent(hr->d2h, ev[1 + n_bat + b], 0), "wait I"));
                TRY(cuda_fail(cudaMemcpyAsync((char*)st->I_out + t0 * frame_i, d_I + t0 * frame_i, (size_t)(t1 - t0) * frame_i,
                                              cudaMemcpyDeviceToHost, hr->d2h), "D2H I"));
            }
        }
        // reductions: g2 (+ its ring means) on the caller's stream, its (largest) result streaming back while the S
        // rings and XSVS run concurrently on the side stream
        xpcs_opts ro = io;
        ro.in_dtype = io.out_dtype;                  // the series fed to the reductions is I (out_dtype)
        xpcs_opts so = ro;
        so.stream = (void*)hr->red;
        Opts so_o;
        TRY(parse_opts(&so, so_o));
        TRY(cuda_fail(cudaStreamWaitEvent(hr->red, ev[2 * n_bat], 0), "fork reductions"));   // the last batch's I
        if (st->form_factors) TRY(cuda_fail(cudaStreamWaitEvent(hr->red, ev_f, 0), "wait f"));
        // S(q,t) normalisation sum f^2 from the caller's form factors, read at THEIR dtype (in_dtype)
        if (st->S_rings) TRY(structure_factor_shells(d_I, T, n_q, st->form_factors ? (const void*)d_ff : nullptr,
                                                     o.in_f64 ? 1 : 0, N, st->bin_of_q, st->n_bins, d_sr, so_o));
        if (st->n_windows && st->beta)
            TRY(xsvs_contrast(d_I, T, n_q, st->bin_of_q, st->n_bins, st->windows, st->n_windows, d_beta, &so));
        if (st->n_lags) {
            TRY(xpcs_g2(d_I, T, n_q, st->lags, st->n_lags, d_g2, &ro));
            TRY(cuda_fail(cudaEventRecord(ev_g2, o.s), "event"));
            if (st->g2_out) {
                TRY(cuda_fail(cudaStreamWaitEvent(hr->d2h, ev_g2, 0), "wait g2"));
                TRY(cuda_fail(cudaMemcpyAsync(st->g2_out, d_g2, g2_bytes, cudaMemcpyDeviceToHost, hr->d2h), "D2H g2"));
            }
            if (st->g2_rings) {
                xpcs_opts go = ro;
                go.in_dtype = io.out_dtype;
                TRY(xpcs_shell_mean(d_g2, st->n_lags, n_q, st->bin_of_q, st->n_bins, 1.0, d_g2r, &go));
            }
        }
        return XPCS_OK;
    };
    const int rc = body();
    // join: the reductions' side stream first (the small results are copied back after it on o.s), then the copies
    cudaEventRecord(ev_red, hr->red);
    cudaStreamWaitEvent(o.s, ev_red, 0);
    if (rc == XPCS_OK) {
        // small results back on the caller's stream (after the reductions)
        if (st->S_rings)
            TRY(cuda_fail(cudaMemcpyAsync(st->S_rings, d_sr, sizeof(double) * (size_t)T * nb, cudaMemcpyDeviceToHost, o.s), "D2H S"));
        if (st->n_lags && st->g2_rings)
            TRY(cuda_fail(cudaMemcpyAsync(st->g2_rings, d_g2r, sizeof(double) * (size_t)st->n_lags * nb,
                                          cudaMemcpyDeviceToHost, o.s), "D2H g2 rings"));
        if (st->n_windows && st->beta)
            TRY(cuda_fail(cudaMemcpyAsync(st->beta, d_beta, sizeof(double) * (size_t)st->n_windows * nb,
                                          cudaMemcpyDeviceToHost, o.s), "D2H beta"));
    }
    cudaEventRecord(ev_d2h, hr->d2h);
    cudaStreamWaitEvent(o.s, ev_d2h, 0);
    cudaEventRecord(ev_h2d, hr->h2d);
    cudaStreamWaitEvent(o.s, ev_h2d, 0);
    if (rc != XPCS_OK) return rc;
    return check_sticky();
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
