// k_stats.cu -- speckle statistics on the stored intensity series:
//   K4 g2(q, tau)                        Eq.(14), PAPER.md:170-174 (literal estimator, R6)
//   K6 ring averages / S(q) by ring       PAPER.md:192; Eq.(12)-(13)
//   K5 XSVS contrast beta_{W,b}           Eq.(15), Eq.(17), averaging PAPER.md:429
// All sums are FP64 and in a fixed order (deterministic, no float atomics).
#include "common.cuh"
#include <algorithm>
#include <climits>
#include <vector>


namespace xpcs {

// =====================================================================================================
// K4: g2.  A warp owns 32 pixels (lanes) x LPW lags.  The pixels' time series are staged through shared memory (as
// FP64: products of two fp32 are exact in FP64) in chunks of GC frames plus a halo of max_lag frames (zero beyond T,
// so products with t + tau >= T vanish and each lag sums exactly over t < T - tau).  Consecutive lag groups
// (tau_l = tau_0 + l) use a register-blocked sliding window: per 16 frames 16 + 16 + LPW - 1 shared loads feed
// 16 LPW DFMA; other lag lists fall back to one shared load per DFMA.
// =====================================================================================================
namespace {
#ifndef XPCS_G2_GC
#define XPCS_G2_GC 128
#endif
constexpr int G2_WARPS = 8, GC = XPCS_G2_GC;   // frames per staged chunk (each chunk also stages the max-lag halo)
constexpr int G2_LPW = 8, G2_LAGS_PER_BLOCK = G2_LPW * G2_WARPS;   // the ISF kernel's tiling (below)
}

// 16 "a" rows r0 .. r0 + 15 (TAIL: only those < rlim) against the sliding window of LPW consecutive lags from t0l:
// per 16 rows 16 + 16 + LPW - 1 shared loads feed 16 LPW DFMA.  acc has room for the largest LPW (compile-time
// indices only, so it stays in registers whichever LPW a warp runs).
template <int LPW, bool TAIL, int CAP>
__device__ __forceinline__ void g2_rows16(const double* __restrict__ S, int lane, int r0, int rlim, int t0l,
                                          double (&acc)[CAP]) {
    static_assert(LPW <= CAP, "accumulator too small");
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = (!TAIL || r0 + i < rlim) ? S[(r0 + i) * 32 + lane] : 0.0;
#pragma unroll
    for (int j = 0; j < 16 + LPW - 1; ++j) {
        const double w = S[(r0 + t0l + j) * 32 + lane];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (j - i >= 0 && j - i < LPW) acc[j - i] = fma(a[i], w, acc[j - i]);
    }
}

template <int LPW, int CAP>
__device__ __forceinline__ void g2_rows(const double* __restrict__ S, int lane, int rlim, int t0l, double (&acc)[CAP]) {
    int r0 = 0;
    for (; r0 + 16 <= rlim; r0 += 16) g2_rows16<LPW, false>(S, lane, r0, rlim, t0l, acc);   // whole groups
    if (r0 < rlim) g2_rows16<LPW, true>(S, lane, r0, rlim, t0l, acc);                      // the tail
}

// A block owns 32 pixels (lanes) and up to G2_WARPS x G2_MAXLPW entries of the lag list (one block row for lists of
// <= 256 lags, so the series is staged once per pixel block); the block's lags are dealt to its warps in groups of
// 8, balanced (config 3's 200 lags: seven warps of 24 and one of 32), and each warp runs the register-blocked loop
// of the smallest width in {8, 16, 24, 32} that holds its lags.  The series mean is summed by warp 0.
constexpr int G2_MAXLPW = 32;
template <typename In, typename Out>
__global__ void __launch_bounds__(256, 2)
k_g2(const In* __restrict__ I, int64_t T, int64_t n_q, const int32_t* __restrict__ lags, int64_t n_lags,
     int halo, int lpb, Out* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char g2_smem[];
    double* S = reinterpret_cast<double*>(g2_smem);       // [(GC + halo + 16)][32]
    __shared__ double mean_sh[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t px = (int64_t)blockIdx.x * 32 + lane;
    const int64_t lblk = (int64_t)blockIdx.y * lpb;
    const int nlb = (int)max((int64_t)0, min((int64_t)lpb, n_lags - lblk));   // lags of this block
    const int ng = (nlb + 7) / 8;                                              // groups of 8
    const int g0 = warp * ng / G2_WARPS, g1 = (warp + 1) * ng / G2_WARPS;
    const int64_t lbase = lblk + 8 * g0;
    const int nl = min(8 * g1, nlb) - 8 * g0;                                 // this warp's lags
    const bool active = nl > 0;
    const int width = (nl + 7) / 8 * 8;                                       // 8, 16, 24 or 32
    bool consecutive = true;
    for (int l = 1; l < nl; ++l)
        if (lags[lbase + l] != lags[lbase] + l) consecutive = false;
    const int t0l = active ? lags[lbase] : 0;
    double acc[G2_MAXLPW];
#pragma unroll
    for (int l = 0; l < G2_MAXLPW; ++l) acc[l] = 0.0;
    double sum = 0.0;
    const int rows = GC + halo + 16;
    for (int64_t t0 = 0; t0 < T; t0 += GC) {
        __syncthreads();
        const int rv = (int)min((int64_t)rows, T - t0);                      // rows inside the series
#pragma unroll 4
        for (int r = warp; r < rv; r += G2_WARPS) S[r * 32 + lane] = px < n_q ? (double)I[(t0 + r) * n_q + px] : 0.0;
        for (int r = rv + ((warp - rv) % G2_WARPS + G2_WARPS) % G2_WARPS; r < rows; r += G2_WARPS) S[r * 32 + lane] = 0.0;
        __syncthreads();
        const int rmax = (int)min((int64_t)GC, T - t0);
        if (warp == 0)
            for (int r = 0; r < rmax; ++r) sum += S[r * 32 + lane];
        if (!active) continue;
        if (consecutive) {
            // rows t with t + tau_0 >= T only meet the zero halo: stop before them (the warp's smallest lag)
            const int rlim = (int)min((int64_t)rmax, max((int64_t)0, T - t0 - t0l));
            if (width == 8) g2_rows<8>(S, lane, rlim, t0l, acc);
            else if (width == 16) g2_rows<16>(S, lane, rlim, t0l, acc);
            else if (width == 24) g2_rows<24>(S, lane, rlim, t0l, acc);
            else g2_rows<32>(S, lane, rlim, t0l, acc);
        } else {
            for (int r = 0; r < rmax; ++r) {
                const double a = S[r * 32 + lane];
#pragma unroll
                for (int l = 0; l < G2_MAXLPW; ++l)
                    if (l < nl) acc[l] = fma(a, S[(r + lags[lbase + l]) * 32 + lane], acc[l]);
            }
        }
    }
    if (warp == 0) mean_sh[lane] = sum / (double)T;
    __syncthreads();
    if (px >= n_q || !active) return;
    const double mean = mean_sh[lane];
    const double den = mean * mean;
#pragma unroll
    for (int l = 0; l < G2_MAXLPW; ++l) {
        if (l >= nl) break;
        const double num = acc[l] / (double)(T - lags[lbase + l]);
        out[(lbase + l) * n_q + px] = (Out)(den > 0.0 ? num / den : __longlong_as_double(0x7ff8000000000000ll));
    }
}

cudaError_t launch_g2(const void* I, int in_f64, int64_t T, int64_t n_q, const int32_t* lags_dev,
                      int64_t n_lags, int max_lag, void* out, int out_f64, cudaStream_t s) {
    const size_t smem = sizeof(double) * 32 * (GC + max_lag + 16 + 16);   // the series is staged in FP64
    note_launch();
    // block rows of at most G2_WARPS x G2_MAXLPW lags, balanced in groups of 8
    const int64_t cap = (int64_t)G2_WARPS * G2_MAXLPW;
    const int64_t ny = (n_lags + cap - 1) / cap;
    const int lpb = (int)(((n_lags + ny - 1) / ny + 7) / 8 * 8);
    dim3 grid((unsigned)((n_q + 31) / 32), (unsigned)ny);
#define G2_CASE(IN, OUT)                                                                                        \
    {                                                                                                           \
        auto kern = k_g2<IN, OUT>;                                                                              \
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        kern<<<grid, 256, smem, s>>>((const IN*)I, T, n_q, lags_dev, n_lags, max_lag + 16, lpb, (OUT*)out);    \
    }
    if (in_f64) { if (out_f64) G2_CASE(double, double) else G2_CASE(double, float) }
    else { if (out_f64) G2_CASE(float, double) else G2_CASE(float, float) }
#undef G2_CASE
    return cudaGetLastError();
}


// =====================================================================================================
// Block-streamed g2 ("update in blocks of B frames"; Eq.(14)): a series longer
// than device memory arrives in blocks.  For a block of B frames starting at global frame t0, with the P =
// min(max_lag, t0) frames before it held in a device ring (frame g in slot g mod R), the pairs (t, t + tau) whose
// LATER frame lies in the block are added to acc[l][px]; the block's frames are added to sum[px]; then the block's
// last min(B, R) frames replace the ring's oldest.  Reversing time, D_u = C_{P+B-1-u} over C = [ring frames | block],
// the block's pairs are sum_{u < B} D_u D_{u+tau} with D = 0 past P + B (frames before the series): the k_g2 loop
// with the "a" rows limited to the block.  FP64 products and sums, as k_g2.
// =====================================================================================================
template <typename In, int LPW>
__global__ void __launch_bounds__(256)
k_g2_accum(const In* __restrict__ blk, int64_t B, const In* __restrict__ ring, int64_t R, int64_t ring0, int64_t P,
           int64_t n_q, const int32_t* __restrict__ lags, int64_t n_lags, int halo, int lpb, double* __restrict__ acc_out,
           double* __restrict__ sum_out) {
    extern __shared__ __align__(16) unsigned char g2a_smem[];
    double* S = reinterpret_cast<double*>(g2a_smem);      // [(GC + halo + 16)][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t px = (int64_t)blockIdx.x * 32 + lane;
    const int64_t lblk = (int64_t)blockIdx.y * lpb;
    const int64_t lbase = lblk + warp * LPW;
    const int64_t lend = min(n_lags, lblk + lpb);
    const bool active = lbase < lend;
    int tau[LPW];
    bool consecutive = true;
#pragma unroll
    for (int l = 0; l < LPW; ++l) {
        tau[l] = (lbase + l < lend) ? lags[lbase + l] : (active ? lags[lbase] + l : 0);
        if (tau[l] != tau[0] + l) consecutive = false;
    }
    double acc[LPW];
#pragma unroll
    for (int l = 0; l < LPW; ++l) acc[l] = 0.0;
    double sum = 0.0;
    const int64_t len = P + B;                             // combined series [ring frames | block]
    const int rows = GC + halo + 16;
    for (int64_t u0 = 0; u0 < B; u0 += GC) {
        __syncthreads();
        {
            // row u = u0 + r of the combined series (index i = len - 1 - u): block frame B - 1 - u for u < B, frame
            // t0 - P + i in ring slot (ring0 + i) mod R for B <= u < len (0 <= i < P <= R: one conditional
            // subtraction), zero past len.  Three simple loops (so each unrolls and keeps its loads in flight).
            const int rb = (int)max((int64_t)0, min((int64_t)rows, B - u0));
            const int rl = (int)max((int64_t)rb, min((int64_t)rows, len - u0));
            const int first = [&](int lo) { return lo + ((warp - lo) % G2_WARPS + G2_WARPS) % G2_WARPS; }(0);
            const In* src = blk + (B - 1 - u0) * n_q + px;
            for (int r = first; r < rb; r += G2_WARPS) S[r * 32 + lane] = px < n_q ? (double)src[-(int64_t)r * n_q] : 0.0;
            int r = rb + ((warp - rb) % G2_WARPS + G2_WARPS) % G2_WARPS;
            for (; r < rl; r += G2_WARPS) {
                const int64_t sl = ring0 + (len - 1 - u0 - r);
                S[r * 32 + lane] = px < n_q ? (double)ring[(sl >= R ? sl - R : sl) * n_q + px] : 0.0;
            }
            for (r = rl + ((warp - rl) % G2_WARPS + G2_WARPS) % G2_WARPS; r < rows; r += G2_WARPS) S[r * 32 + lane] = 0.0;
        }
        __syncthreads();
        const int rmax = (int)min((int64_t)GC, B - u0);     // "a" rows: the block's frames only
        if (warp == 0 && blockIdx.y == 0)
            for (int r = 0; r < rmax; ++r) sum += S[r * 32 + lane];
        if (!active) continue;
        if (consecutive) {
            const int t0l = tau[0];
            const int rlim = (int)min((int64_t)rmax, max((int64_t)0, len - u0 - t0l));   // later rows meet zeros only
            int r0 = 0;
            for (; r0 + 16 <= rlim; r0 += 16) g2_rows16<LPW, false>(S, lane, r0, rlim, t0l, acc);   // whole groups
            if (r0 < rlim) g2_rows16<LPW, true>(S, lane, r0, rlim, t0l, acc);                      // the tail
        } else {
            for (int r = 0; r < rmax; ++r) {
                const double a = S[r * 32 + lane];
#pragma unroll
                for (int l = 0; l < LPW; ++l) acc[l] = fma(a, S[(r + tau[l]) * 32 + lane], acc[l]);
            }
        }
    }
    if (px >= n_q) return;
    if (warp == 0 && blockIdx.y == 0) sum_out[px] += sum;
    if (!active) return;
#pragma unroll
    for (int l = 0; l < LPW; ++l) {
        if (lbase + l >= lend) break;
        acc_out[(lbase + l) * n_q + px] += acc[l];
    }
}

// the block's last min(B, R) frames into the ring (frame g -> slot g mod R), after k_g2_accum has read the ring
template <typename In>
__global__ void __launch_bounds__(256)
k_g2_ring_update(const In* __restrict__ blk, int64_t B, In* __restrict__ ring, int64_t R, int64_t t0, int64_t n_q) {
    const int64_t keep = min(B, R), first = B - keep;
    for (int64_t f = first + blockIdx.y; f < B; f += gridDim.y) {       // y: frames, x: pixels
        const int64_t slot = (t0 + f) % R;
        for (int64_t px = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; px < n_q; px += (int64_t)gridDim.x * blockDim.x)
            ring[slot * n_q + px] = blk[f * n_q + px];
    }
}

// g2 = (acc / (T - tau)) / (sum / T)^2 (NaN where the mean is 0), as k_g2's epilogue
template <typename Out>
__global__ void __launch_bounds__(256)
k_g2_finalize(const double* __restrict__ acc, const double* __restrict__ sum, int64_t T, int64_t n_q,
              const int32_t* __restrict__ lags, int64_t n_lags, Out* __restrict__ out) {
    for (int64_t l = blockIdx.y; l < n_lags; l += gridDim.y) {          // y: lags, x: pixels
        const double w = 1.0 / (double)(T - lags[l]);
        for (int64_t px = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; px < n_q; px += (int64_t)gridDim.x * blockDim.x) {
            const double mean = sum[px] / (double)T;
            const double den = mean * mean;
            const double num = acc[l * n_q + px] * w;
            out[l * n_q + px] = (Out)(den > 0.0 ? num / den : __longlong_as_double(0x7ff8000000000000ll));
        }
    }
}

static dim3 grid_rows(int64_t rows, int64_t n) {     // x: 256-wide pixel blocks, y: rows (strided)
    const int64_t bx = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16));
    const int64_t by = std::max<int64_t>(1, std::min<int64_t>({rows, (int64_t)sm_count() * 64 / bx + 1, (int64_t)65535}));
    return dim3((unsigned)bx, (unsigned)by);
}

cudaError_t launch_g2_accumulate(const void* blk, int in_f64, int64_t B, void* ring, int64_t R, int64_t t0,
                                 int64_t n_q, const int32_t* lags_dev, int64_t n_lags, int max_lag, double* acc,
                                 double* sum, cudaStream_t s) {
    const int64_t P = std::min<int64_t>(max_lag, t0);
    const int64_t ring0 = R > 0 ? (t0 - P) % R : 0;          // slot of the first ring frame used
    const size_t smem = sizeof(double) * 32 * (GC + max_lag + 16 + 16);
    const int lpw = n_lags >= 64 ? 16 : 8;
    const int64_t ny = (n_lags + (int64_t)G2_WARPS * lpw - 1) / ((int64_t)G2_WARPS * lpw);
    const int lpb = (int)(((n_lags + ny - 1) / ny + lpw - 1) / lpw * lpw);
    const dim3 grid((unsigned)((n_q + 31) / 32), (unsigned)ny);
    note_launch(R > 0 ? 2 : 1);
#define G2A_CASE(IN)                                                                                             \
    {                                                                                                            \
        auto kern = lpw == 16 ? k_g2_accum<IN, 16> : k_g2_accum<IN, 8>;                                          \
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        kern<<<grid, 256, smem, s>>>((const IN*)blk, B, (const IN*)ring, R, ring0, P, n_q, lags_dev, n_lags,     \
                                     max_lag + 16, lpb, acc, sum);                                               \
        if (R > 0)                                                                                               \
            k_g2_ring_update<IN><<<grid_rows(std::min(B, R), n_q), 256, 0, s>>>((const IN*)blk, B, (IN*)ring, R, t0, n_q); \
    }
    if (in_f64) G2A_CASE(double) else G2A_CASE(float)
#undef G2A_CASE
    return cudaGetLastError();
}

cudaError_t launch_g2_finalize(const double* acc, const double* sum, int64_t T, int64_t n_q, const int32_t* lags_dev,
                               int64_t n_lags, void* out, int out_f64, cudaStream_t s) {
    note_launch();
    const dim3 gr = grid_rows(n_lags, n_q);
    if (out_f64) k_g2_finalize<double><<<gr, 256, 0, s>>>(acc, sum, T, n_q, lags_dev, n_lags, (double*)out);
    else k_g2_finalize<float><<<gr, 256, 0, s>>>(acc, sum, T, n_q, lags_dev, n_lags, (float*)out);
    return cudaGetLastError();
}

// =====================================================================================================
// Intermediate scattering function, Eq.(22), PAPER.md:218-223:
//     F(q, tau) = (1 / (T - tau)) sum_{t < T - tau} p(q, t) p*(q, t + tau)  /  sum_j f_j^2
// from the complex amplitude series p [T][n_q] (re, im).  Same tiling as K4: a warp owns 32 pixels x 16 lags,
// the series are staged through shared memory with a zero halo; FP64 accumulation.
// =====================================================================================================
template <typename In>
__global__ void __launch_bounds__(256)
k_isf(const In* __restrict__ A, int64_t T, int64_t n_q, const int32_t* __restrict__ lags, int64_t n_lags, int halo,
      const double* __restrict__ norm, double norm_const, double* __restrict__ F) {
    extern __shared__ __align__(16) unsigned char isf_smem[];
    double2* S = reinterpret_cast<double2*>(isf_smem);   // [(GC + halo)][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t px = (int64_t)blockIdx.x * 32 + lane;
    const int64_t lbase = (int64_t)blockIdx.y * G2_LAGS_PER_BLOCK + warp * G2_LPW;
    int tau[G2_LPW];
#pragma unroll
    for (int l = 0; l < G2_LPW; ++l) tau[l] = (lbase + l < n_lags) ? lags[lbase + l] : 0;
    double ar[G2_LPW], ai[G2_LPW];
#pragma unroll
    for (int l = 0; l < G2_LPW; ++l) ar[l] = ai[l] = 0.0;
    const int rows = GC + halo;
    for (int64_t t0 = 0; t0 < T; t0 += GC) {
        __syncthreads();
        for (int r = warp; r < rows; r += G2_WARPS) {
            const int64_t t = t0 + r;
            double2 v = make_double2(0.0, 0.0);
            if (t < T && px < n_q) v = make_double2((double)A[2 * (t * n_q + px)], (double)A[2 * (t * n_q + px) + 1]);
            S[r * 32 + lane] = v;
        }
        __syncthreads();
        if (lbase >= n_lags) continue;
        const int rmax = (int)min((int64_t)GC, T - t0);
        for (int r = 0; r < rmax; ++r) {
            const double2 p = S[r * 32 + lane];
#pragma unroll
            for (int l = 0; l < G2_LPW; ++l) {
                const double2 q2 = S[(r + tau[l]) * 32 + lane];      // p(t) conj(p(t + tau))
                ar[l] = fma(p.x, q2.x, fma(p.y, q2.y, ar[l]));
                ai[l] = fma(p.y, q2.x, fma(-p.x, q2.y, ai[l]));
            }
        }
    }
    if (px >= n_q || lbase >= n_lags) return;
    const double nrm = norm ? norm[0] : norm_const;
#pragma unroll
    for (int l = 0; l < G2_LPW; ++l) {
        if (lbase + l >= n_lags) break;
        const double w = 1.0 / ((double)(T - tau[l]) * nrm);
        F[2 * ((lbase + l) * n_q + px)] = ar[l] * w;
        F[2 * ((lbase + l) * n_q + px) + 1] = ai[l] * w;
    }
}

cudaError_t launch_isf(const void* A, int in_f64, int64_t T, int64_t n_q, const int32_t* lags_dev, int64_t n_lags,
                       int max_lag, const double* norm, double norm_const, double* F_out, cudaStream_t s) {
    dim3 grid((unsigned)((n_q + 31) / 32), (unsigned)((n_lags + G2_LAGS_PER_BLOCK - 1) / G2_LAGS_PER_BLOCK));
    const size_t smem = sizeof(double2) * 32 * (GC + max_lag);
    note_launch();
    if (in_f64) {
        auto k = k_isf<double>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, 256, smem, s>>>((const double*)A, T, n_q, lags_dev, n_lags, max_lag, norm, norm_const, F_out);
    } else {
        auto k = k_isf<float>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, 256, smem, s>>>((const float*)A, T, n_q, lags_dev, n_lags, max_lag, norm, norm_const, F_out);
    }
    return cudaGetLastError();
}
// =====================================================================================================
// Ring plan: pixels sorted by (ring, pixel index) -- stable and deterministic.
//   k_bin_count : per 1024-pixel block, per-ring counts (shared-memory integer atomics: exact)
//   k_bin_scan  : per ring, exclusive scan over blocks (+ ring offsets and warp offsets)
//   k_bin_fill  : per block, warps in order; within a warp equal rings are ranked with __match_any_sync
// =====================================================================================================
constexpr int PLAN_BLOCK = 1024;

__global__ void __launch_bounds__(256) k_bin_count(const int32_t* __restrict__ bins, int64_t n_q, int32_t n_bins,
                                                   int32_t* __restrict__ bcounts) {
    extern __shared__ int cnt[];
    for (int b = threadIdx.x; b < n_bins; b += 256) cnt[b] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * PLAN_BLOCK;
    for (int k = threadIdx.x; k < PLAN_BLOCK; k += 256) {
        const int64_t i = base + k;
        if (i < n_q) {
            const int b = bins[i];
            if (b >= 0 && b < n_bins) atomicAdd(&cnt[b], 1);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < n_bins; b += 256) bcounts[(int64_t)blockIdx.x * n_bins + b] = cnt[b];
}

__global__ void __launch_bounds__(256) k_bin_scan(int32_t* __restrict__ bcounts, int nblk, int32_t n_bins,
                                                  int32_t* __restrict__ offsets, int32_t* __restrict__ warp_off,
                                                  int32_t* __restrict__ sw_off) {
    // one thread per ring: in-place exclusive scan of its counts over blocks -> per-block start (relative)
    __shared__ int tot[1024];
    for (int b0 = 0; b0 < n_bins; b0 += 1024) {
        for (int b = b0 + threadIdx.x; b < min(n_bins, b0 + 1024); b += 256) {
            int run = 0;
            for (int k = 0; k < nblk; ++k) {
                const int c = bcounts[(int64_t)k * n_bins + b];
                bcounts[(int64_t)k * n_bins + b] = run;
                run += c;
            }
            tot[b - b0] = run;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int o = b0 == 0 ? 0 : offsets[b0], w = b0 == 0 ? 0 : warp_off[b0], x = b0 == 0 ? 0 : sw_off[b0];
            for (int b = b0; b < min(n_bins, b0 + 1024); ++b) {
                offsets[b] = o;
                warp_off[b] = w;
                sw_off[b] = x;
                o += tot[b - b0];
                w += (tot[b - b0] + 31) / 32;
                x += (tot[b - b0] + 32 * XSVS_PX - 1) / (32 * XSVS_PX);
            }
            offsets[min(n_bins, b0 + 1024)] = o;
            warp_off[min(n_bins, b0 + 1024)] = w;
            sw_off[min(n_bins, b0 + 1024)] = x;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_bin_fill(const int32_t* __restrict__ bins, int64_t n_q, int32_t n_bins,
                                                  const int32_t* __restrict__ bstart,
                                                  const int32_t* __restrict__ offsets, int32_t* __restrict__ perm) {
    extern __shared__ int run[];
    for (int b = threadIdx.x; b < n_bins; b += 256) run[b] = offsets[b] + bstart[(int64_t)blockIdx.x * n_bins + b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * PLAN_BLOCK;
    for (int round = 0; round < PLAN_BLOCK / 256; ++round) {
        const int64_t i = base + round * 256 + threadIdx.x;
        const int b = (i < n_q) ? bins[i] : -1;
        const bool valid = b >= 0 && b < n_bins;
        const unsigned same = __match_any_sync(0xffffffffu, valid ? b : -1);
        const int rank = __popc(same & ((1u << lane) - 1u));
        const bool leader = rank == 0;
        for (int w = 0; w < 8; ++w) {          // warps in pixel order: stable
            __syncthreads();
            if (w == warp && valid) {
                perm[run[b] + rank] = (int32_t)i;
                __syncwarp(same);
                if (leader) run[b] += __popc(same);
            }
        }
    }
}

cudaError_t launch_binplan(const int32_t* bins, int64_t n_q, int32_t n_bins, BinPlan plan, cudaStream_t s) {
    const int nblk = (int)((n_q + PLAN_BLOCK - 1) / PLAN_BLOCK);
    const size_t sh = sizeof(int) * (size_t)n_bins;
    note_launch(3);
    k_bin_count<<<nblk, 256, sh, s>>>(bins, n_q, n_bins, plan.bcounts);
    k_bin_scan<<<1, 256, 0, s>>>(plan.bcounts, nblk, n_bins, plan.offsets, plan.warp_off, plan.sw_off);
    k_bin_fill<<<nblk, 256, sh, s>>>(bins, n_q, n_bins, plan.bcounts, plan.offsets, plan.perm);
    return cudaGetLastError();
}

// =====================================================================================================
// K6: ring means.  One block per (ring, row); fixed-order block tree.  Optional normalisation by sum_j f_j^2
// (Eq. 12-13), itself reduced on the device in fixed order.
// =====================================================================================================
__device__ __forceinline__ double block_sum_d(double v, double* sh) {
    const int tid = threadIdx.x;
    sh[tid] = v;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (tid < off) sh[tid] += sh[tid + off];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

template <typename F>
__global__ void __launch_bounds__(256) k_sum_f2(const F* __restrict__ f, int64_t N, double* out) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += 256) {
        const double v = (double)f[i];
        acc += v * v;
    }
    const double t = block_sum_d(acc, sh);
    if (threadIdx.x == 0) out[0] = t;
}

template <typename In>
__global__ void __launch_bounds__(256)
k_shell_mean(const In* __restrict__ v, int64_t n_q, const int32_t* __restrict__ perm, const int32_t* __restrict__ off,
             double scale, const double* __restrict__ norm, double* __restrict__ out, int32_t n_bins) {
    __shared__ double sh[256];
    const int b = blockIdx.x;
    const int64_t row = blockIdx.y;
    const In* V = v + row * n_q;
    double acc = 0.0, cnt = 0.0;
    for (int i = off[b] + threadIdx.x; i < off[b + 1]; i += 256) {
        const double x = (double)V[perm[i]];
        if (isfinite(x)) { acc += x; cnt += 1.0; }
    }
    const double s = block_sum_d(acc, sh);
    const double c = block_sum_d(cnt, sh);
    if (threadIdx.x == 0) {
        double r = c > 0.0 ? scale * (s / c) : __longlong_as_double(0x7ff8000000000000ll);
        if (norm) r = r / norm[0];
        out[row * n_bins + b] = r;
    }
}

// ring moments per row (count of finite values, their sum) in the fixed block order of k_shell_mean
template <typename In>
__global__ void __launch_bounds__(256)
k_shell_moments(const In* __restrict__ v, int64_t n_q, const int32_t* __restrict__ perm, const int32_t* __restrict__ off,
                double* __restrict__ out, int32_t n_bins) {
    __shared__ double sh[256];
    const int b = blockIdx.x;
    const int64_t row = blockIdx.y;
    const In* V = v + row * n_q;
    double acc = 0.0, cnt = 0.0;
    for (int i = off[b] + threadIdx.x; i < off[b + 1]; i += 256) {
        const double x = (double)V[perm[i]];
        if (isfinite(x)) { acc += x; cnt += 1.0; }
    }
    const double sm = block_sum_d(acc, sh);
    const double c = block_sum_d(cnt, sh);
    if (threadIdx.x == 0) {
        out[(row * n_bins + b) * 2] = c;
        out[(row * n_bins + b) * 2 + 1] = sm;
    }
}

__global__ void __launch_bounds__(256)
k_ring_means_from_moments(const double* __restrict__ mom, int64_t n, double scale, const double* __restrict__ norm,
                          double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double c = mom[2 * i], sm = mom[2 * i + 1];
        double r = c > 0.0 ? scale * (sm / c) : __longlong_as_double(0x7ff8000000000000ll);
        if (norm) r = r / norm[0];
        out[i] = r;
    }
}

cudaError_t launch_shell_moments(const void* v, int in_f64, int64_t rows, int64_t n_q, BinPlan plan, int32_t n_bins,
                                 double* out, cudaStream_t s) {
    dim3 grid((unsigned)n_bins, (unsigned)rows);
    note_launch();
    if (in_f64) k_shell_moments<double><<<grid, 256, 0, s>>>((const double*)v, n_q, plan.perm, plan.offsets, out, n_bins);
    else k_shell_moments<float><<<grid, 256, 0, s>>>((const float*)v, n_q, plan.perm, plan.offsets, out, n_bins);
    return cudaGetLastError();
}

cudaError_t launch_ring_means_from_moments(const double* mom, int64_t n, double scale, const double* norm, double* out,
                                           cudaStream_t s) {
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096));
    note_launch();
    k_ring_means_from_moments<<<(unsigned)blocks, 256, 0, s>>>(mom, n, scale, norm, out);
    return cudaGetLastError();
}

cudaError_t launch_sum_f2(const void* f, int f_f64, int64_t N, double* out, cudaStream_t s) {
    note_launch();
    if (f_f64) k_sum_f2<double><<<1, 256, 0, s>>>((const double*)f, N, out);
    else k_sum_f2<float><<<1, 256, 0, s>>>((const float*)f, N, out);
    return cudaGetLastError();
}

cudaError_t launch_shell_mean(const void* v, int in_f64, int64_t rows, int64_t n_q, BinPlan plan,
                              int32_t n_bins, double scale, const double* norm, double* out, cudaStream_t s) {
    dim3 grid((unsigned)n_bins, (unsigned)rows);
    note_launch();
    if (in_f64) k_shell_mean<double><<<grid, 256, 0, s>>>((const double*)v, n_q, plan.perm, plan.offsets, scale, norm, out, n_bins);
    else k_shell_mean<float><<<grid, 256, 0, s>>>((const float*)v, n_q, plan.perm, plan.offsets, scale, norm, out, n_bins);
    return cudaGetLastError();
}

// =====================================================================================================
// K5: XSVS.  Per warp: 32 pixels of a ring segment; each lane streams its pixel's series, keeps the running
// window sums (registers) and at each window close the warp's moments (sum I_W, sum I_W^2) for slot (W, s) are
// formed in a fixed order.  k_xsvs_warp2 (used by xsvs_contrast) reads the series once for all windows of the pass;
// k_xsvs_warp (one warp per window, shuffle reductions) serves the single-window speckle histogram and
// XPCS_XSVS_V1=1 builds.  A second kernel sums the warps of each ring in fixed order, forms beta_{W,b,s}
// (population variance / mean^2) and averages over s.
// =====================================================================================================
#ifndef XPCS_XWPW
#define XPCS_XWPW 1
#endif
#ifndef XPCS_XSVS_V1
#define XPCS_XSVS_V1 0       // 1: the previous one-warp-per-window kernel (timing comparisons)
#endif
namespace { constexpr int XW = 8, XWPW = XPCS_XWPW; }   // windows per pass / per warp
struct WinSet {
    int n;
    int W[XW], S[XW], base[XW];
    int total_slots;
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename In>
__global__ void __launch_bounds__(128)
k_xsvs_warp(const In* __restrict__ I, int64_t T, int64_t n_q, const int32_t* __restrict__ perm,
            const int32_t* __restrict__ off, const int32_t* __restrict__ woff, int32_t n_bins, int64_t total_warps,
            WinSet ws, double2* __restrict__ mom) {
    // one warp per (32 pixels of a ring segment, group of XWPW exposure windows blockIdx.y): a few windows share one
    // read of the series, the groups are independent warps (more parallelism than one warp walking all windows)
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int w0 = blockIdx.y * XWPW;
    if (gw >= total_warps || gw >= woff[n_bins] || w0 >= ws.n) return;
    const int nw = min(XWPW, ws.n - w0);
    int lo = 0, hi = n_bins;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (woff[mid] <= gw) lo = mid; else hi = mid;
    }
    const int b = lo;
    const int64_t idx = off[b] + (gw - woff[b]) * 32 + lane;
    const bool valid = idx < off[b + 1];
    const int64_t px = valid ? perm[idx] : 0;
    double run[XWPW];
    int cnt[XWPW], sidx[XWPW];
    int64_t Tuse = 0;                        // frames beyond the last complete window of every window are not read
#pragma unroll
    for (int k = 0; k < XWPW; ++k) {
        run[k] = 0.0;
        cnt[k] = k < nw ? ws.W[w0 + k] : 1;
        sidx[k] = 0;
        if (k < nw) Tuse = max(Tuse, (int64_t)ws.S[w0 + k] * ws.W[w0 + k]);
    }
    // frames are read 8 at a time (independent loads in flight: the series of one ring pixel is a strided walk
    // through I, and a single outstanding load per lane left this kernel latency-bound)
    constexpr int TB = 8;
    for (int64_t t0 = 0; t0 < Tuse; t0 += TB) {
        double vb[TB];
#pragma unroll
        for (int u = 0; u < TB; ++u) vb[u] = (valid && t0 + u < Tuse) ? (double)I[(t0 + u) * n_q + px] : 0.0;
#pragma unroll
        for (int u = 0; u < TB; ++u) {
            if (t0 + u >= Tuse) break;
#pragma unroll
            for (int k = 0; k < XWPW; ++k) {
                if (k >= nw) break;
                run[k] += vb[u];
                if (--cnt[k] == 0) {
                    if (sidx[k] < ws.S[w0 + k]) {
                        const double m1 = warp_sum_d(run[k]);
                        const double m2 = warp_sum_d(run[k] * run[k]);
                        if (lane == 0) mom[(int64_t)(ws.base[w0 + k] + sidx[k]) * total_warps + gw] = make_double2(m1, m2);
                        ++sidx[k];
                    }
                    run[k] = 0.0;
                    cnt[k] = ws.W[w0 + k];
                }
            }
        }
    }
}

// One warp per 32 pixels of a ring segment and ALL windows of the pass: the series is read once (the windows share
// it), gathered by cp.async into a warp-private double-buffered shared ring (FC frames per chunk, every load of a
// chunk in flight at once: the gather is latency-bound otherwise).  A window close writes the lane's (I_W, I_W^2)
// into a warp-private buffer [slot][lane] (rows padded to 33 double2: conflict-free both ways); every XB closes the
// warp sums the buffered slots across lanes (one lane per slot, 32 loads in lane order: a fixed order) and writes
// the warp's moments.
#ifndef XPCS_XSVS_XB
#define XPCS_XSVS_XB 16
#endif
#ifndef XPCS_XSVS_WIDE_MIN
#define XPCS_XSVS_WIDE_MIN 2   // warps per SM the wide grid must reach
#endif
#ifndef XPCS_XSVS_STAGES
#define XPCS_XSVS_STAGES 2   // staged chunks per warp (cp.async ring depth)
#endif
#ifndef XPCS_XSVS_WARPS
#define XPCS_XSVS_WARPS 4
#endif
#ifndef XPCS_XSVS_UNROLL
#define XPCS_XSVS_UNROLL 8   // 4-frame groups of a chunk unrolled
#endif
#ifndef XPCS_XSVS_FRAMES
#define XPCS_XSVS_FRAMES 16   // pixel-frames staged per lane per chunk
#endif
namespace { constexpr int XB = XPCS_XSVS_XB, XWARPS = XPCS_XSVS_WARPS, XFRAMES = XPCS_XSVS_FRAMES, XST = XPCS_XSVS_STAGES, XUN = XPCS_XSVS_UNROLL; }
// frames per staged chunk: 32 pixel-frames in flight per lane for XP pixels per lane
template <int XP> __host__ __device__ constexpr int xsvs_fc() { return XFRAMES / XP; }
static_assert(XB == 8 || XB == 16 || XB == 32, "the fold gives each buffered close 32 / XB lanes");
// per-frame close masks (bit k: window k of the pass closes after frame t) are built once per block in shared
// memory, so a frame costs one byte test instead of a scan over the windows; the window state stays in registers
constexpr int XMASK_MAX = 16384;   // frames a pass can cover with the shared-memory mask (longer series: k_xsvs_warp)
template <typename In, int XP>
__host__ __device__ constexpr size_t xsvs2_warp_smem() {
    return (size_t)XB * 33 * sizeof(double2) + (size_t)XB * sizeof(int) + XST * XFRAMES * 32 * sizeof(In);
}
// one byte per frame, rounded up to whole chunks (the loop reads the mask of every frame of its last chunk) and 16 B
__host__ __device__ constexpr size_t xsvs2_mask_bytes(int64_t tuse) {
    return (size_t)((tuse + 16 * XFRAMES - 1) / (16 * XFRAMES)) * (16 * XFRAMES);
}
template <typename In, int XP>
__host__ __device__ constexpr size_t xsvs2_smem(int64_t tuse) {
    return xsvs2_mask_bytes(tuse) + (size_t)XWARPS * xsvs2_warp_smem<In, XP>();
}
// One warp per 32 XP consecutive ring-ordered pixels of one ring (plan.sw_off), XP per lane (pixel j of lane l is
// entry 32 j + l), all windows of the pass.  Each lane keeps a running prefix sum P per pixel; window k's sum at
// its close is P - (P at its previous close).  At a close the lane adds its XP pixels' (I_W, I_W^2) in pixel order
// and writes one pair into a padded [slot][lane] shared buffer; every XB closes the warp folds the buffer (one lane
// per slot, lane order) into mom[slot][warp].  The series is gathered by cp.async into a double-buffered
// [XFC frames][XP][32] warp-private ring.
#ifndef XPCS_XSVS_CARVE
#define XPCS_XSVS_CARVE 0
#endif
#ifndef XPCS_XSVS_MINB
#define XPCS_XSVS_MINB 0     // > 0: minimum resident blocks per SM for the register allocator (experiments)
#endif
#if XPCS_XSVS_MINB > 0
#define XSVS2_BOUNDS __launch_bounds__(32 * XWARPS, XPCS_XSVS_MINB)
#else
#define XSVS2_BOUNDS __launch_bounds__(32 * XWARPS)
#endif
template <typename In, int XP>
__global__ void XSVS2_BOUNDS
k_xsvs_warp2(const In* __restrict__ I, int64_t T, int64_t n_q, const int32_t* __restrict__ perm,
             const int32_t* __restrict__ off, const int32_t* __restrict__ swoff, int32_t n_bins, int64_t total_warps,
             WinSet ws, double2* __restrict__ mom) {
    constexpr int XFC = xsvs_fc<XP>();
    static_assert(XFC % 4 == 0, "the close-mask loop reads four frames per word");
    extern __shared__ __align__(16) unsigned char xs_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = ws.n;
    int64_t Tuse = 0;
#pragma unroll
    for (int k = 0; k < XW; ++k)
        if (k < nw) Tuse = max(Tuse, (int64_t)ws.S[k] * ws.W[k]);
    uint32_t* cmask = reinterpret_cast<uint32_t*>(xs_smem);      // byte t: windows closing after frame t
    unsigned char* base = xs_smem + xsvs2_mask_bytes(Tuse) + (size_t)wib * xsvs2_warp_smem<In, XP>();
    double2 (*B)[33] = reinterpret_cast<double2 (*)[33]>(base);
    In* ser = reinterpret_cast<In*>(base + XB * 33 * sizeof(double2));          // [XST][XFC][XP][32]
    int* ids = reinterpret_cast<int*>(base + XB * 33 * sizeof(double2) + XST * XFC * XP * 32 * sizeof(In));
    // close masks: frame s W_k - 1 closes window k's snapshot s (windows aligned at t = 0, remainder dropped)
    for (int i = threadIdx.x; i < (int)(xsvs2_mask_bytes(Tuse) / 4); i += blockDim.x) cmask[i] = 0u;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < XW; ++k)   // static k: ws stays in the parameter bank (no local copy)
        if (k < nw)
            for (int sI = threadIdx.x; sI < ws.S[k]; sI += blockDim.x) {
                const int t = (sI + 1) * ws.W[k] - 1;
                atomicOr(&cmask[t >> 2], (1u << k) << (8 * (t & 3)));
            }
    __syncthreads();
    const int64_t gw = (int64_t)blockIdx.x * XWARPS + wib;
    if (gw >= total_warps || gw >= swoff[n_bins]) return;
    int lo = 0, hi = n_bins;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (swoff[mid] <= gw) lo = mid; else hi = mid;
    }
    const int b = lo;
    const int64_t idx0 = off[b] + (gw - swoff[b]) * (32 * XP) + lane;
    const In* src0[XP];
    uint32_t src_bytes[XP];
#pragma unroll
    for (int j = 0; j < XP; ++j) {
        const bool valid = idx0 + 32 * j < off[b + 1];
        src0[j] = I + (valid ? perm[idx0 + 32 * j] : 0);
        src_bytes[j] = valid ? (uint32_t)sizeof(In) : 0u;
    }
    double P[XP], lastP[XW][XP];
    int sidx[XW];
#pragma unroll
    for (int j = 0; j < XP; ++j) P[j] = 0.0;
#pragma unroll
    for (int k = 0; k < XW; ++k) {
        sidx[k] = 0;
#pragma unroll
        for (int j = 0; j < XP; ++j) lastP[k][j] = 0.0;
    }
    const int n_chunks = (int)((Tuse + XFC - 1) / XFC);
    auto prefetch = [&](int c) {
        if (c < n_chunks) {
            const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(ser + (size_t)(c % XST) * XFC * XP * 32 + lane);
            const int64_t t0 = (int64_t)c * XFC;
            const int un = (int)min((int64_t)XFC, Tuse - t0);
            if (un == XFC) {                      // whole chunk
#pragma unroll
                for (int j = 0; j < XP; ++j) {
                    const In* src = src0[j] + t0 * n_q;
#pragma unroll
                    for (int u = 0; u < XFC; ++u) {
                        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;"
                                     ::"r"(dst0 + (uint32_t)((u * XP + j) * 32 * sizeof(In))), "l"(src),
                                     "n"(sizeof(In)), "r"(src_bytes[j])
                                     : "memory");
                        src += n_q;
                    }
                }
            } else {                              // the last chunk: frames past Tuse zero-filled
#pragma unroll
                for (int j = 0; j < XP; ++j) {
                    const In* src = src0[j] + t0 * n_q;
                    for (int u = 0; u < XFC; ++u) {
                        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;"
                                     ::"r"(dst0 + (uint32_t)((u * XP + j) * 32 * sizeof(In))),
                                     "l"(u < un ? src : src0[j]), "n"(sizeof(In)), "r"(u < un ? src_bytes[j] : 0u)
                                     : "memory");
                        src += n_q;
                    }
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int nb = 0;                                   // buffered closes (warp-uniform)
    auto flush = [&]() {   // LPS lanes per buffered close, 32 / LPS lanes' pairs each, then a fixed-order tree
        constexpr int LPS = 32 / XB;
        __syncwarp();
        const int slot = lane / LPS, part = lane % LPS;
        double m1 = 0.0, m2 = 0.0;
        if (slot < nb) {
#pragma unroll
            for (int i = 0; i < 32 / LPS; ++i) {
                const double2 v = B[slot][part * (32 / LPS) + i];
                m1 += v.x;
                m2 += v.y;
            }
        }
#pragma unroll
        for (int o = 1; o < LPS; o <<= 1) {
            m1 += __shfl_xor_sync(0xffffffffu, m1, o);
            m2 += __shfl_xor_sync(0xffffffffu, m2, o);
        }
        if (part == 0 && slot < nb)
            mom[(int64_t)ids[slot] * total_warps + gw] = make_double2(m1, m2);   // slot-major: a ring's warps contiguous
        __syncwarp();
        nb = 0;
    };
#pragma unroll
    for (int c = 0; c < XST - 1; ++c) prefetch(c);
    for (int c = 0; c < n_chunks; ++c) {
        prefetch(c + XST - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(XST - 1) : "memory");
        __syncwarp();
        const In* sc = ser + (size_t)(c % XST) * XFC * XP * 32 + lane;
        const int t0 = c * XFC;
#pragma unroll (XUN)
        for (int u0 = 0; u0 < XFC; u0 += 4) {          // frames past Tuse are zero-filled and close nothing
            const uint32_t m4 = cmask[(t0 + u0) >> 2];     // one word per 4 frames, warp-uniform
#pragma unroll
            for (int i = 0; i < 4; ++i) {
#pragma unroll
                for (int j = 0; j < XP; ++j) P[j] += (double)sc[((u0 + i) * XP + j) * 32];
                uint32_t m = (m4 >> (8 * i)) & 0xFFu;
                if (m == 0u) continue;
#pragma unroll
                for (int k = 0; k < XW; ++k) {
                    if (m == 0u) break;                   // stop after the last closing window
                    if (m & 1u) {
                        double s1 = 0.0, s2 = 0.0;
#pragma unroll
                        for (int j = 0; j < XP; ++j) {
                            const double val = P[j] - lastP[k][j];
                            lastP[k][j] = P[j];
                            s1 += val;
                            s2 = fma(val, val, s2);
                        }
                        B[nb][lane] = make_double2(s1, s2);
                        if (lane == 0) ids[nb] = ws.base[k] + sidx[k];
                        ++sidx[k];
                        if (++nb == XB) flush();
                    }
                    m >>= 1;
                }
            }
        }
        __syncwarp();                             // chunk c's buffer is refilled by prefetch(c + XST)
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (nb > 0) flush();
}

// per (slot, ring) moments (m0 = ring pixel count, m1, m2) summed over the ring's warps in warp order, for
// xsvs_moments (a q-sharded detector adds these over ranks before forming beta)
__global__ void __launch_bounds__(256)
k_xsvs_final_moments(const double2* __restrict__ mom, const int32_t* __restrict__ off, const int32_t* __restrict__ woff,
                     WinSet ws, int64_t slot_first, int32_t n_bins, int64_t total_warps, double* __restrict__ out) {
    const int w = blockIdx.x, b = blockIdx.y;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double m0 = (double)(off[b + 1] - off[b]);
    const int64_t g0 = woff[b], g1 = woff[b + 1];
    const int sI = blockIdx.z * 8 + wid;                      // one warp per snapshot, fixed-order shuffle tree
    if (sI < ws.S[w]) {
        const double2* row = mom + (int64_t)(ws.base[w] + sI) * total_warps;
        double m1 = 0.0, m2 = 0.0;
#pragma unroll 4
        for (int64_t g = g0 + lane; g < g1; g += 32) {
            const double2 v = row[g];
            m1 += v.x;
            m2 += v.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            m1 += __shfl_xor_sync(0xffffffffu, m1, o);
            m2 += __shfl_xor_sync(0xffffffffu, m2, o);
        }
        if (lane == 0) {
            double* o = out + ((slot_first + ws.base[w] + sI) * n_bins + b) * 3;
            o[0] = m0;
            o[1] = m1;
            o[2] = m2;
        }
    }
}

// beta_{W,b} from summed moments (Eq. 17 per snapshot, population variance, then the mean over snapshots); block =
// (window, ring), threads over snapshots, a fixed-order tree (deterministic)
__global__ void __launch_bounds__(128)
k_xsvs_beta_from_moments(const double* __restrict__ mom, WinSet ws, int64_t slot_first, int w_first, int32_t n_bins,
                         double* __restrict__ beta_out) {
    __shared__ double sh[128];
    const int w = blockIdx.x, b = blockIdx.y, S = ws.S[w];
    double acc = 0.0;
    int bad = S <= 0;
    for (int sI = threadIdx.x; sI < S; sI += 128) {
        const double* o = mom + ((slot_first + ws.base[w] + sI) * n_bins + b) * 3;
        if (!(o[0] > 0.0)) { bad = 1; continue; }
        const double mean = o[1] / o[0];
        acc += (o[2] / o[0] - mean * mean) / (mean * mean);
    }
    sh[threadIdx.x] = acc;
    bad = __syncthreads_or(bad);
    for (int h = 64; h > 0; h >>= 1) {
        if (threadIdx.x < h) sh[threadIdx.x] += sh[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        beta_out[(int64_t)(w_first + w) * n_bins + b] = bad ? __longlong_as_double(0x7ff8000000000000ll) : sh[0] / S;
}

cudaError_t launch_xsvs_beta_from_moments(const double* mom, int64_t T, const int32_t* windows_host, int64_t n_windows,
                                          int32_t n_bins, double* beta_out, cudaStream_t s) {
    int64_t slot_first = 0;
    for (int64_t w0 = 0; w0 < n_windows; w0 += XW) {
        WinSet ws{};
        ws.n = (int)min((int64_t)XW, n_windows - w0);
        int slots = 0;
        for (int i = 0; i < ws.n; ++i) {
            ws.W[i] = windows_host[w0 + i];
            ws.S[i] = (int)(T / ws.W[i]);
            ws.base[i] = slots;
            slots += ws.S[i];
        }
        ws.total_slots = slots;
        note_launch();
        k_xsvs_beta_from_moments<<<dim3(ws.n, n_bins), 128, 0, s>>>(mom, ws, slot_first, (int)w0, n_bins, beta_out);
        slot_first += slots;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_xsvs(const void* I, int in_f64, int64_t T, int64_t n_q, BinPlan plan, int32_t n_bins,
                        const int32_t* windows_host, int64_t n_windows, int64_t max_warps, double* warp_moments,
                        double* mom_out, cudaStream_t s) {
    int64_t slot_first = 0;
    for (int64_t w0 = 0; w0 < n_windows; w0 += XW) {
        WinSet ws{};
        ws.n = (int)min((int64_t)XW, n_windows - w0);
        int slots = 0;
        for (int i = 0; i < ws.n; ++i) {
            ws.W[i] = windows_host[w0 + i];
            ws.S[i] = (int)(T / ws.W[i]);
            ws.base[i] = slots;
            slots += ws.S[i];
        }
        ws.total_slots = slots;
        note_launch(2);
        int64_t tuse = 0;
        for (int i = 0; i < ws.n; ++i) tuse = std::max<int64_t>(tuse, (int64_t)ws.S[i] * ws.W[i]);
        const int32_t* woff = plan.warp_off;
        if (tuse > XMASK_MAX) {   // very long series: one warp per window (no shared-memory close mask)
            const dim3 gr((unsigned)((max_warps + 3) / 4), (unsigned)((ws.n + XWPW - 1) / XWPW));
            if (max_warps > 0) {
                if (in_f64) k_xsvs_warp<double><<<gr, 128, 0, s>>>((const double*)I, T, n_q, plan.perm, plan.offsets, plan.warp_off, n_bins, max_warps, ws, (double2*)warp_moments);
                else k_xsvs_warp<float><<<gr, 128, 0, s>>>((const float*)I, T, n_q, plan.perm, plan.offsets, plan.warp_off, n_bins, max_warps, ws, (double2*)warp_moments);
            }
        } else {
            // XSVS_PX pixels per lane when that still fills the GPU, else one (plan.warp_off)
            const int64_t max_sw = std::min<int64_t>(max_warps, (n_q + 32 * XSVS_PX - 1) / (32 * XSVS_PX) + n_bins);
            const bool wide = XSVS_PX > 1 && max_sw >= (int64_t)sm_count() * XPCS_XSVS_WIDE_MIN;
            const int64_t n_w = wide ? max_sw : max_warps;
            const unsigned blocks = (unsigned)((n_w + XWARPS - 1) / XWARPS);
            woff = wide ? plan.sw_off : plan.warp_off;
            auto go = [&](auto kern, size_t sm, const auto* src) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
#if XPCS_XSVS_CARVE
                cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
#endif
                kern<<<blocks, 32 * XWARPS, sm, s>>>(src, T, n_q, plan.perm, plan.offsets, woff, n_bins, max_warps, ws,
                                                     (double2*)warp_moments);
            };
            if (blocks > 0) {
                if (in_f64) {
                    if (wide) go(k_xsvs_warp2<double, XSVS_PX>, xsvs2_smem<double, XSVS_PX>(tuse), (const double*)I);
                    else go(k_xsvs_warp2<double, 1>, xsvs2_smem<double, 1>(tuse), (const double*)I);
                } else {
                    if (wide) go(k_xsvs_warp2<float, XSVS_PX>, xsvs2_smem<float, XSVS_PX>(tuse), (const float*)I);
                    else go(k_xsvs_warp2<float, 1>, xsvs2_smem<float, 1>(tuse), (const float*)I);
                }
            }
        }
        int max_s = 0;
        for (int i = 0; i < ws.n; ++i) max_s = std::max(max_s, ws.S[i]);
        if (max_s > 0)
            k_xsvs_final_moments<<<dim3(ws.n, n_bins, (max_s + 7) / 8), 256, 0, s>>>(
                (const double2*)warp_moments, plan.offsets, woff, ws, slot_first, n_bins, max_warps, mom_out);
        slot_first += ws.total_slots;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// =====================================================================================================
// Speckle statistics (Eq.(37)-(38) PAPER.md:560-569): histogram of kappa = I_M / <I_M>_ring over
// the pixels of each ring and all snapshots, I_M the sum of M consecutive frames (incoherent superposition).
// Pass 1 = the XSVS warp moments with the single window M (ring sums per snapshot); pass 2 forms the ring means in
// fixed order; pass 3 streams the series again, bins kappa in FP64 and counts with warp-aggregated integer
// atomics (the counts are exact and order-independent).
// =====================================================================================================
__global__ void __launch_bounds__(256)
k_ring_snapshot_mean(const double2* __restrict__ mom, const int32_t* __restrict__ off, const int32_t* __restrict__ woff,
                     int S, int64_t total_warps, int32_t n_bins, double* __restrict__ mean) {
    const int b = blockIdx.x;
    const int m0 = off[b + 1] - off[b];
    for (int s = threadIdx.x; s < S; s += 256) {
        double m1 = 0.0;
        for (int g = woff[b]; g < woff[b + 1]; ++g) m1 += mom[(int64_t)s * total_warps + g].x;   // slot-major
        mean[(int64_t)s * n_bins + b] = m0 > 0 ? m1 / m0 : 0.0;
    }
}

template <typename In>
__global__ void __launch_bounds__(128)
k_speckle_hist(const In* __restrict__ I, int64_t T, int64_t n_q, const int32_t* __restrict__ perm,
               const int32_t* __restrict__ off, const int32_t* __restrict__ woff, int32_t n_bins, int64_t total_warps,
               int M, int S, const double* __restrict__ mean, int n_hist, double kappa_max,
               unsigned long long* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (gw >= total_warps || gw >= woff[n_bins]) return;
    int lo = 0, hi = n_bins;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (woff[mid] <= gw) lo = mid; else hi = mid;
    }
    const int b = lo;
    const int64_t idx = off[b] + (gw - woff[b]) * 32 + lane;
    const bool valid = idx < off[b + 1];
    const int64_t px = valid ? perm[idx] : 0;
    const double nh = (double)n_hist;
    for (int s = 0; s < S; ++s) {
        double run = 0.0;
        for (int t = 0; t < M; ++t) run += valid ? (double)I[((int64_t)s * M + t) * n_q + px] : 0.0;
        const double mu = mean[(int64_t)s * n_bins + b];
        int h = -1;
        if (valid && mu > 0.0) {
            const double u = (run / mu) * nh / kappa_max;      // same operation order as the oracle
            if (u < nh) h = (int)floor(u);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, h);
        if (h >= 0 && lane == __ffs(peers) - 1)
            atomicAdd(&counts[(int64_t)b * n_hist + h], (unsigned long long)__popc(peers));
    }
}

cudaError_t launch_speckle_hist(const void* I, int in_f64, int64_t T, int64_t n_q, BinPlan plan, int32_t n_bins,
                                int32_t M, int64_t max_warps, double* warp_moments, double* means, int32_t n_hist,
                                double kappa_max, int64_t* counts, cudaStream_t s) {
    const int S = (int)(T / M);
    WinSet ws{};
    ws.n = 1;
    ws.W[0] = M;
    ws.S[0] = S;
    ws.base[0] = 0;
    ws.total_slots = S;
    const unsigned blocks = (unsigned)((max_warps + 3) / 4);
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)n_bins * (size_t)n_hist, s);
    if (e != cudaSuccess) return e;
    if (blocks == 0) return cudaSuccess;
    note_launch(3);
    if (in_f64) k_xsvs_warp<double><<<blocks, 128, 0, s>>>((const double*)I, T, n_q, plan.perm, plan.offsets, plan.warp_off, n_bins, max_warps, ws, (double2*)warp_moments);
    else k_xsvs_warp<float><<<blocks, 128, 0, s>>>((const float*)I, T, n_q, plan.perm, plan.offsets, plan.warp_off, n_bins, max_warps, ws, (double2*)warp_moments);
    k_ring_snapshot_mean<<<n_bins, 256, 0, s>>>((const double2*)warp_moments, plan.offsets, plan.warp_off, S, max_warps, n_bins, means);
    if (in_f64) k_speckle_hist<double><<<blocks, 128, 0, s>>>((const double*)I, T, n_q, plan.perm, plan.offsets, plan.warp_off, n_bins, max_warps, M, S, means, n_hist, kappa_max, (unsigned long long*)counts);
    else k_speckle_hist<float><<<blocks, 128, 0, s>>>((const float*)I, T, n_q, plan.perm, plan.offsets, plan.warp_off, n_bins, max_warps, M, S, means, n_hist, kappa_max, (unsigned long long*)counts);
    return cudaGetLastError();
}

}  // namespace xpcs
