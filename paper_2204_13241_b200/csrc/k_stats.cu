// k_stats.cu -- speckle statistics on the stored intensity series:
//   K4 g2(q, tau)                        Eq.(14), PAPER.md:170-174 (literal estimator, R6)
//   K6 ring averages / S(q) by ring       PAPER.md:192; Eq.(12)-(13)
//   K5 XSVS contrast beta_{W,b}           Eq.(15), Eq.(17), averaging PAPER.md:429
// All sums are FP64 and in a fixed order (deterministic, no float atomics).
#include "common.cuh"
#include <vector>

namespace xpcs {

// =====================================================================================================
// K4: g2.  Block = 32 pixels (lanes) x 8 warps; warp w owns up to 16 lags.  The time series of the 32 pixels
// are staged through shared memory in chunks of GC frames plus a halo of max_lag frames (zero beyond T, so the
// products with t + tau >= T vanish and each lag sums exactly over t < T - tau).  fp32 x fp32 products are exact
// in FP64; the hot loop is one LDS + one DFMA per (pixel, lag, frame).
// =====================================================================================================
namespace { constexpr int G2_LPW = 16, G2_WARPS = 8, G2_LAGS_PER_BLOCK = G2_LPW * G2_WARPS, GC = 128; }

template <typename In, typename Out>
__global__ void __launch_bounds__(256)
k_g2(const In* __restrict__ I, int64_t T, int64_t n_q, const int32_t* __restrict__ lags, int64_t n_lags,
     int halo, Out* __restrict__ out) {
    extern __shared__ double S[];                    // [(GC + halo)][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t px = (int64_t)blockIdx.x * 32 + lane;
    const int64_t lbase = (int64_t)blockIdx.y * G2_LAGS_PER_BLOCK + warp * G2_LPW;
    int tau[G2_LPW];
#pragma unroll
    for (int l = 0; l < G2_LPW; ++l) tau[l] = (lbase + l < n_lags) ? lags[lbase + l] : 0;
    double acc[G2_LPW];
#pragma unroll
    for (int l = 0; l < G2_LPW; ++l) acc[l] = 0.0;
    double sum = 0.0;
    const int rows = GC + halo;
    for (int64_t t0 = 0; t0 < T; t0 += GC) {
        __syncthreads();
        for (int r = warp; r < rows; r += G2_WARPS) {
            const int64_t t = t0 + r;
            S[r * 32 + lane] = (t < T && px < n_q) ? (double)I[t * n_q + px] : 0.0;
        }
        __syncthreads();
        const int rmax = (int)min((int64_t)GC, T - t0);
        for (int r = 0; r < rmax; ++r) {
            const double a = S[r * 32 + lane];
            sum += a;
#pragma unroll
            for (int l = 0; l < G2_LPW; ++l) acc[l] = fma(a, S[(r + tau[l]) * 32 + lane], acc[l]);
        }
    }
    if (px >= n_q) return;
    const double mean = sum / (double)T;
    const double den = mean * mean;
#pragma unroll
    for (int l = 0; l < G2_LPW; ++l) {
        if (lbase + l >= n_lags) break;
        const double num = acc[l] / (double)(T - tau[l]);
        out[(lbase + l) * n_q + px] = (Out)(den > 0.0 ? num / den : __longlong_as_double(0x7ff8000000000000ll));
    }
}

cudaError_t launch_g2(const void* I, int in_f64, int64_t T, int64_t n_q, const int32_t* lags_dev,
                      int64_t n_lags, int max_lag, void* out, int out_f64, cudaStream_t s) {
    dim3 grid((unsigned)((n_q + 31) / 32), (unsigned)((n_lags + G2_LAGS_PER_BLOCK - 1) / G2_LAGS_PER_BLOCK));
    const size_t smem = sizeof(double) * 32 * (GC + max_lag);
    note_launch();
#define G2_CASE(IN, OUT)                                                                              \
    {                                                                                                 \
        auto kern = k_g2<IN, OUT>;                                                                    \
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        kern<<<grid, 256, smem, s>>>((const IN*)I, T, n_q, lags_dev, n_lags, max_lag, (OUT*)out);     \
    }
    if (in_f64) { if (out_f64) G2_CASE(double, double) else G2_CASE(double, float) }
    else { if (out_f64) G2_CASE(float, double) else G2_CASE(float, float) }
#undef G2_CASE
    return cudaGetLastError();
}

// =====================================================================================================
// Ring plan: pixels sorted by (ring, pixel index), stable and deterministic (one block per ring, block scan).
// =====================================================================================================
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int& total) {
    // 256-thread exclusive scan of v (Hillis-Steele in shared memory)
    const int tid = threadIdx.x;
    sh[tid] = v;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        const int x = tid >= off ? sh[tid - off] : 0;
        __syncthreads();
        sh[tid] += x;
        __syncthreads();
    }
    total = sh[255];
    const int incl = sh[tid];
    __syncthreads();
    return incl - v;
}

__global__ void __launch_bounds__(256) k_bin_count(const int32_t* __restrict__ bins, int64_t n_q, int32_t* counts) {
    __shared__ int sh[256];
    const int b = blockIdx.x;
    int c = 0;
    for (int64_t i = threadIdx.x; i < n_q; i += 256) c += (bins[i] == b);
    int total;
    block_excl_scan(c, sh, total);
    if (threadIdx.x == 0) counts[b] = total;
}

__global__ void k_bin_scan(const int32_t* counts, int32_t n_bins, int32_t* offsets, int32_t* warp_off) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int o = 0, w = 0;
    for (int b = 0; b < n_bins; ++b) {
        const int c = counts[b];          // counts may alias warp_off: read before overwriting
        offsets[b] = o;
        warp_off[b] = w;
        o += c;
        w += (c + 31) / 32;
    }
    offsets[n_bins] = o;
    warp_off[n_bins] = w;
}

__global__ void __launch_bounds__(256) k_bin_fill(const int32_t* __restrict__ bins, int64_t n_q,
                                                  const int32_t* __restrict__ offsets, int32_t* __restrict__ perm) {
    __shared__ int sh[256];
    const int b = blockIdx.x;
    int base = offsets[b];
    for (int64_t i0 = 0; i0 < n_q; i0 += 256) {
        const int64_t i = i0 + threadIdx.x;
        const int flag = (i < n_q) && (bins[i] == b);
        int total;
        const int pos = block_excl_scan(flag, sh, total);
        if (flag) perm[base + pos] = (int32_t)i;
        base += total;
    }
}

cudaError_t launch_binplan(const int32_t* bins, int64_t n_q, int32_t n_bins, BinPlan plan, cudaStream_t s) {
    int32_t* counts = plan.warp_off;   // temporary; k_bin_scan reads each count before overwriting it
    note_launch(3);
    k_bin_count<<<n_bins, 256, 0, s>>>(bins, n_q, counts);
    k_bin_scan<<<1, 1, 0, s>>>(counts, n_bins, plan.offsets, plan.warp_off);
    k_bin_fill<<<n_bins, 256, 0, s>>>(bins, n_q, plan.offsets, plan.perm);
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
// K5: XSVS.  One warp per 32 pixels of a ring segment (pixels from the ring plan).  Each lane streams its pixel's
// series once, keeps one running window sum per exposure W (registers), and when a window closes the warp
// reduces (I_W, I_W^2) with shuffles; lane 0 writes the warp's moments for slot (W, s).  A second kernel sums
// the warps of each ring in fixed order, forms beta_{W,b,s} (population variance / mean^2) and averages over s.
// =====================================================================================================
namespace { constexpr int XW = 16; }
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
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (gw >= total_warps || gw >= woff[n_bins]) return;
    // ring of this warp (binary search in the warp prefix)
    int lo = 0, hi = n_bins;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (woff[mid] <= gw) lo = mid; else hi = mid;
    }
    const int b = lo;
    const int64_t idx = off[b] + (gw - woff[b]) * 32 + lane;
    const bool valid = idx < off[b + 1];
    const int64_t px = valid ? perm[idx] : 0;
    double run[XW];
    int cnt[XW], sidx[XW];
#pragma unroll
    for (int w = 0; w < XW; ++w) { run[w] = 0.0; cnt[w] = w < ws.n ? ws.W[w] : 1; sidx[w] = 0; }
    for (int64_t t = 0; t < T; ++t) {
        const double v = valid ? (double)I[t * n_q + px] : 0.0;
#pragma unroll
        for (int w = 0; w < XW; ++w) {
            if (w >= ws.n) break;
            run[w] += v;
            if (--cnt[w] == 0) {
                if (sidx[w] < ws.S[w]) {
                    const double m1 = warp_sum_d(run[w]);
                    const double m2 = warp_sum_d(run[w] * run[w]);
                    if (lane == 0) mom[gw * ws.total_slots + ws.base[w] + sidx[w]] = make_double2(m1, m2);
                    ++sidx[w];
                }
                run[w] = 0.0;
                cnt[w] = ws.W[w];
            }
        }
    }
}

__global__ void __launch_bounds__(256)
k_xsvs_final(const double2* __restrict__ mom, const int32_t* __restrict__ off, const int32_t* __restrict__ woff,
             WinSet ws, int w_first, int32_t n_bins, double* __restrict__ beta_out) {
    __shared__ double sh[256];
    const int w = blockIdx.x, b = blockIdx.y;
    const int m0 = off[b + 1] - off[b];
    const int S = ws.S[w];
    double acc = 0.0;
    for (int s = threadIdx.x; s < S; s += 256) {
        double m1 = 0.0, m2 = 0.0;
        for (int g = woff[b]; g < woff[b + 1]; ++g) {
            const double2 v = mom[(int64_t)g * ws.total_slots + ws.base[w] + s];
            m1 += v.x;
            m2 += v.y;
        }
        const double mean = m1 / m0;
        acc += (m2 / m0 - mean * mean) / (mean * mean);           // Eq.(17), population variance
    }
    const double tot = block_sum_d(acc, sh);
    if (threadIdx.x == 0)
        beta_out[(int64_t)(w_first + w) * n_bins + b] = m0 > 0 ? tot / S : __longlong_as_double(0x7ff8000000000000ll);
}

cudaError_t launch_xsvs(const void* I, int in_f64, int64_t T, int64_t n_q, BinPlan plan, int32_t n_bins,
                        const int32_t* windows_host, int64_t n_windows, int64_t max_warps, double* warp_moments,
                        int32_t* /*dev_windows*/, double* beta_out, cudaStream_t s) {
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
        const unsigned blocks = (unsigned)((max_warps + 3) / 4);
        note_launch(2);
        if (blocks > 0) {
            if (in_f64) k_xsvs_warp<double><<<blocks, 128, 0, s>>>((const double*)I, T, n_q, plan.perm, plan.offsets, plan.warp_off, n_bins, max_warps, ws, (double2*)warp_moments);
            else k_xsvs_warp<float><<<blocks, 128, 0, s>>>((const float*)I, T, n_q, plan.perm, plan.offsets, plan.warp_off, n_bins, max_warps, ws, (double2*)warp_moments);
        }
        k_xsvs_final<<<dim3(ws.n, n_bins), 256, 0, s>>>((const double2*)warp_moments, plan.offsets, plan.warp_off, ws,
                                                        (int)w0, n_bins, beta_out);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace xpcs
