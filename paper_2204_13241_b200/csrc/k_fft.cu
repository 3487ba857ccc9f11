// k_fft.cu -- Algorithm 2, the FFT-based method (a cross-check / second
// workload beside the direct method, which stays the product's hot path).
//
//   step 1-2  rho^eta on an n^3 grid: each atom's normalised Gaussian (Eq. 30) on the k x k x k grid points nearest
//             to it (indices wrapped periodically).  One warp per (atom, frame); the Gaussian is separable, so the
//             warp forms 3 x k one-dimensional factors and deposits their k^3 products with FP64 red.global.add
//             (the deposit order varies, the sums agree to FP64 rounding).
//   step 3    p^eta = FFT(rho^eta): cuFFT D2Z (library call), batched over frames; sign e^{-i q.r} as Eq.(31).
//   step 4    f^eta(q) = FFT of the truncated Gaussian centred at the origin.  That kernel is separable and (k odd)
//             symmetric, so its 3-D DFT is the product of three real 1-D sums
//                 G(h) = c1 [1 + 2 sum_{j=1}^{(k-1)/2} exp(-(j dx)^2 / 2 eta^2) cos(2 pi h j / n)]
//             evaluated exactly per q in the epilogue (the same numbers as a 3-D FFT of the sampled kernel).
//   step 5    I = f(q)^2 |p^eta|^2 / f^eta^2 (Eq. 35) on the requested (h, k, l) block, from the half spectrum
//             (Hermitian symmetry for l < 0).
#include "common.cuh"

#include <cufft.h>

namespace xpcs {

template <typename P>
__global__ void __launch_bounds__(256) k_spread(const P* __restrict__ pos, int64_t N, int64_t frames, double L,
                                                int n, double eta, int k, double* __restrict__ rho) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const double dx = L / n;
    const double c1 = 1.0 / (2.5066282746310005024 * eta);      // (sqrt(2 pi) eta)^-1 per axis
    const double inv2e2 = 1.0 / (2.0 * eta * eta);
    const int64_t n3 = (int64_t)n * n * n;
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < N * frames; w += warps) {
        const int64_t t = w / N;
        const P* r = pos + 3 * w;
        int n0[3];
        double x[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            x[a] = box_fraction((double)r[a], L) * L;                 // wrapped coordinate in [0, L)
            n0[a] = (int)floor(x[a] / dx - 0.5 * k) + 1;              // the k grid indices nearest to x / dx
        }
        // 1-D factors: lanes 0..k-1 hold axis-x, y, z weights of grid offset i = lane
        double wx = 0.0, wy = 0.0, wz = 0.0;
        if (lane < k) {
            const double ex = (n0[0] + lane) * dx - x[0], ey = (n0[1] + lane) * dx - x[1], ez = (n0[2] + lane) * dx - x[2];
            wx = c1 * exp(-ex * ex * inv2e2);
            wy = c1 * exp(-ey * ey * inv2e2);
            wz = c1 * exp(-ez * ez * inv2e2);
        }
        double* R = rho + t * n3;
        const int kk = k * k, k3 = kk * k;
        for (int p0 = 0; p0 < k3; p0 += 32) {      // whole-warp iterations: every lane takes part in the shuffles
            const int p = min(p0 + lane, k3 - 1);
            const int i = p / kk, j = (p / k) % k, l = p % k;
            const double v = __shfl_sync(0xffffffffu, wx, i) * __shfl_sync(0xffffffffu, wy, j) *
                             __shfl_sync(0xffffffffu, wz, l);
            if (p0 + lane >= k3) continue;
            int gx = (n0[0] + i) % n, gy = (n0[1] + j) % n, gz = (n0[2] + l) % n;
            gx += gx < 0 ? n : 0;
            gy += gy < 0 ? n : 0;
            gz += gz < 0 ? n : 0;
            atomicAdd(R + ((int64_t)gx * n + gy) * n + gz, v);
        }
    }
}

template <typename Fq, typename O>
__global__ void __launch_bounds__(256) k_fft_epilogue(const double2* __restrict__ spec, int n, int64_t frames,
                                                      int64_t h0, int64_t n_h, int64_t k0, int64_t n_k, int64_t l0,
                                                      int64_t n_l, double L, double eta, int kc,
                                                      const Fq* __restrict__ fq, O* __restrict__ out) {
    const int64_t blk = n_l * n_h * n_k;
    const int64_t total = frames * blk;
    const int64_t nz = n / 2 + 1;
    const int64_t spec_frame = (int64_t)n * n * nz;
    const double dx = L / n, inv2e2 = 1.0 / (2.0 * eta * eta), c1 = 1.0 / (2.5066282746310005024 * eta);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / blk, r = i - t * blk;
        const int64_t il = r / (n_h * n_k), r2 = r - il * (n_h * n_k), ih = r2 / n_k, ik = r2 - ih * n_k;
        const int64_t f3[3] = {h0 + ih, k0 + ik, l0 + il};
        // f^eta = G(h) G(k) G(l)
        double Gp = 1.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            double g = 1.0;
            for (int j = 1; j <= kc / 2; ++j) {
                int64_t m = (f3[a] * j) % n;
                if (m < 0) m += n;
                g += 2.0 * exp(-(j * dx) * (j * dx) * inv2e2) * cospi(2.0 * (double)m / (double)n);
            }
            Gp *= c1 * g;
        }
        int64_t ix = f3[0] % n, iy = f3[1] % n, iz = f3[2] % n;
        ix += ix < 0 ? n : 0;
        iy += iy < 0 ? n : 0;
        iz += iz < 0 ? n : 0;
        double2 X;
        if (iz < nz) {
            X = spec[t * spec_frame + (ix * n + iy) * nz + iz];
        } else {   // Hermitian symmetry of the real-input transform: X(h,k,l) = conj X(-h,-k,-l)
            const int64_t jx = (n - ix) % n, jy = (n - iy) % n, jz = (n - iz) % n;
            X = spec[t * spec_frame + (jx * n + jy) * nz + jz];
            X.y = -X.y;
        }
        double I = (X.x * X.x + X.y * X.y) / (Gp * Gp);
        if (fq) {
            const double f = (double)fq[r];
            I *= f * f;
        }
        out[i] = (O)I;
    }
}

namespace {
struct FftPlan {
    cufftHandle plan = 0;
    int n = 0, batch = 0;
    cudaStream_t stream = nullptr;
    bool ok = false;
};
FftPlan g_plans[4];   // a full batch and the tail batch of the same call both stay cached
int g_next = 0;

cufftHandle* get_plan(int n, int batch) {
    for (auto& p : g_plans)
        if (p.ok && p.n == n && p.batch == batch) return &p.plan;
    FftPlan& p = g_plans[g_next];
    g_next = (g_next + 1) % 4;
    if (p.ok) cufftDestroy(p.plan);
    p = FftPlan{};
    int dims[3] = {n, n, n};
    if (cufftPlanMany(&p.plan, 3, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, batch) != CUFFT_SUCCESS) return nullptr;
    p.n = n;
    p.batch = batch;
    p.ok = true;
    return &p.plan;
}
}  // namespace

cudaError_t fft_release_plan() {
    for (auto& p : g_plans) {
        if (p.ok) cufftDestroy(p.plan);
        p = FftPlan{};
    }
    return cudaSuccess;
}

int launch_fft_intensity(const void* pos, int pos_f64, int64_t N, int64_t frames, double L, int n, double eta, int k,
                         double* rho, double2* spec, int64_t h0, int64_t n_h, int64_t k0, int64_t n_k, int64_t l0,
                         int64_t n_l, const void* fq, int fq_f64, void* out, int out_f64, cudaStream_t s,
                         const char** what) {
    const int64_t n3 = (int64_t)n * n * n;
    *what = "memset";
    if (cudaMemsetAsync(rho, 0, sizeof(double) * (size_t)(n3 * frames), s) != cudaSuccess) return 2;
    {
        const int64_t warps = N * frames;
        int64_t blocks = (warps + 7) / 8;
        blocks = blocks < (int64_t)sm_count() * 32 ? blocks : (int64_t)sm_count() * 32;
        note_launch();
        if (pos_f64) k_spread<double><<<(unsigned)blocks, 256, 0, s>>>((const double*)pos, N, frames, L, n, eta, k, rho);
        else k_spread<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)pos, N, frames, L, n, eta, k, rho);
        *what = "spread";
        if (cudaGetLastError() != cudaSuccess) return 2;
    }
    *what = "cufftPlanMany";
    cufftHandle* plan = get_plan(n, (int)frames);
    if (!plan) return 3;
    *what = "cufftExecD2Z";
    if (cufftSetStream(*plan, s) != CUFFT_SUCCESS) return 3;
    if (cufftExecD2Z(*plan, rho, (cufftDoubleComplex*)spec) != CUFFT_SUCCESS) return 3;
    {
        const int64_t total = frames * n_l * n_h * n_k;
        int64_t blocks = (total + 255) / 256;
        blocks = blocks < (int64_t)sm_count() * 16 ? blocks : (int64_t)sm_count() * 16;
        note_launch();
#define XPCS_FE(F, O) k_fft_epilogue<F, O><<<(unsigned)blocks, 256, 0, s>>>(spec, n, frames, h0, n_h, k0, n_k, l0, n_l, L, eta, k, (const F*)fq, (O*)out)
        if (fq_f64) { if (out_f64) XPCS_FE(double, double); else XPCS_FE(double, float); }
        else { if (out_f64) XPCS_FE(float, double); else XPCS_FE(float, float); }
#undef XPCS_FE
        *what = "epilogue";
        if (cudaGetLastError() != cudaSuccess) return 2;
    }
    return 0;
}

}  // namespace xpcs
