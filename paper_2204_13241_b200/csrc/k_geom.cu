// k_geom.cu -- q geometry on the device:
//   Ewald-sphere detector q (Eq.(1); Fig. 5 'spherical slice in q-space', PAPER.md:445;
//   DESIGN.md reading R4), integer-exact lattice rings and |q| rings (R8).
#include "common.cuh"

namespace xpcs {

template <typename O>
__global__ void __launch_bounds__(256)
k_ewald(double k, int64_t npx, int64_t npy, double pitch, O* __restrict__ q) {
    const int64_t total = npx * npy;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = p / npy, j = p % npy;
        const double psx = __dmul_rn(__dsub_rn((double)i, 0.5 * (double)(npx - 1)), pitch);
        const double psy = __dmul_rn(__dsub_rn((double)j, 0.5 * (double)(npy - 1)), pitch);
        double sx, cx, sy, cy;
        sincos(psx, &sx, &cx);
        sincos(psy, &sy, &cy);
        // k_f = k u, u = (sin psi_x cos psi_y, sin psi_y, cos psi_x cos psi_y);  k_i = k z;  q = k_f - k_i
        // explicit round-to-nearest ops (no FMA contraction): the same operation sequence as the definition
        q[3 * p + 0] = (O)__dmul_rn(k, __dmul_rn(sx, cy));
        q[3 * p + 1] = (O)__dmul_rn(k, sy);
        q[3 * p + 2] = (O)__dmul_rn(k, __dsub_rn(__dmul_rn(cx, cy), 1.0));
    }
}

__device__ __forceinline__ int64_t isqrt64(int64_t r2) {
    int64_t s = (int64_t)sqrt((double)r2);
    while (s * s > r2) --s;
    while ((s + 1) * (s + 1) <= r2) ++s;
    return s;
}

__global__ void __launch_bounds__(256)
k_lattice_bins(LatticeGeom g, int32_t n_bins, int32_t w, int32_t* __restrict__ out) {
    const int64_t total = g.n_h * g.n_k;
    const int64_t lim = (int64_t)n_bins * w;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = g.h0 + p / g.n_k, k = g.k0 + p % g.n_k;
        int64_t r2 = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int64_t m = (int64_t)g.m0[c] + h * g.ma[c] + k * g.mb[c];
            r2 += m * m;
        }
        int32_t b = -1;
        if (r2 > 0 && r2 < lim * lim) b = (int32_t)(isqrt64(r2) / w);
        out[p] = b;
    }
}

template <typename Q>
__global__ void __launch_bounds__(256)
k_radial_bins(const Q* __restrict__ q, int64_t n_q, double q_max, int32_t n_bins, int32_t* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_q; p += (int64_t)gridDim.x * blockDim.x) {
        const double x = (double)q[3 * p], y = (double)q[3 * p + 1], z = (double)q[3 * p + 2];
        const double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
        int32_t b = -1;
        if (r > 0.0 && r < q_max) b = (int32_t)floor(__dmul_rn(__ddiv_rn(r, q_max), (double)n_bins));
        out[p] = b;
    }
}

static dim3 ggrid(int64_t total) {
    int64_t b = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    return dim3((unsigned)(b < cap ? (b > 0 ? b : 1) : cap));
}

cudaError_t launch_ewald(double wavelength, int64_t npx, int64_t npy, double pitch, void* q, int out_f64,
                         cudaStream_t s) {
    const double k = 2.0 * 3.14159265358979323846 / wavelength;
    note_launch();
    if (out_f64) k_ewald<double><<<ggrid(npx * npy), 256, 0, s>>>(k, npx, npy, pitch, (double*)q);
    else k_ewald<float><<<ggrid(npx * npy), 256, 0, s>>>(k, npx, npy, pitch, (float*)q);
    return cudaGetLastError();
}

cudaError_t launch_lattice_bins(const LatticeGeom& g, int32_t n_bins, int32_t w, int32_t* out, cudaStream_t s) {
    note_launch();
    k_lattice_bins<<<ggrid(g.n_h * g.n_k), 256, 0, s>>>(g, n_bins, w, out);
    return cudaGetLastError();
}

cudaError_t launch_radial_bins(const void* q, int q_f64, int64_t n_q, double q_max, int32_t n_bins,
                               int32_t* out, cudaStream_t s) {
    note_launch();
    if (q_f64) k_radial_bins<double><<<ggrid(n_q), 256, 0, s>>>((const double*)q, n_q, q_max, n_bins, out);
    else k_radial_bins<float><<<ggrid(n_q), 256, 0, s>>>((const float*)q, n_q, q_max, n_bins, out);
    return cudaGetLastError();
}

}  // namespace xpcs
