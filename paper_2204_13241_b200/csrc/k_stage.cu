// k_stage.cu -- K0 frame staging.
//
// Positions arrive as the caller's AoS [T][N][3] (fp32 or fp64).  Each atom is wrapped into the periodic box
// (on the reciprocal lattice the image choice is irrelevant) and converted ONCE per frame into
// exact fixed-point phase turns, so that the hot kernels never multiply a rounded q by a large coordinate
// (R9 / "precision budget"):
//   generic q   : Xi_c = round(frac(r_c / L) * 2^32)   -> 2 x uint4 {Xi_x, Xi_y, Xi_z, f}{xi_x, xi_y, xi_z, 0}
//   lattice q   : Theta_v = v . Xi (mod 2^32) for v = ma, mb, m0           -> uint4 {Th_a, Th_b, Th_0, f}
// because q . r / 2 pi = (m . r) / L for q = (2 pi / L) m with integer m, so the phase in turns is the integer
// combination of the box fractions, exact modulo 1.  fp64 inputs use 64-bit turns (ulonglong4).
// HBM-bound: reads 12-24 B and writes 16-32 B per atom per frame (32 B for the generic fp32 record).
#include "common.cuh"

namespace xpcs {

template <typename P, typename F>
__global__ void __launch_bounds__(256) k_stage_lattice32(const P* __restrict__ pos, const F* __restrict__ f,
                                                         int64_t N, int64_t total, LatticeGeom g,
                                                         uint4* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const P* r = pos + 3 * i;
        uint32_t X[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) X[c] = frac_to_fixed32(box_fraction((double)r[c], g.L));
        uint32_t th[3];
        const int32_t* m[3] = {g.ma, g.mb, g.m0};
#pragma unroll
        for (int v = 0; v < 3; ++v)
            th[v] = (uint32_t)m[v][0] * X[0] + (uint32_t)m[v][1] * X[1] + (uint32_t)m[v][2] * X[2];
        const float fj = f ? (float)f[i % N] : 1.0f;
        out[i] = make_uint4(th[0], th[1], th[2], __float_as_uint(fj));
    }
}

__global__ void __launch_bounds__(256) k_stage_lattice64(const double* __restrict__ pos, const double* __restrict__ f,
                                                         int64_t N, int64_t total, LatticeGeom g,
                                                         ulonglong4* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const double* r = pos + 3 * i;
        uint64_t X[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) X[c] = frac_to_fixed64(box_fraction(r[c], g.L));
        uint64_t th[3];
        const int32_t* m[3] = {g.ma, g.mb, g.m0};
#pragma unroll
        for (int v = 0; v < 3; ++v)
            th[v] = (uint64_t)(int64_t)m[v][0] * X[0] + (uint64_t)(int64_t)m[v][1] * X[1] +
                    (uint64_t)(int64_t)m[v][2] * X[2];
        const double fj = f ? f[i % N] : 1.0;
        out[i] = make_ulonglong4(th[0], th[1], th[2], (unsigned long long)__double_as_longlong(fj));
    }
}

// generic record (32 B): {Xi_x, Xi_y, Xi_z, f} exact 32-bit box fractions + {xi_x, xi_y, xi_z, 0} the same
// fractions as fp32 (for the fractional part of q.r, see k_generic.cu)
template <typename P, typename F>
__global__ void __launch_bounds__(256) k_stage_generic32(const P* __restrict__ pos, const F* __restrict__ f,
                                                         int64_t N, int64_t total, double L,
                                                         uint4* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const P* r = pos + 3 * i;
        const double ux = box_fraction((double)r[0], L), uy = box_fraction((double)r[1], L),
                     uz = box_fraction((double)r[2], L);
        const uint32_t x = frac_to_fixed32(ux), y = frac_to_fixed32(uy), z = frac_to_fixed32(uz);
        const float fj = f ? (float)f[i % N] : 1.0f;
        out[2 * i] = make_uint4(x, y, z, __float_as_uint(fj));
        // fp32 fractions of the same fixed-point values (x * 2^-32 rounded once)
        out[2 * i + 1] = make_uint4(__float_as_uint((float)((double)x * 2.3283064365386963e-10)),
                                    __float_as_uint((float)((double)y * 2.3283064365386963e-10)),
                                    __float_as_uint((float)((double)z * 2.3283064365386963e-10)), 0u);
    }
}

__global__ void __launch_bounds__(256) k_stage_generic64(const double* __restrict__ pos, const double* __restrict__ f,
                                                         int64_t N, int64_t total, double L,
                                                         ulonglong4* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const double* r = pos + 3 * i;
        const double fj = f ? f[i % N] : 1.0;
        out[i] = make_ulonglong4(frac_to_fixed64(box_fraction(r[0], L)), frac_to_fixed64(box_fraction(r[1], L)),
                                 frac_to_fixed64(box_fraction(r[2], L)),
                                 (unsigned long long)__double_as_longlong(fj));
    }
}

static dim3 grid_for(int64_t total) {
    int64_t b = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    return dim3((unsigned)(b < cap ? (b > 0 ? b : 1) : cap));
}

cudaError_t launch_stage_lattice32(const void* pos, int pos_f64, const void* f, int f_f64, int64_t N,
                                   int64_t frames, const LatticeGeom& g, uint4* out, cudaStream_t s) {
    const int64_t total = N * frames;
    note_launch();
    if (pos_f64) {
        if (f_f64) k_stage_lattice32<double, double><<<grid_for(total), 256, 0, s>>>((const double*)pos, (const double*)f, N, total, g, out);
        else k_stage_lattice32<double, float><<<grid_for(total), 256, 0, s>>>((const double*)pos, (const float*)f, N, total, g, out);
    } else {
        if (f_f64) k_stage_lattice32<float, double><<<grid_for(total), 256, 0, s>>>((const float*)pos, (const double*)f, N, total, g, out);
        else k_stage_lattice32<float, float><<<grid_for(total), 256, 0, s>>>((const float*)pos, (const float*)f, N, total, g, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_stage_lattice64(const void* pos, const void* f, int64_t N, int64_t frames,
                                   const LatticeGeom& g, ulonglong4* out, cudaStream_t s) {
    const int64_t total = N * frames;
    note_launch();
    k_stage_lattice64<<<grid_for(total), 256, 0, s>>>((const double*)pos, (const double*)f, N, total, g, out);
    return cudaGetLastError();
}

cudaError_t launch_stage_generic32(const void* pos, int pos_f64, const void* f, int f_f64, int64_t N,
                                   int64_t frames, double L, uint4* out, cudaStream_t s) {
    const int64_t total = N * frames;
    note_launch();
    if (pos_f64) {
        if (f_f64) k_stage_generic32<double, double><<<grid_for(total), 256, 0, s>>>((const double*)pos, (const double*)f, N, total, L, out);
        else k_stage_generic32<double, float><<<grid_for(total), 256, 0, s>>>((const double*)pos, (const float*)f, N, total, L, out);
    } else {
        if (f_f64) k_stage_generic32<float, double><<<grid_for(total), 256, 0, s>>>((const float*)pos, (const double*)f, N, total, L, out);
        else k_stage_generic32<float, float><<<grid_for(total), 256, 0, s>>>((const float*)pos, (const float*)f, N, total, L, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_stage_generic64(const void* pos, const void* f, int64_t N, int64_t frames, double L,
                                   ulonglong4* out, cudaStream_t s) {
    const int64_t total = N * frames;
    note_launch();
    k_stage_generic64<<<grid_for(total), 256, 0, s>>>((const double*)pos, (const double*)f, N, total, L, out);
    return cudaGetLastError();
}

}  // namespace xpcs
