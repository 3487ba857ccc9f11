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
// Staging also realises the 3-D q blocks (one virtual frame per (frame, l-plane)) and the species gather.
#include "common.cuh"
#include <algorithm>

namespace xpcs {

// Record i = vi * N + j of a batch is staged atom j of virtual frame v = m.v0 + vi; virtual frame v is source frame
// t = v / m.n_l and reciprocal-lattice plane l = m.l0 + v % m.n_l (3-D q blocks: Th_0 = (m0 + l mc) . Xi); staged
// atom j reads source atom m.idx[j] (species gather) or j.  Source frames hold m.n_src atoms.  The grid is 2-D
// (atoms x virtual frames): no per-record 64-bit division.
#define STAGE_LOOPS(N, V)                                                                                          \
    for (int64_t vi = blockIdx.y; vi < (V); vi += gridDim.y)                                                       \
        for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < (N); j += (int64_t)gridDim.x * blockDim.x)
__device__ __forceinline__ void stage_frame(const StageMap& m, int64_t vi, int64_t& t, int64_t& l) {
    const int64_t v = m.v0 + vi;
    t = m.n_l == 1 ? v : v / m.n_l;
    l = m.l0 + (v - t * m.n_l);
}
__device__ __forceinline__ int64_t stage_atom(const StageMap& m, int64_t j) { return m.idx ? (int64_t)m.idx[j] : j; }

template <typename P, typename F>
__global__ void __launch_bounds__(256) k_stage_lattice32(const P* __restrict__ pos, const F* __restrict__ f,
                                                         int64_t N, int64_t V, LatticeGeom g, StageMap m,
                                                         uint4* __restrict__ out) {
    // Xi = round(frac(x / L) 2^32) = rint(x (2^32 / L)) mod 2^32: the integer part of x / L only moves bits >= 32,
    // and x (2^32 / L) = (x / L) 2^32 exactly (power-of-two scaling), so one DMUL + one F2I per coordinate
    const double s32 = (1.0 / g.L) * 4294967296.0;
    for (int64_t vi = blockIdx.y; vi < V; vi += gridDim.y) {
        int64_t t, l;
        stage_frame(m, vi, t, l);
        int32_t m0[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) m0[c] = g.m0[c] + (int32_t)l * m.mc[c];
        const P* base = pos + 3 * t * m.n_src;
        uint4* o = out + vi * N;
#pragma unroll 1
        for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
            const int64_t src = stage_atom(m, j);
            const P* r = base + 3 * src;
            uint32_t X[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) X[c] = (uint32_t)(unsigned long long)llrint((double)r[c] * s32);
            uint32_t th[3];
            th[0] = (uint32_t)g.ma[0] * X[0] + (uint32_t)g.ma[1] * X[1] + (uint32_t)g.ma[2] * X[2];
            th[1] = (uint32_t)g.mb[0] * X[0] + (uint32_t)g.mb[1] * X[1] + (uint32_t)g.mb[2] * X[2];
            th[2] = (uint32_t)m0[0] * X[0] + (uint32_t)m0[1] * X[1] + (uint32_t)m0[2] * X[2];
            const float fj = f ? (float)f[src] : 1.0f;
            o[j] = make_uint4(th[0], th[1], th[2], __float_as_uint(fj));
        }
    }
}

__global__ void __launch_bounds__(256) k_stage_lattice64(const double* __restrict__ pos, const double* __restrict__ f,
                                                         int64_t N, int64_t V, LatticeGeom g, StageMap m,
                                                         ulonglong4* __restrict__ out) {
    STAGE_LOOPS(N, V) {
        int64_t t, l;
        stage_frame(m, vi, t, l);
        const int64_t src = stage_atom(m, j), i = vi * N + j;
        const double* r = pos + 3 * (t * m.n_src + src);
        uint64_t X[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) X[c] = frac_to_fixed64(box_fraction(r[c], g.L));
        uint64_t th[3];
        int64_t m0[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) m0[c] = (int64_t)g.m0[c] + l * (int64_t)m.mc[c];
        const int64_t mv[3][3] = {{g.ma[0], g.ma[1], g.ma[2]}, {g.mb[0], g.mb[1], g.mb[2]}, {m0[0], m0[1], m0[2]}};
#pragma unroll
        for (int k = 0; k < 3; ++k)
            th[k] = (uint64_t)mv[k][0] * X[0] + (uint64_t)mv[k][1] * X[1] + (uint64_t)mv[k][2] * X[2];
        const double fj = f ? f[src] : 1.0;
        out[i] = make_ulonglong4(th[0], th[1], th[2], (unsigned long long)__double_as_longlong(fj));
    }
}

// generic record (32 B): {Xi_x, Xi_y, Xi_z, f} exact 32-bit box fractions + {xi_x, xi_y, xi_z, 0} the same
// fractions as fp32 (for the fractional part of q.r, see k_generic.cu)
template <typename P, typename F>
__global__ void __launch_bounds__(256) k_stage_generic32(const P* __restrict__ pos, const F* __restrict__ f,
                                                         int64_t N, int64_t V, double L, StageMap m,
                                                         uint4* __restrict__ out) {
    const double invL = 1.0 / L;
    STAGE_LOOPS(N, V) {
        const int64_t v = m.v0 + vi, src = stage_atom(m, j), i = vi * N + j;
        const P* r = pos + 3 * (v * m.n_src + src);
        const double ux = box_fraction_fast((double)r[0], invL), uy = box_fraction_fast((double)r[1], invL),
                     uz = box_fraction_fast((double)r[2], invL);
        const uint32_t x = frac_to_fixed32(ux), y = frac_to_fixed32(uy), z = frac_to_fixed32(uz);
        const float fj = f ? (float)f[src] : 1.0f;
        out[2 * i] = make_uint4(x, y, z, __float_as_uint(fj));
        // fp32 fractions of the same fixed-point values (x * 2^-32 rounded once)
        out[2 * i + 1] = make_uint4(__float_as_uint((float)((double)x * 2.3283064365386963e-10)),
                                    __float_as_uint((float)((double)y * 2.3283064365386963e-10)),
                                    __float_as_uint((float)((double)z * 2.3283064365386963e-10)), 0u);
    }
}

__global__ void __launch_bounds__(256) k_stage_generic64(const double* __restrict__ pos, const double* __restrict__ f,
                                                         int64_t N, int64_t V, double L, StageMap m,
                                                         ulonglong4* __restrict__ out) {
    STAGE_LOOPS(N, V) {
        const int64_t v = m.v0 + vi, src = stage_atom(m, j), i = vi * N + j;
        const double* r = pos + 3 * (v * m.n_src + src);
        const double fj = f ? f[src] : 1.0;
        out[i] = make_ulonglong4(frac_to_fixed64(box_fraction(r[0], L)), frac_to_fixed64(box_fraction(r[1], L)),
                                 frac_to_fixed64(box_fraction(r[2], L)),
                                 (unsigned long long)__double_as_longlong(fj));
    }
}

// atoms x virtual frames, ~16 blocks of 256 threads per SM in total
static dim3 grid_for(int64_t N, int64_t V) {
    const int64_t cap = (int64_t)sm_count() * 16;
    const int64_t bx = std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, cap));
    const int64_t by = std::max<int64_t>(1, std::min<int64_t>({V, (cap + bx - 1) / bx, (int64_t)65535}));
    return dim3((unsigned)bx, (unsigned)by);
}

cudaError_t launch_stage_lattice32(const void* pos, int pos_f64, const void* f, int f_f64, int64_t N,
                                   int64_t frames, const LatticeGeom& g, const StageMap& m, uint4* out, cudaStream_t s) {
    note_launch();
    const dim3 gr = grid_for(N, frames);
    if (pos_f64) {
        if (f_f64) k_stage_lattice32<double, double><<<gr, 256, 0, s>>>((const double*)pos, (const double*)f, N, frames, g, m, out);
        else k_stage_lattice32<double, float><<<gr, 256, 0, s>>>((const double*)pos, (const float*)f, N, frames, g, m, out);
    } else {
        if (f_f64) k_stage_lattice32<float, double><<<gr, 256, 0, s>>>((const float*)pos, (const double*)f, N, frames, g, m, out);
        else k_stage_lattice32<float, float><<<gr, 256, 0, s>>>((const float*)pos, (const float*)f, N, frames, g, m, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_stage_lattice64(const void* pos, const void* f, int64_t N, int64_t frames,
                                   const LatticeGeom& g, const StageMap& m, ulonglong4* out, cudaStream_t s) {
    note_launch();
    k_stage_lattice64<<<grid_for(N, frames), 256, 0, s>>>((const double*)pos, (const double*)f, N, frames, g, m, out);
    return cudaGetLastError();
}

cudaError_t launch_stage_generic32(const void* pos, int pos_f64, const void* f, int f_f64, int64_t N,
                                   int64_t frames, double L, const StageMap& m, uint4* out, cudaStream_t s) {
    note_launch();
    const dim3 gr = grid_for(N, frames);
    if (pos_f64) {
        if (f_f64) k_stage_generic32<double, double><<<gr, 256, 0, s>>>((const double*)pos, (const double*)f, N, frames, L, m, out);
        else k_stage_generic32<double, float><<<gr, 256, 0, s>>>((const double*)pos, (const float*)f, N, frames, L, m, out);
    } else {
        if (f_f64) k_stage_generic32<float, double><<<gr, 256, 0, s>>>((const float*)pos, (const double*)f, N, frames, L, m, out);
        else k_stage_generic32<float, float><<<gr, 256, 0, s>>>((const float*)pos, (const float*)f, N, frames, L, m, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_stage_generic64(const void* pos, const void* f, int64_t N, int64_t frames, double L,
                                   const StageMap& m, ulonglong4* out, cudaStream_t s) {
    note_launch();
    k_stage_generic64<<<grid_for(N, frames), 256, 0, s>>>((const double*)pos, (const double*)f, N, frames, L, m, out);
    return cudaGetLastError();
}

}  // namespace xpcs
