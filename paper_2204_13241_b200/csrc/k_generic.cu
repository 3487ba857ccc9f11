// k_generic.cu -- K1: direct structure-factor sum at an explicit list of q vectors (any q: Ewald detector pixels,
// off-lattice points), and the FP64 kernels.  SURVEY 8(a) rows a3/a4; Eq.(7)-(8), PAPER.md:127-138;
// Algorithm 1 step 2, PAPER.md:296 ("summing e^{-i q.r_i} over each atom").
//
// Phase arithmetic: the phase in turns is q . r / 2 pi = sum_c g_c u_c with
// g_c = q_c L / 2 pi (per q, formed once in FP64) and u_c = r_c / L in [0, 1) (per atom, staged as 32-bit fixed
// point Xi_c and as fp32 xi_c).  Writing g_c = n_c + phi_c (integer part, fraction in [0, 1)):
//     turns = [ sum_c n_c Xi_c mod 2^32 ] * 2^-32  +  sum_c phi_c xi_c
// the first term exact in integer arithmetic (3 IMAD; one I2FP rounds the signed turns to fp32, <= 2^-25 turns), the
// second in fp32 FFMA (|error| <~ 2e-7 turns, and the per-q rounding of phi_c only moves q by < 1e-7 of a
// reciprocal-lattice spacing).  No rounded 2 pi ever multiplies a large argument.
// The angle then goes to the SFU: FFMA -> FMUL.RZ -> MUFU.SIN / MUFU.COS (2 XU ops per atom.q pair, the
// pipe that bounds this kernel), and f_j cos / f_j sin accumulate in fp32 for at most SUB atoms before being
// folded into FP64 registers.
#include "common.cuh"

namespace xpcs {

#ifndef XPCS_GEN_QT
#define XPCS_GEN_QT 2          // q per thread (c4: 2 q x 3 CTAs/SM 1.915e12 pairs/s vs 4 q x 2 CTAs/SM 1.881e12)
#endif
#ifndef XPCS_GEN_I2F
#define XPCS_GEN_I2F 1         // integer turns -> fp32 by one I2FP (c4: 1.97e12 pairs/s) instead of the shift /
                               // exponent-OR trick (0: SHF + LOP3 + FFMA, 1.89e12)
#endif
#ifndef XPCS_GEN_DERIVE
#define XPCS_GEN_DERIVE 0      // 1: the fp32 fractions xi_c = Xi_c 2^-32 by I2FP in the thread (one shared record per atom)
#endif
#ifndef XPCS_GEN_MINB
#define XPCS_GEN_MINB 3        // resident CTAs per SM the register budget is sized for
#endif
namespace {
constexpr int GT = 256;     // threads per CTA
constexpr int QT = XPCS_GEN_QT;       // q per thread
constexpr int SUB = 512;    // atoms per shared-memory sub-block (also the fp32 accumulation length)
}

int generic_q_per_block() { return GT * QT; }
int generic_blocks_per_sm() { return XPCS_GEN_MINB; }

__device__ __forceinline__ void q_split(double qc, double L_over_2pi, uint32_t& n, float& two_pi_phi) {
    const double gq = qc * L_over_2pi;
    const double fl = floor(gq);
    n = (uint32_t)(unsigned long long)(long long)fl;
    two_pi_phi = (float)((gq - fl) * 6.283185307179586476925);
}

template <typename Q>
__global__ void __launch_bounds__(GT, XPCS_GEN_MINB)
k_generic32(const uint4* __restrict__ staged, int64_t N, const Q* __restrict__ q, int64_t n_q, double L_over_2pi,
            int64_t chunk_atoms, int64_t frames, double2* __restrict__ partial) {
    __shared__ uint4 As[2 * SUB];
    const int64_t t = blockIdx.z;
    const int64_t chunk = blockIdx.y;
    const int64_t a_begin = chunk * chunk_atoms, a_end = min(N, a_begin + chunk_atoms);
    const uint4* S = staged + 2 * t * N;

    uint32_t nx[QT], ny[QT], nz[QT];
    float px[QT], py[QT], pz[QT];
    int64_t iq[QT];
#pragma unroll
    for (int i = 0; i < QT; ++i) {
        iq[i] = (int64_t)blockIdx.x * (GT * QT) + threadIdx.x + GT * i;
        const int64_t qq = iq[i] < n_q ? iq[i] : 0;
        q_split((double)q[3 * qq + 0], L_over_2pi, nx[i], px[i]);
        q_split((double)q[3 * qq + 1], L_over_2pi, ny[i], py[i]);
        q_split((double)q[3 * qq + 2], L_over_2pi, nz[i], pz[i]);
#if XPCS_GEN_DERIVE
        px[i] *= 2.3283064365386963e-10f;                     // 2^-32: exact
        py[i] *= 2.3283064365386963e-10f;
        pz[i] *= 2.3283064365386963e-10f;
#endif
    }
    double dre[QT], dim[QT];
#pragma unroll
    for (int i = 0; i < QT; ++i) dre[i] = dim[i] = 0.0;

    for (int64_t a0 = a_begin; a0 < a_end; a0 += SUB) {
        const int cnt = (int)min((int64_t)SUB, a_end - a0);
        __syncthreads();
#if XPCS_GEN_DERIVE
        for (int e = threadIdx.x; e < SUB; e += GT) As[e] = e < cnt ? S[2 * (a0 + e)] : make_uint4(0, 0, 0, 0);
#else
        for (int e = threadIdx.x; e < 2 * SUB; e += GT) As[e] = (e >> 1) < cnt ? S[2 * a0 + e] : make_uint4(0, 0, 0, 0);
#endif
        __syncthreads();
        float re[QT], im[QT];
#pragma unroll
        for (int i = 0; i < QT; ++i) re[i] = im[i] = 0.f;
#pragma unroll 4
        for (int a = 0; a < SUB; ++a) {
#if XPCS_GEN_DERIVE
            const uint4 at = As[a];                               // broadcast: exact fractions + f
            const float fj = __uint_as_float(at.w);               // 0 for padding atoms
            // xi_c 2^32 (the 2^-32 sits in px / py / pz)
            const float xf = __uint2float_rn(at.x), yf = __uint2float_rn(at.y), zf = __uint2float_rn(at.z);
#else
            const uint4 at = As[2 * a];                           // broadcast: exact fractions + f
            const uint4 af = As[2 * a + 1];                       // fp32 fractions
            const float fj = __uint_as_float(at.w);               // 0 for padding atoms
            const float xf = __uint_as_float(af.x), yf = __uint_as_float(af.y), zf = __uint_as_float(af.z);
#endif
#pragma unroll
            for (int i = 0; i < QT; ++i) {
                uint32_t T = nx[i] * at.x;
                T = ny[i] * at.y + T;
                T = nz[i] * at.z + T;
#if XPCS_GEN_I2F
                // signed turns to fp32 by one I2FP (round to nearest), scaled inside the last FFMA
                float th = fmaf(px[i], xf, fmaf(py[i], yf, pz[i] * zf));  // 2 pi sum_c phi_c xi_c
                th = fmaf(__int2float_rn((int32_t)T), 1.46291807926715968e-9f, th);   // + 2 pi T 2^-32
#else
                float th = turns_to_radians(T);                   // integer part of the phase, in [-pi, pi)
                th = fmaf(px[i], xf, th);                         // + 2 pi sum_c phi_c xi_c
                th = fmaf(py[i], yf, th);
                th = fmaf(pz[i], zf, th);
#endif
                float s, c;
                __sincosf(th, &s, &c);
                re[i] = fmaf(fj, c, re[i]);
                im[i] = fmaf(fj, s, im[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < QT; ++i) { dre[i] += (double)re[i]; dim[i] += (double)im[i]; }
    }
    double2* P = partial + (chunk * frames + t) * n_q;
#pragma unroll
    for (int i = 0; i < QT; ++i)
        if (iq[i] < n_q) P[iq[i]] = make_double2(dre[i], -dim[i]);     // e^{-i phase}: Im = -sum f sin
}

// ---- FP64 generic: 64-bit turns, sincospi in FP64 (config-1 class precision)
__device__ __forceinline__ void q_to_fixed64(double qc, double L_over_2pi, uint64_t& n, uint64_t& phi) {
    const double gq = qc * L_over_2pi;
    const double fl = floor(gq);
    const double fr = gq - fl;
    n = (uint64_t)(long long)fl;
    // fraction to 64-bit fixed point (fr has <= 53 significant bits: exact)
    const double hi = floor(fr * 4294967296.0);
    const double lo = (fr * 4294967296.0 - hi) * 4294967296.0;
    phi = ((uint64_t)hi << 32) + (uint64_t)llrint(lo);
}

__global__ void __launch_bounds__(128)
k_generic64(const ulonglong4* __restrict__ staged, int64_t N, const double* __restrict__ q, int64_t n_q,
            double L_over_2pi, int64_t frames, double2* __restrict__ partial) {
    __shared__ ulonglong4 As[128];
    const int64_t t = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x;
    const int64_t qq = i < n_q ? i : 0;
    uint64_t n[3], p[3];
    for (int c = 0; c < 3; ++c) q_to_fixed64(q[3 * qq + c], L_over_2pi, n[c], p[c]);
    const ulonglong4* S = staged + t * N;
    double re = 0.0, im = 0.0;
    for (int64_t a0 = 0; a0 < N; a0 += 128) {
        __syncthreads();
        const int64_t j = a0 + threadIdx.x;
        As[threadIdx.x] = j < N ? S[j] : make_ulonglong4(0, 0, 0, 0);
        __syncthreads();
        const int cnt = (int)min((int64_t)128, N - a0);
        for (int a = 0; a < cnt; ++a) {
            const ulonglong4 at = As[a];
            uint64_t T = n[0] * at.x + n[1] * at.y + n[2] * at.z;
            T += __umul64hi(p[0], at.x) + __umul64hi(p[1], at.y) + __umul64hi(p[2], at.z);
            double s, c;
            sincospi(2.0 * turns_signed64(T), &s, &c);
            const double fj = __longlong_as_double((long long)at.w);
            re += fj * c;
            im -= fj * s;
        }
    }
    if (i < n_q) partial[t * n_q + i] = make_double2(re, im);
}

// ---- FP64 lattice: one pixel per thread, 64-bit turns (exact h*Th_a + k*Th_b + Th_0 mod 2^64)
template <typename O>
__global__ void __launch_bounds__(128)
k_lattice64(const ulonglong4* __restrict__ staged, int64_t N, LatticeGeom g, O* __restrict__ I_out, int mode,
            int64_t chunk_atoms, int64_t frames, double2* __restrict__ partial) {
    // partial != NULL: atom chunk blockIdx.z of chunk_atoms atoms -> partial[chunk][t][pix] (re, im), folded by
    // k_amp_reduce (split-K: a small plane x few frames cannot fill the device with one pixel per thread)
    __shared__ ulonglong4 As[128];
    const int64_t t = blockIdx.y;
    const int64_t n_q = g.n_h * g.n_k;
    const int64_t pix = (int64_t)blockIdx.x * 128 + threadIdx.x;
    const int64_t pp = pix < n_q ? pix : 0;
    const uint64_t h = (uint64_t)(g.h0 + pp / g.n_k), k = (uint64_t)(g.k0 + pp % g.n_k);
    const ulonglong4* S = staged + t * N;
    const int64_t a_begin = partial ? (int64_t)blockIdx.z * chunk_atoms : 0;
    const int64_t a_end = partial ? min(N, a_begin + chunk_atoms) : N;
    double re = 0.0, im = 0.0;
    for (int64_t a0 = a_begin; a0 < a_end; a0 += 128) {
        __syncthreads();
        const int64_t j = a0 + threadIdx.x;
        As[threadIdx.x] = j < a_end ? S[j] : make_ulonglong4(0, 0, 0, 0);
        __syncthreads();
        const int cnt = (int)min((int64_t)128, a_end - a0);
        for (int a = 0; a < cnt; ++a) {
            const ulonglong4 at = As[a];
            const uint64_t T = h * at.x + k * at.y + at.z;
            double s, c;
            sincospi(2.0 * turns_signed64(T), &s, &c);
            const double fj = __longlong_as_double((long long)at.w);
            re += fj * c;
            im -= fj * s;
        }
    }
    if (pix < n_q) {
        if (partial) partial[((int64_t)blockIdx.z * frames + t) * n_q + pix] = make_double2(re, im);
        else if (mode == 0) I_out[t * n_q + pix] = (O)(re * re + im * im);          // Eq.(8)
        else { I_out[2 * (t * n_q + pix)] = (O)re; I_out[2 * (t * n_q + pix) + 1] = (O)im; }   // Eq.(7)
    }
}

// ---- |sum_c P_c|^2 (FP64 fold of the atom chunks, fixed order)
// mode 0: I = |p|^2 (Eq. 8);  mode 1: p = (re, im) (Eq. 7);  mode 2: the partials hold conj(p) -> p
template <typename P, typename O>
__global__ void __launch_bounds__(256)
k_amp_reduce(const P* __restrict__ partial, int64_t C, int64_t total, O* __restrict__ out, int mode, BrightSink bs) {
    const double F = bs.count ? bright_F(bs) : 1.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        double re = 0.0, im = 0.0;
        int64_t c = 0;
        for (; c + 4 <= C; c += 4) {          // four loads in flight, added in chunk order
            P v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = partial[(c + u) * total + i];
#pragma unroll
            for (int u = 0; u < 4; ++u) { re += (double)v[u].x; im += (double)v[u].y; }
        }
        for (; c < C; ++c) {
            const P v = partial[c * total + i];
            re += (double)v.x;
            im += (double)v.y;
        }
        if (mode == 0) out[i] = (O)(re * re + im * im);          // Eq.(8): I = p p*
        else { out[2 * i] = (O)re; out[2 * i + 1] = (O)(mode == 2 ? -im : im); }
        bright_append(bs, re * re + im * im, F, i);
    }
}

cudaError_t launch_generic32(const uint4* staged, int64_t N, int64_t frames, const void* q, int q_f64,
                             int64_t n_q, double L, int64_t chunk_atoms, int64_t n_chunks, double2* partial,
                             cudaStream_t s) {
    dim3 grid((unsigned)((n_q + GT * QT - 1) / (GT * QT)), (unsigned)n_chunks, (unsigned)frames);
    const double l2p = L / (2.0 * 3.14159265358979323846);
    note_launch();
    if (q_f64) k_generic32<double><<<grid, GT, 0, s>>>(staged, N, (const double*)q, n_q, l2p, chunk_atoms, frames, partial);
    else k_generic32<float><<<grid, GT, 0, s>>>(staged, N, (const float*)q, n_q, l2p, chunk_atoms, frames, partial);
    return cudaGetLastError();
}

cudaError_t launch_generic64(const ulonglong4* staged, int64_t N, int64_t frames, const void* q,
                             int64_t n_q, double L, double2* partial, cudaStream_t s) {
    dim3 grid((unsigned)((n_q + 127) / 128), (unsigned)frames);
    note_launch();
    k_generic64<<<grid, 128, 0, s>>>(staged, N, (const double*)q, n_q, L / (2.0 * 3.14159265358979323846), frames, partial);
    return cudaGetLastError();
}

cudaError_t launch_lattice_f64(const ulonglong4* staged, int64_t N, int64_t frames, const LatticeGeom& g,
                               void* I_out, int out_f64, int mode, cudaStream_t s, double2* partial,
                               int64_t chunk_atoms, int64_t n_chunks) {
    const int64_t n_q = g.n_h * g.n_k;
    dim3 grid((unsigned)((n_q + 127) / 128), (unsigned)frames, (unsigned)(partial ? n_chunks : 1));
    note_launch();
    if (out_f64) k_lattice64<double><<<grid, 128, 0, s>>>(staged, N, g, (double*)I_out, mode, chunk_atoms, frames, partial);
    else k_lattice64<float><<<grid, 128, 0, s>>>(staged, N, g, (float*)I_out, mode, chunk_atoms, frames, partial);
    return cudaGetLastError();
}

static dim3 rgrid(int64_t total) {
    int64_t b = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    return dim3((unsigned)(b < cap ? (b > 0 ? b : 1) : cap));
}

cudaError_t launch_amp_reduce_f(const float2* partial, int64_t C, int64_t frames, int64_t n_q, void* I_out,
                                int out_f64, int mode, cudaStream_t s, const BrightSink* bright) {
    const int64_t total = frames * n_q;
    const BrightSink bs = bright ? *bright : BrightSink{nullptr, nullptr, 0.0, nullptr};
    note_launch();
    if (out_f64) k_amp_reduce<float2, double><<<rgrid(total), 256, 0, s>>>(partial, C, total, (double*)I_out, mode, bs);
    else k_amp_reduce<float2, float><<<rgrid(total), 256, 0, s>>>(partial, C, total, (float*)I_out, mode, bs);
    return cudaGetLastError();
}

cudaError_t launch_amp_reduce_d(const double2* partial, int64_t C, int64_t frames, int64_t n_q, void* I_out,
                                int out_f64, int mode, cudaStream_t s) {
    const int64_t total = frames * n_q;
    note_launch();
    const BrightSink bs{nullptr, nullptr, 0.0, nullptr};
    if (out_f64) k_amp_reduce<double2, double><<<rgrid(total), 256, 0, s>>>(partial, C, total, (double*)I_out, mode, bs);
    else k_amp_reduce<double2, float><<<rgrid(total), 256, 0, s>>>(partial, C, total, (float*)I_out, mode, bs);
    return cudaGetLastError();
}

}  // namespace xpcs
