// k_lattice_simt.cu -- K2: lattice-plane amplitude on FP32 CUDA cores.
//
// For q = (2 pi / L)(m0 + h ma + k mb) the phase factorises per axis (exact identity of Eq. 7):
//     p^e(h,k) = sum_j X_h(j) W_k(j),   X_h(j) = e^{-2 pi i h Th_a(j)},  W_k(j) = f_j e^{-2 pi i (Th_0(j) + k Th_b(j))}
// with Th_v the staged 32-bit turns (k_stage.cu).  Per CTA: a TH x TK pixel tile of one frame and a chunk of
// <= chunk_atoms atoms.  Per 16-atom sub-block the CTA generates the 16 x (TH + TK) phasors into shared memory
// (exact integer turns h * Th_a mod 2^32 -> SFU sin/cos, |error| < 1e-6 per phasor), then every thread accumulates a
// RH x RK register tile of complex MACs with packed FFMA2:
//     (re, im) += (xr, xr) * (wr, wi) ;  (re, im) += (-xi, xi) * (wi, wr)        -> 2 FFMA2 per atom.q pair
// fp32 accumulation never spans more than chunk_atoms (<= 4096) atoms; chunks are combined in FP64 by the
// reduction kernel.  Output: partial[c][t][pixel] (float2).
#include "common.cuh"

namespace xpcs {

namespace {
constexpr int TH = 64, TK = 128, RH = 4, RK = 8, SB = 16, NT = 256;
static_assert((TH / RH) * (TK / RK) == NT, "thread tiling");
}

__global__ void __launch_bounds__(NT, 2)
k_lattice_simt(const uint4* __restrict__ staged, int64_t N, LatticeGeom g, int64_t chunk_atoms,
               int tiles_k, float2* __restrict__ partial, int64_t frames) {
    extern __shared__ float4 smem[];
    float4* Xs = smem;                 // [SB][TH]   (xr, xr, -xi, xi)
    float4* Ws = smem + SB * TH;       // [SB][TK]   (wr, wi, wi, wr)

    const int tile = blockIdx.x;
    const int th0 = (tile / tiles_k) * TH, tk0 = (tile % tiles_k) * TK;
    const int64_t chunk = blockIdx.y;
    const int64_t t = blockIdx.z;
    const int64_t a_begin = chunk * chunk_atoms;
    const int64_t a_end = min(N, a_begin + chunk_atoms);
    const uint4* S = staged + t * N;

    const int tid = threadIdx.x;
    const int hg = tid / (TK / RK);          // 0..15 : rows hg*RH .. +RH-1
    const int kg = tid % (TK / RK);          // 0..15 : cols kg + 16 j

    unsigned long long acc[RH][RK];
#pragma unroll
    for (int i = 0; i < RH; ++i)
#pragma unroll
        for (int j = 0; j < RK; ++j) acc[i][j] = 0ull;

    for (int64_t a0 = a_begin; a0 < a_end; a0 += SB) {
        // ---- generate phasors for atoms a0 .. a0+SB-1 (zero beyond a_end)
        for (int e = tid; e < SB * TH; e += NT) {
            const int a = e / TH, m = e % TH;
            const int64_t j = a0 + a;
            float c = 0.f, s = 0.f;
            if (j < a_end) {
                const uint4 st = S[j];
                const uint32_t T = (uint32_t)(g.h0 + th0 + m) * st.x;       // h * Th_a mod 2^32 (exact)
                __sincosf(turns_to_radians(T), &s, &c);
            }
            // X = cos - i sin  ->  (xr, xr, -xi, xi) = (c, c, s, -s)
            Xs[a * TH + m] = make_float4(c, c, s, -s);
        }
        for (int e = tid; e < SB * TK; e += NT) {
            const int a = e / TK, m = e % TK;
            const int64_t j = a0 + a;
            float c = 0.f, s = 0.f, f = 0.f;
            if (j < a_end) {
                const uint4 st = S[j];
                const uint32_t T = st.z + (uint32_t)(g.k0 + tk0 + m) * st.y;  // Th_0 + k Th_b mod 2^32
                __sincosf(turns_to_radians(T), &s, &c);
                f = __uint_as_float(st.w);
            }
            const float wr = f * c, wi = -f * s;
            Ws[a * TK + m] = make_float4(wr, wi, wi, wr);
        }
        __syncthreads();
#pragma unroll 2
        for (int a = 0; a < SB; ++a) {
            float4 x[RH], w[RK];
#pragma unroll
            for (int i = 0; i < RH; ++i) x[i] = Xs[a * TH + hg * RH + i];
#pragma unroll
            for (int jj = 0; jj < RK; ++jj) w[jj] = Ws[a * TK + kg + (TK / RK) * jj];
#pragma unroll
            for (int i = 0; i < RH; ++i) {
                const unsigned long long xa = pack2(x[i].x, x[i].y), xb = pack2(x[i].z, x[i].w);
#pragma unroll
                for (int jj = 0; jj < RK; ++jj) {
                    acc[i][jj] = ffma2(xa, pack2(w[jj].x, w[jj].y), acc[i][jj]);
                    acc[i][jj] = ffma2(xb, pack2(w[jj].z, w[jj].w), acc[i][jj]);
                }
            }
        }
        __syncthreads();
    }

    // ---- write the fp32 partial amplitudes of this atom chunk
    const int64_t n_q = g.n_h * g.n_k;
    float2* P = partial + (chunk * frames + t) * n_q;
#pragma unroll
    for (int i = 0; i < RH; ++i) {
        const int64_t ih = th0 + hg * RH + i;
        if (ih >= g.n_h) continue;
#pragma unroll
        for (int jj = 0; jj < RK; ++jj) {
            const int64_t ik = tk0 + kg + (TK / RK) * jj;
            if (ik < g.n_k) P[ih * g.n_k + ik] = make_float2(lo2(acc[i][jj]), hi2(acc[i][jj]));
        }
    }
}

cudaError_t launch_lattice_simt(const uint4* staged, int64_t N, int64_t frames, const LatticeGeom& g,
                                int64_t chunk_atoms, int64_t n_chunks, float2* partial, cudaStream_t s) {
    const int tiles_h = (int)((g.n_h + TH - 1) / TH), tiles_k = (int)((g.n_k + TK - 1) / TK);
    const size_t smem = sizeof(float4) * SB * (TH + TK);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_lattice_simt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    dim3 grid(tiles_h * tiles_k, (unsigned)n_chunks, (unsigned)frames);
    note_launch();
    k_lattice_simt<<<grid, NT, smem, s>>>(staged, N, g, chunk_atoms, tiles_k, partial, frames);
    return cudaGetLastError();
}

}  // namespace xpcs
