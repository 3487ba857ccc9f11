// k_fixup.cu -- exact recompute of the brightest pixels after the tensor engines (k_lattice_i8.cu, k_lattice_tc.cu).
//
// The tensor engines' per-term errors are independent across atoms for disordered frames and add like a random walk
// (rms |dI| ~ 3e-5 N), but where the phasors repeat -- q = 0 of any frame, where the conjugate-pair
// factors X_d and W are conjugates for every atom, and the Bragg peaks of a PERFECT crystal -- they add coherently:
// the integer engine's 16-bit limbs up to ~2e-5 of I (tools/i8_limb_emulation.py), the split-FP16 engine's
// truncating FP32 TMEM accumulator ~1.5e-5; both above the 1e-5 relative branch of the per-pixel gate (DESIGN.md
// R11), which only matters where I > 100 N.  So every pixel whose intensity exceeds
//     thresh(q) = min(64 N, N^2 / 4) * F(q)^2,   F(q) = max |f| of the call's atoms at q,
// is recomputed here by the plain Eq.(7)/(8) sum over the staged atoms: exact 32-bit phase turns
// -> sincospi (FP32, ~1 ulp per term, ~1e-7 of I even when coherent) -> FP64 sums, fixed-order reductions
// (deterministic).  A disordered frame has no such pixel except q = 0 (I = (sum f)^2; P(I > 64 <I>) = e^-64), so the
// cost is one N-atom sum per frame; a crystal adds its Bragg peaks.
// The epilogue that writes the batch's I (the integer engine's direct drain, the chunk fold or the species combine)
// appends bright pixels to a list (BrightSink, common.cuh); the kernels here recompute the listed pixels.
#include "common.cuh"

namespace xpcs {

namespace {

__device__ __forceinline__ double fix_weight(const FixGroups& G, int g, int64_t v, int64_t pix, int64_t n_q) {
    if (!G.fq) return 1.0;
    const int64_t row = (G.v0 + v) % G.n_l;
    const int64_t i = (int64_t)G.kind[g] * G.n_l * n_q + row * n_q + pix;
    return G.fq_f64 ? ((const double*)G.fq)[i] : (double)((const float*)G.fq)[i];
}

// p = sum_j f e^{-i q.r_j} of each listed pixel from the staged exact turns: sincospi in FP32 on the turn
// fraction (|error| ~ 1 ulp per term), FP64 sums, fixed-order reductions (deterministic).  The first FIX_SPLIT_MAX
// entries are split into atom chunks of FIX_CHUNK over many blocks (a disordered frame has ~1 entry, so one pixel per
// block would leave the GPU idle for a whole N-atom latency chain): item (entry, chunk) -> partial[entry][chunk];
// pass 3 folds the chunks in order.  Entries beyond FIX_SPLIT_MAX (only pathological, bright-everywhere inputs) take
// one block each.
constexpr int FIX_THREADS = 256, FIX_U = 8, FIX_CHUNK = FIX_THREADS * FIX_U * 2;   // 4096 atoms per item
constexpr uint32_t FIX_SPLIT_MAX = 4096;

__device__ __forceinline__ void fix_pixel(const FixGroups& G, const LatticeGeom& g, int64_t e, int64_t n_q, int64_t a0,
                                          int64_t a1, double& pre, double& pim) {
    // atoms [a0, a1) of the concatenated groups, this thread's share; returns the block-reduced FP64 sum in thread 0
    __shared__ double red[2][FIX_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t v = e / n_q, pix = e - v * n_q;
    const int64_t ih = pix / g.n_k, ik = pix - ih * g.n_k;
    const uint32_t h = (uint32_t)(g.h0 + ih), k = (uint32_t)(g.k0 + ik);
    pre = 0.0; pim = 0.0;
    int64_t gbase = 0;
    for (int s = 0; s < G.n_groups; ++s) {
        const int64_t n = G.n[s];
        const int64_t lo = max(a0 - gbase, (int64_t)0), hi = min(a1 - gbase, n);
        double sre = 0.0, sim = 0.0;
        if (lo < hi) {
            const uint4* S = G.st[s] + v * n;
            for (int64_t j0 = lo + threadIdx.x; j0 < hi; j0 += (int64_t)FIX_THREADS * FIX_U) {
                uint4 r[FIX_U];
#pragma unroll
                for (int u = 0; u < FIX_U; ++u) {
                    const int64_t j = j0 + (int64_t)u * FIX_THREADS;
                    r[u] = j < hi ? __ldg(S + j) : make_uint4(0u, 0u, 0u, 0u);   // f = 0: no contribution
                }
#pragma unroll
                for (int u = 0; u < FIX_U; ++u) {
                    const uint32_t T = r[u].z + h * r[u].x + k * r[u].y;     // q.r / 2 pi in turns, exact mod 1
                    float sn, cs;
                    sincospif(2.0f * turns_signed(T), &sn, &cs);
                    const float f = __uint_as_float(r[u].w);
                    sre += (double)(f * cs);                                   // f * cs exact-ish: f in {1, 2, ...}
                    sim -= (double)(f * sn);                                   // e^{-i q.r} (Eq. 7)
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sre += __shfl_xor_sync(0xffffffffu, sre, o);
            sim += __shfl_xor_sync(0xffffffffu, sim, o);
        }
        __syncthreads();
        if (lane == 0) { red[0][wid] = sre; red[1][wid] = sim; }
        __syncthreads();
        if (threadIdx.x == 0) {
            sre = 0.0; sim = 0.0;
            for (int w = 0; w < FIX_THREADS / 32; ++w) { sre += red[0][w]; sim += red[1][w]; }
            const double wgt = fix_weight(G, s, v, pix, n_q);
            pre += wgt * sre;
            pim += wgt * sim;
        }
        gbase += n;
    }
}

__device__ __forceinline__ void fix_store(void* out, int64_t e, int out_f64, int amp, double pre, double pim) {
    if (amp) {
        if (out_f64) { ((double*)out)[2 * e] = pre; ((double*)out)[2 * e + 1] = pim; }
        else ((float2*)out)[e] = make_float2((float)pre, (float)pim);
    } else {
        const double I = pre * pre + pim * pim;
        if (out_f64) ((double*)out)[e] = I;
        else ((float*)out)[e] = (float)I;
    }
}

__global__ void __launch_bounds__(FIX_THREADS) k_fix_chunks(FixGroups G, LatticeGeom g, int64_t n_atoms,
                                                            const uint32_t* __restrict__ count,
                                                            const uint32_t* __restrict__ list,
                                                            double2* __restrict__ partial) {
    const int64_t n_q = g.n_h * g.n_k;
    const int64_t n_ch = (n_atoms + FIX_CHUNK - 1) / FIX_CHUNK;
    const int64_t items = (int64_t)min(*count, FIX_SPLIT_MAX) * n_ch;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t li = it / n_ch, c = it - li * n_ch;
        double pre, pim;
        fix_pixel(G, g, (int64_t)list[li], n_q, c * FIX_CHUNK, min((c + 1) * FIX_CHUNK, n_atoms), pre, pim);
        if (threadIdx.x == 0) partial[it] = make_double2(pre, pim);
    }
}

__global__ void __launch_bounds__(FIX_THREADS) k_fix_whole(FixGroups G, LatticeGeom g, int64_t n_atoms,
                                                           const uint32_t* __restrict__ count,
                                                           const uint32_t* __restrict__ list,
                                                           void* __restrict__ out, int out_f64, int amp) {
    const int64_t n_q = g.n_h * g.n_k;
    for (uint32_t li = FIX_SPLIT_MAX + blockIdx.x; li < *count; li += gridDim.x) {
        double pre, pim;
        fix_pixel(G, g, (int64_t)list[li], n_q, 0, n_atoms, pre, pim);
        if (threadIdx.x == 0) fix_store(out, (int64_t)list[li], out_f64, amp, pre, pim);
    }
}

__global__ void __launch_bounds__(256) k_fix_fold(int64_t n_atoms, const uint32_t* __restrict__ count,
                                                  const uint32_t* __restrict__ list, const double2* __restrict__ partial,
                                                  void* __restrict__ out, int out_f64, int amp) {
    const int64_t n_ch = (n_atoms + FIX_CHUNK - 1) / FIX_CHUNK;
    const uint32_t n = min(*count, FIX_SPLIT_MAX);
    for (uint32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < n; li += gridDim.x * blockDim.x) {
        double pre = 0.0, pim = 0.0;
        for (int64_t c = 0; c < n_ch; ++c) { const double2 z = partial[li * n_ch + c]; pre += z.x; pim += z.y; }
        fix_store(out, (int64_t)list[li], out_f64, amp, pre, pim);
    }
}

}  // namespace

static int64_t fix_atoms(const FixGroups& G) {
    int64_t n = 0;
    for (int i = 0; i < G.n_groups; ++i) n += G.n[i];
    return n;
}

size_t fixup_scratch_bytes(int64_t vb, int64_t n_q, int64_t n_atoms) {
    const size_t n_ch = (size_t)((n_atoms + FIX_CHUNK - 1) / FIX_CHUNK);
    return 256 + ((sizeof(uint32_t) * (size_t)(vb * n_q) + 255) / 256) * 256 + sizeof(double2) * FIX_SPLIT_MAX * n_ch;
}

cudaError_t fixup_prepare(void* scratch_buf, int64_t n_atoms, const float* fmax, BrightSink& out, cudaStream_t s) {
    const double na = (double)n_atoms;
    out.count = (uint32_t*)scratch_buf;
    out.list = (uint32_t*)((char*)scratch_buf + 256);
    out.thr = std::min(64.0 * na, 0.25 * na * na);
    out.fmax = fmax;
    return cudaMemsetAsync(out.count, 0, sizeof(uint32_t), s);
}

cudaError_t launch_fixup(const FixGroups& G, const LatticeGeom& g, int64_t vb, void* out, int out_f64, int amp,
                         void* scratch_buf, cudaStream_t s) {
    const int64_t n_q = g.n_h * g.n_k, total = vb * n_q;
    if (total > (int64_t)0xFFFFFFFFu) return cudaErrorInvalidValue;
    const int64_t n_call = fix_atoms(G);
    const uint32_t* count = (const uint32_t*)scratch_buf;
    const uint32_t* list = (const uint32_t*)((const char*)scratch_buf + 256);
    double2* partial = (double2*)((char*)scratch_buf + 256 + ((sizeof(uint32_t) * (size_t)total + 255) / 256) * 256);
    note_launch(3);
    k_fix_chunks<<<(unsigned)(sm_count() * 8), FIX_THREADS, 0, s>>>(G, g, n_call, count, list, partial);
    k_fix_whole<<<(unsigned)(sm_count() * 4), FIX_THREADS, 0, s>>>(G, g, n_call, count, list, out, out_f64, amp);
    k_fix_fold<<<(unsigned)sm_count(), 256, 0, s>>>(n_call, count, list, partial, out, out_f64, amp);
    return cudaGetLastError();
}

}  // namespace xpcs
