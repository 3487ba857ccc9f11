// k_lattice_i8.cu -- K3b: lattice-plane amplitude on the tcgen05 INTEGER tensor cores (kind::i8, exact int32
// accumulation in TMEM), the fast engine for uniform form factors.
//
// Factorisation of Eq.(7) on a reciprocal-lattice plane: the phase in turns of
// pixel (h, k) is h Th_a + Th_0 + k Th_b (exact integer turns, k_stage.cu), so the amplitude is a complex matrix
// product over atoms.  CONJUGATE ROW PAIRS: a CTA pair owns 256 consecutive rows h = c +- d around the tile centre
// c = H0 + 127.5 (d = 1/2, 3/2, ..., 255/2).  With
//     X_d(j) = e^{2 pi i d Th_a(j)} = a + i b,   W_k(j) = (f_j / F) e^{2 pi i (Th_0 + k Th_b + c Th_a)(j)} = wr + i wi
// the tile holds q(h) = conj(p(h)) (the paper's sign e^{-iq.r}, R1) as
//     q(c + d, k) = sum_j X_d W_k       = (AR - BI) + i (AI + BR)
//     q(c - d, k) = sum_j conj(X_d) W_k = (AR + BI) + i (AI - BR),   AR = sum a.wr, AI = sum a.wi, BR = sum b.wr, BI = sum b.wi
// because X_{-d} = conj(X_d) exactly.  So ONE real matrix product [a; b] x [wr | wi]^T (M = 2 x 128 d, N = 2 x 128 k)
// yields both rows of every conjugate pair: 2 real MACs per pixel instead of the 4 of a complex MAC, and the X
// phasor table is half as long.  Every pixel is still evaluated from all N atoms (nothing is mirrored or skipped).
//
// Every phasor component v in [-1, 1] is written as two int8 limbs (Q16):
//     x = rint(32512 v) = 256 hi + lo,  hi = round(x / 256) in [-127, 127],  lo in [-128, 127]
// (|v - x / 32512| <= 1 / 65024 = 1.54e-5).  One FFMA t = fma(v, 32512, 1.5 * 2^23 + 128) leaves y = x + 128 in the
// low 16 bits of t: byte 1 = hi, byte 0 = lo + 128, so both limbs come from one instruction and two byte permutes.
// Each real product is
//     v w ~ [65536 hi.hi' + 256 (hi.lo' + lo.hi')] / 32512^2      (the dropped lo.lo' term is <= 1.55e-5, zero-mean)
// i.e. three int8 MMAs into two TMEM accumulators, HH = sum hi.hi' and X = sum (hi.lo' + lo.hi').  The integer
// accumulation is EXACT (no TMEM rounding, unlike the FP32 accumulator of the split-FP16 engine), so
// a chunk of up to 65536 atoms accumulates in TMEM and is drained once (int32 bound: |HH| <= 65536 x 127^2 and
// |X| <= 65536 x 2 x 127 x 128 = 2130706432 < 2^31; the drain converts each accumulator to FP32 before the
// conjugate-pair sums and differences).
// The int8 tensor rate is twice the fp16 rate on sm_100a (measured 8192 vs 4096 MAC/clk/SM, tools/mma_rate.cu).
//
// CTA pair (cluster of 2, cta_group::2): M = 256 (each CTA: rows [a | b] of its 64 d), N = 256 (each CTA: B rows
// [wr | wi] of its 64 k), K = 32 atoms per stage, 3 MMAs per stage:  HH += A_hi.B_hi,  X += A_hi.B_lo + A_lo.B_hi.
//
// Producers: NGROUPS groups of one X warp and one W warp, each covering the stage's 32 atoms (XPCS_I8_OCT = 0: 2 + 2
// warps, one per 16-atom K half); group g fills stages i = g mod NGROUPS of a STAGES-deep ring (16 KB per stage; the
// group count must not exceed the stage count, see the empty-barrier parity note in DESIGN.md 6.1).  A warp thread
// owns 8 consecutive atoms (two 32-bit words per row and limb plane, one STS.64) and 8 rows spaced 8 apart: rows 0
// and 1 from a start phasor and one angle-addition step X_{m+8} = X_m X_8 (2 SFU sincos per atom per thread), the
// rest by the sign-alternating Chebyshev recurrence (one packed FFMA per phasor-row); it quantises with one packed
// magic-number FFMA per phasor and packs limb bytes with PRMT.  After the last stage, warps 0-7 drain both accumulators through a
// shared-memory tile in 4 rounds of 32 k: p-components v = (65536 HH + 256 X) F / 32512^2 in FP32, then the
// conjugate-pair combination above with row-contiguous global writes of the partial amplitude or, with a single
// atom chunk, the final I = |p|^2 (or p) itself.
#include "common.cuh"
#include <type_traits>

namespace xpcs {

namespace ti8 {
constexpr int HD = 64;                              // d values per CTA (the pair covers 128 d = 256 h rows)
constexpr int TM = 2 * HD;                          // A rows per CTA: [a | b]
constexpr int PAIR_H = 4 * HD;                      // 256 output rows h per pair tile
#ifndef XPCS_I8_KS
#define XPCS_I8_KS 32
#endif
constexpr int TN = 128, KS = XPCS_I8_KS;            // pair tile cols (k), atoms per stage (32 or 64)
static_assert(KS == 32 || KS == 64, "stage of 32 or 64 atoms");
constexpr int KQ = KS / 16;                         // 16-atom K slices per stage (one X and one W warp each)
constexpr int RG = 8 * KS;                          // bytes per 8-row core-matrix group of a plane (SBO)
constexpr int BK = TN / 2;                          // k per CTA; B rows per CTA: [wr | wi] = 128
constexpr int PAIR_M = 2 * TM;                      // MMA M = 256
constexpr int PLANE = TM * KS;                      // int8 plane: 128 rows x KS atoms (A and B alike)
constexpr int HALF_ROWS = HD / 8 * RG;              // byte offset of row 64 in a plane
constexpr int STAGE_BYTES = 4 * PLANE;              // A_hi A_lo B_hi B_lo = 16 KB (KS = 32) / 32 KB (KS = 64)
#ifndef XPCS_I8_STAGES
#define XPCS_I8_STAGES (XPCS_I8_KS == 64 ? 6 : 8)
#endif
constexpr int STAGES = XPCS_I8_STAGES;
#ifndef XPCS_I8_OCT
#define XPCS_I8_OCT 1   // 1: a producer thread owns 8 consecutive atoms (STS.64; one X and one W warp per group cover
                        // K = 32); 0: 4 atoms (one X and one W warp per 16-atom K slice)
#endif
#ifndef XPCS_I8_GROUPS
#define XPCS_I8_GROUPS (XPCS_I8_KS == 64 ? 3 : (XPCS_I8_OCT ? 6 : 4))   // DESIGN.md 6.2 sweeps
#endif
constexpr int AT = XPCS_I8_OCT ? 8 : 4;             // atoms per producer thread
static_assert(AT == 4 || KS == 32, "8 atoms per thread: 32-atom stages");
constexpr int NGROUPS = XPCS_I8_GROUPS;
constexpr int GROUP_WARPS = AT == 8 ? 2 : 2 * KQ;   // per group: X and W warps (AT = 4: one per 16-atom K slice)
static_assert(NGROUPS <= STAGES, "mbarrier parity: producer groups must not exceed the stage count");
constexpr int NPROD_WARPS = NGROUPS * GROUP_WARPS;
constexpr int MMA_WARP = NPROD_WARPS;               // producer warps 0-7 (two per TMEM lane quarter) also drain the tile
static_assert(NPROD_WARPS >= 8, "the drain needs 8 producer warps");
constexpr int NTHREADS = (MMA_WARP + 1) * 32;
constexpr int MMA_N = 2 * TN;                       // 256
constexpr int TMEM_COLS = 512;                      // HH cols [0, 256), X cols [256, 512)
constexpr int ASL = 4;                              // atom-record slots per warp (cp.async prefetch distance ASL - 1)
constexpr int WREC = AT == 8 ? KS : 16;             // records a producer warp needs per stage
// record r of a warp's stage sits in 16-B unit r ^ ((r & 8) >> 2) of its slot: the cp.async writes (8 lanes per
// phase, records 0-7 / 8-15) and the per-field 32-bit reads of records {u, 4 + u, 8 + u, 12 + u} (one per quad)
// both hit distinct banks, one wavefront per instruction
constexpr int WSLOT = WREC;
constexpr int ASLOT_BYTES = NPROD_WARPS * ASL * WSLOT * 16;
constexpr int VLD = 65;                             // drain tile [128 rows][64 + 1] fp32
static_assert(TM * VLD * 4 <= STAGES * STAGE_BYTES, "drain tile must fit the stage ring");
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + ASLOT_BYTES + 1024 + 256;
constexpr float MAGIC = 12582912.0f;                // 1.5 * 2^23
// Q16 limbs: x = rint(QS v) in [-QS, QS], x = 256 hi + lo with hi in [-127, 127], lo in [-128, 127]; one FFMA
// t = fma(v, QS, M + 128) holds y = x + 128 in its low 16 bits: byte 1 = hi, byte 0 = lo + 128 (= lo ^ 0x80)
constexpr float QS = 32512.0f;
constexpr float QMAGIC = MAGIC + 128.0f;
#ifndef XPCS_I8_THREE_TERM
#define XPCS_I8_THREE_TERM 1   // rows by the sign-alternating Chebyshev recurrence (0: complex multiply per row)
#endif
#ifndef XPCS_I8_EXPERIMENTS
#define XPCS_I8_EXPERIMENTS 0   // 1: honour XPCS_I8_DEBUG bit 1 (skip production) in the producers' hot loop
#endif
// Global rotation: W carries an extra phase GAMMA (turns x 2^32), so both rows of a pair hold q e^{i Gamma} (Gamma =
// 2 pi GAMMA / 2^32) and the drain rotates it back (ROT_C, ROT_S = cos, sin Gamma).  Without it, X_d and W are exact
// conjugates (or equals) at q = 0 (X_d = e^{i pi Th_a}, W = e^{-i pi Th_a}), so their limbs' rounding errors -- and
// the dropped lo.lo' term -- add coherently over all atoms (2e-5 relative on I(0)); with the rotation the limbs of
// W are those of a rotated copy of X, which decorrelates them (tools/i8_limb_emulation.py).  |p|^2 is unchanged by a
// global phase.  (Perfect crystals repeat phasor values, so their Bragg peaks keep a coherent limb error of up to
// ~2e-5: k_fixup.cu recomputes such bright pixels exactly.)
constexpr uint32_t GAMMA = 0x3147AE14u;             // 0.1925 turns
constexpr float ROT_C = 0.35347484443612665f, ROT_S = 0.935444030581657f;
}  // namespace ti8

namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void i8_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
#ifndef XPCS_I8_WAIT_NS
#define XPCS_I8_WAIT_NS 0   // try_wait suspend-time hint in ns (0: none; 1 us - 1 ms hints measured no different on c2)
#endif
__device__ __forceinline__ void i8_mbar_wait(uint64_t* bar, uint32_t parity) {
#if XPCS_I8_WAIT_NS > 0
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WI8_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WI8_%=;\n\t}" ::"r"(su32(bar)),
        "r"(parity), "n"(XPCS_I8_WAIT_NS)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WI8_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WI8_%=;\n\t}" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
#endif
}
__device__ __forceinline__ void i8_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ uint32_t i8_mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t i8_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void i8_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t i8_desc(uint32_t saddr) {
    // K-major, no swizzle: core matrix 8 rows x 16 B; LBO = 128 B (K-adjacent core matrices), SBO = 256 B (8-row groups)
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128u >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(((uint32_t)ti8::RG >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
// kind::i8 instruction descriptor: D s32 (2), A/B signed int8 (1), K-major, N = 256, M = 256 (cta_group::2)
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(ti8::MMA_N >> 3) << 17) |
                              ((uint32_t)(ti8::PAIR_M >> 4) << 24);
// warp-uniform issue: the whole warp executes the stage's MMAs and commit, elect.sync picks the issuing lane (always
// lane 0, so the commit tracks that lane's MMAs); operands stay warp-uniform (no per-instruction ELECT loops).
// One K = 32 step: HH += A_hi.B_hi, X += A_hi.B_lo + A_lo.B_hi; `acc` = 0 overwrites the accumulators.
__device__ __forceinline__ void umma2_i8_kstep(uint32_t tmem, uint64_t a_h, uint64_t a_l, uint64_t b_h, uint64_t b_l,
                                               uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %7, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %2, %4, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%1], %2, %5, %6, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%1], %3, %4, %6, 1;\n\t}"
        ::"r"(tmem), "r"(tmem + 256u), "l"(a_h), "l"(a_l), "l"(b_h), "l"(b_l), "r"(kIdescI8), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void i8_commit_both_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\telect.sync _|e, 0xffffffff;\n\tmov.b16 m, 3;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}"
        ::"r"(bar) : "memory");
}
__device__ __forceinline__ void i8_cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ unsigned long long f2mul(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long swap2(unsigned long long v) { return (v >> 32) | (v << 32); }

// Q16: four magic words (atoms 0..3) -> (hi bytes, lo bytes) words, byte t = atom t
__device__ __forceinline__ void q16_pack(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, uint32_t& hi, uint32_t& lo) {
    const uint32_t p01 = __byte_perm(t0, t1, 0x5140), p23 = __byte_perm(t2, t3, 0x5140);   // [b0 b0' b1 b1']
    hi = __byte_perm(p01, p23, 0x7632);
    lo = __byte_perm(p01, p23, 0x5410) ^ 0x80808080u;
}
template <int OFF>
__device__ __forceinline__ void i8_sts(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.b32 [%0+%2], %1;" ::"r"(addr), "r"(v), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void i8_sts64(uint32_t addr, uint32_t v0, uint32_t v1) {
    asm volatile("st.shared.v2.b32 [%0+%3], {%1, %2};" ::"r"(addr), "r"(v0), "r"(v1), "n"(OFF));
}

#define I8_TMEM_LD8(taddr, r)                                                                                      \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                            \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])    \
                 : "r"(taddr))
#define I8_TMEM_LD16(taddr, r)                                                                                     \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                   "=r"(r[15])                                                                                       \
                 : "r"(taddr))

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ti8::NTHREADS, 1)
k_lattice_i8(const uint4* __restrict__ staged, int64_t N, LatticeGeom g, int64_t chunk_atoms, int tiles_k,
             float2* __restrict__ partial, int64_t frames, const float* __restrict__ fmax_dev, int dbg_flags,
             void* __restrict__ direct_out, int out_f64, int mode, BrightSink bs) {
    using namespace ti8;
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint4* aslot = reinterpret_cast<uint4*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + ASLOT_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = i8_rank();
    const int ptile = blockIdx.x >> 1;
    const int tile_h = ptile / tiles_k;
    const int64_t H0 = g.h0 + (int64_t)tile_h * PAIR_H;   // first row h of the pair tile; centre c = H0 + 127.5
    const int tk0 = (ptile % tiles_k) * TN;
    const int bk0 = tk0 + (int)rank * BK;
    const int64_t chunk = blockIdx.y, t = blockIdx.z;
    const int64_t a_begin = chunk * chunk_atoms, a_end = min(N, a_begin + chunk_atoms);
    const int n_stages = (int)((a_end - a_begin + KS - 1) / KS);
    const uint4* S = staged + t * N;
    const float F = fmax_dev ? fmaxf(*fmax_dev, 1e-30f) : 1.0f;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { i8_mbar_init(&full[s], 2 * GROUP_WARPS); i8_mbar_init(&empty[s], 1); }
        i8_mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    i8_cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == MMA_WARP) {
        // ================= MMA issuer: the leader CTA's MMA warp drives the pair (one elected lane issues) ==========
        if (rank == 0) {
            // descriptors of stage slot 0; slot s adds s * STAGE_BYTES / 16 to the 14-bit address field (no carry:
            // shared addresses < 2^18)
            const uint64_t d0 = i8_desc(su32(smem));
            constexpr uint64_t dP = (uint64_t)(PLANE >> 4), dS = (uint64_t)(STAGE_BYTES >> 4);
            for (int i = 0; i < n_stages; ++i) {
                const int s = i % STAGES;
                i8_mbar_wait(&full[s], (uint32_t)((i / STAGES) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t a_h = d0 + (uint64_t)s * dS;
#if XPCS_I8_EXPERIMENTS
                if (dbg_flags & 4) { i8_commit_both_elect(su32(&empty[s])); continue; }
#endif
#pragma unroll
                for (int ks = 0; ks < KS / 32; ++ks) {       // K = 32 per MMA: the next 32 atoms are 2 core matrices on
                    const uint64_t a = a_h + (uint64_t)(ks * 16);  // (256 B >> 4)
                    umma2_i8_kstep(tmem, a, a + dP, a + 2 * dP, a + 3 * dP, (i > 0 || ks > 0) ? 1u : 0u);
                }
                i8_commit_both_elect(su32(&empty[s]));
            }
            i8_commit_both_elect(su32(done));
        }
        __syncwarp();
    } else if (warp < NPROD_WARPS) {
        // ================= producers: group g fills stages g, g + NGROUPS, g + 2 NGROUPS, ... =================
        const int grp = warp / GROUP_WARPS, wi = warp % GROUP_WARPS;
        const int qq = lane & 3, mr = lane >> 2;
        const bool is_x = wi < GROUP_WARPS / 2;
        // AT = 4: K slice qh of the stage (atoms 16 qh + 4 qq + u); AT = 8: the warp covers the stage, the thread
        // owns atoms 8 qq + u (K half qq >> 1, octet qq & 1)
        const int qh = AT == 8 ? 0 : wi % KQ;
        const uint32_t full0 = i8_mapa(su32(full), 0);
        // every warp prefetches its own 16 atom records with cp.async into a private ring: no cross-warp barrier
        const uint32_t slot0 = su32(aslot) + (uint32_t)(warp * ASL * WSLOT * 16);
        const float invF = 1.0f / F;
        // X rows: d = i + 1/2, i = 64 rank + mr + 8 r; phase d Th_a = i Th_a + Th_a / 2 turns.  W rows: k = bk0 + mr + 8 r;
        // phase Th_0 + k Th_b + c Th_a, c Th_a = (H0 + 127) Th_a + Th_a / 2.  Th_a / 2 is taken as Th_a >> 1 on both
        // sides: the pair's phases sum to h Th_a exactly (row c - d) or to within one 2^-32 unit (row c + d).
        const uint32_t i0 = (uint32_t)((int)rank * HD + mr);
        const uint32_t cH = (uint32_t)(H0 + PAIR_H / 2 - 1);
        const uint32_t kk = (uint32_t)(g.k0 + bk0 + mr);
        const uint32_t pbase = AT == 8 ? (uint32_t)((is_x ? 0 : 2 * PLANE) + (qq >> 1) * 128 + mr * 16 + (qq & 1) * 8)
                                       : (uint32_t)((is_x ? 0 : 2 * PLANE) + qh * 128 + mr * 16 + qq * 4);
        auto prefetch = [&](int li) {   // local stage li of this group -> slot li % ASL of this warp
            const int i = grp + li * NGROUPS;
            if (i < n_stages && lane < WREC) {
                const int64_t j = a_begin + (int64_t)i * KS + WREC * qh + lane;
                const bool ok = j < a_end;
                const int unit = AT == 8 ? (lane ^ ((lane >> 3) & 3)) : (lane ^ ((lane & 8) >> 2));
                i8_cp_async16(slot0 + (uint32_t)(((li % ASL) * WSLOT + unit) * 16), S + (ok ? j : 0), ok ? 16u : 0u);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
#pragma unroll
        for (int k = 0; k < ASL - 1; ++k) prefetch(k);
        // the stage loop, specialised per warp role (no per-stage branch between the X and W paths)
        auto produce = [&](auto role) {
            constexpr bool X = decltype(role)::value;
            for (int li = 0;; ++li) {
                const int i = grp + li * NGROUPS;
                if (i >= n_stages) break;
                const int s = i % STAGES;
                asm volatile("cp.async.wait_group %0;" ::"n"(ti8::ASL - 2) : "memory");
                __syncwarp();                 // the warp's records of stage i are visible to all its lanes; every lane
                prefetch(li + ASL - 1);       // has finished reading slot (li - 1) % ASL, which is refilled now
                unsigned long long v[AT], st[AT];
                const uint32_t ra = slot0 + (uint32_t)((li % ASL) * WSLOT * 16);
#pragma unroll
                for (int u = 0; u < AT; ++u) {
                    // record AT qq + u of the warp's slot (swizzled 16-B units: conflict-free reads)
                    const uint32_t a = ra + (uint32_t)((AT == 8 ? ((8 * qq + u) ^ qq) : ((4 * qq + u) ^ (qq & 2))) * 16);
                    float s0, c0, s1, c1;
                    if (X) {
                        uint32_t tha;
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tha) : "r"(a));
                        __sincosf(turns_to_radians(i0 * tha + (tha >> 1)), &s0, &c0);
                        __sincosf(turns_to_radians(8u * tha), &s1, &c1);
                        v[u] = pack2(c0, s0);
                    } else {
                        uint32_t tha, thb, th0, fw;
                        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(tha), "=r"(thb), "=r"(th0), "=r"(fw) : "r"(a));
                        __sincosf(turns_to_radians(kk * thb + th0 + cH * tha + (tha >> 1) + GAMMA), &s0, &c0);
                        __sincosf(turns_to_radians(8u * thb), &s1, &c1);
                        const float fs = __uint_as_float(fw) * invF;
                        v[u] = pack2(fs * c0, fs * s0);
                    }
                    st[u] = pack2(c1, s1);
                }
                i8_mbar_wait(&empty[s], (uint32_t)(((i / STAGES) + 1) & 1));
#if XPCS_I8_EXPERIMENTS
                if (!(dbg_flags & 2))
#endif
                {
                    // rows m = mr + 8 r: real parts (a | wr) into rows m of the hi/lo planes, imaginary parts (b | wi)
                    // into rows 64 + m
                    const uint32_t a0 = su32(smem) + (uint32_t)(s * STAGE_BYTES) + pbase;
                    const unsigned long long QM2 = pack2(QMAGIC, QMAGIC);
#if XPCS_I8_THREE_TERM
                    // rows 0, 1 from the start phasor and one complex step; rows r + 1 = 2 cos(8 Th) X_r - X_{r-1}
                    // (Chebyshev, one packed FFMA per phasor; |U_k| <= k + 1 keeps the FP32 error < 4e-6, far below
                    // the 1.5e-5 Q16 step).  The rows are carried with signs e_r = + + - - + + - -, so the update is
                    // u_{r+1} = (e_{r+1} e_r) c2 u_r + u_{r-1} (no negation) and row r is quantised with e_r QS.
                    unsigned long long up[AT];
                    float c2[AT];
#pragma unroll
                    for (int u = 0; u < AT; ++u) c2[u] = 2.0f * lo2(st[u]);
#endif
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        uint32_t tc[AT], ts[AT];
#if XPCS_I8_THREE_TERM
                        const float er = ((r >> 1) & 1) ? -QS : QS;                       // e_r QS
                        const unsigned long long QS2 = pack2(er, er);
#else
                        const unsigned long long QS2 = pack2(QS, QS);
#endif
#pragma unroll
                        for (int u = 0; u < AT; ++u) {
                            const unsigned long long tq = ffma2(v[u], QS2, QM2);
                            tc[u] = (uint32_t)tq; ts[u] = (uint32_t)(tq >> 32);
#if XPCS_I8_THREE_TERM
                            if (r == 0) {
                                const unsigned long long cd = pack2(lo2(st[u]), lo2(st[u]));
                                const unsigned long long sd = pack2(-hi2(st[u]), hi2(st[u]));
                                up[u] = v[u];
                                v[u] = ffma2(swap2(v[u]), sd, f2mul(v[u], cd));
                            } else if (r < 7) {
                                const float k = (r & 1) ? -c2[u] : c2[u];                      // e_{r+1} e_r c2
                                const unsigned long long nv = ffma2(pack2(k, k), v[u], up[u]);
                                up[u] = v[u];
                                v[u] = nv;
                            }
#else
                            const unsigned long long cd = pack2(lo2(st[u]), lo2(st[u]));
                            const unsigned long long sd = pack2(-hi2(st[u]), hi2(st[u]));
                            v[u] = ffma2(swap2(v[u]), sd, f2mul(v[u], cd));
#endif
                        }
                        uint32_t rh, rl, ih, il;
                        q16_pack(tc[0], tc[1], tc[2], tc[3], rh, rl);
                        q16_pack(ts[0], ts[1], ts[2], ts[3], ih, il);
                        const uint32_t ad = a0 + (uint32_t)(r * RG);
                        if (AT == 8) {                        // atoms 4-7: the next word of each row, one STS.64 each
                            uint32_t rh1, rl1, ih1, il1;
                            q16_pack(tc[AT - 4], tc[AT - 3], tc[AT - 2], tc[AT - 1], rh1, rl1);
                            q16_pack(ts[AT - 4], ts[AT - 3], ts[AT - 2], ts[AT - 1], ih1, il1);
                            i8_sts64<0>(ad, rh, rh1);
                            i8_sts64<PLANE>(ad, rl, rl1);
                            i8_sts64<HALF_ROWS>(ad, ih, ih1);
                            i8_sts64<PLANE + HALF_ROWS>(ad, il, il1);
                        } else {
                            i8_sts<0>(ad, rh);
                            i8_sts<PLANE>(ad, rl);
                            i8_sts<HALF_ROWS>(ad, ih);
                            i8_sts<PLANE + HALF_ROWS>(ad, il);
                        }
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) i8_arrive_cluster(full0 + (uint32_t)(s * 8));
            }
        };
        if (is_x) produce(std::true_type{});
        else produce(std::false_type{});
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    if (warp < 8) {
        // ================= drain (warps 0-7 after production): exact int32 accumulators -> pixels ==================
        // warp w reads TMEM lane quarter w % 4 (the tcgen05.ld lane restriction): lanes 0-63 are the a rows, 64-127
        // the b rows of this CTA's 64 d; w / 4 selects the wr or wi columns.  Four rounds of 32 k: the 128 x 64
        // component tile goes through shared memory (the stage ring is free once `done` fired: every MMA has read
        // its operands), then all 256 threads combine a/b rows into the conjugate pair and write pixel rows
        // contiguously.
        const int quarter = warp & 3, part = warp >> 2;
        i8_mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16);
        const int row = quarter * 32 + lane;
        const int64_t n_q = g.n_h * g.n_k;
        float2* P = partial + (chunk * frames + t) * n_q;
        const float c_hh = (float)(65536.0 * (double)F / (32512.0 * 32512.0));   // v = (65536 HH + 256 X) F / QS^2
        const float c_x = (float)(256.0 * (double)F / (32512.0 * 32512.0));
        float* V = reinterpret_cast<float*>(smem);
        const int tid = threadIdx.x, ol = tid & 31, ow = tid >> 5;   // 0..255
        const int64_t ih_base = (int64_t)tile_h * PAIR_H + PAIR_H / 2;   // output row of h = c + 1/2
        const double F_bright = bs.count ? bright_F(bs) : 1.0;
#pragma unroll 1
        for (int kc = 0; kc < TN / 32; ++kc) {
            const uint32_t col0 = (uint32_t)(128 * (kc >> 1) + 64 * part + 32 * (kc & 1));
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
                uint32_t hh[16], xx[16];
                I8_TMEM_LD16(tb + col0 + 16 * sub, hh);
                I8_TMEM_LD16(tb + 256 + col0 + 16 * sub, xx);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    V[row * VLD + 32 * part + 16 * sub + j] = fmaf((float)(int32_t)hh[j], c_hh, (float)(int32_t)xx[j] * c_x);
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");   // drain warps 0-7 only
            const int64_t col = tk0 + 32 * kc + ol;
            if (col < g.n_k) {
#pragma unroll 2
                for (int jj = 0; jj < HD / 8; ++jj) {
                    const int dl = ow + 8 * jj;
                    const float AR = V[dl * VLD + ol], AI = V[dl * VLD + 32 + ol];
                    const float BR = V[(HD + dl) * VLD + ol], BI = V[(HD + dl) * VLD + 32 + ol];
                    const int di = (int)rank * HD + dl;
#pragma unroll
                    for (int sg = 0; sg < 2; ++sg) {
                        const int64_t ih = sg == 0 ? ih_base + di : ih_base - 1 - di;   // h = c + d, c - d
                        if (ih >= g.n_h) continue;
                        const float rr = sg == 0 ? AR - BI : AR + BI;
                        const float ri = sg == 0 ? AI + BR : AI - BR;
                        const float re = fmaf(rr, ROT_C, ri * ROT_S), im = fmaf(ri, ROT_C, -rr * ROT_S);   // q = x e^{-i Gamma}
                        const int64_t idx = ih * g.n_k + col;
                        if (direct_out == nullptr) {
                            P[idx] = make_float2(re, im);
                            continue;
                        }
                        bright_append(bs, (double)re * (double)re + (double)im * (double)im, F_bright, t * n_q + idx);
                        if (mode == 0) {
                            // single atom chunk: the fold's arithmetic for C = 1 (FP64 |p|^2 of the fp32 amplitude)
                            const double I = (double)re * (double)re + (double)im * (double)im;
                            if (out_f64) ((double*)direct_out)[t * n_q + idx] = I;
                            else ((float*)direct_out)[t * n_q + idx] = (float)I;
                        } else {
                            // the amplitude p = conj(q)
                            if (out_f64) { double* o = (double*)direct_out + 2 * (t * n_q + idx); o[0] = re; o[1] = -(double)im; }
                            else *reinterpret_cast<float2*>((float*)direct_out + 2 * (t * n_q + idx)) = make_float2(re, -im);
                        }
                    }
                }
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    i8_cluster_sync();
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    }
}

__global__ void k_absmax_f(const uint4* __restrict__ staged, int64_t n, float* __restrict__ out) {
    __shared__ float sh[256];
    float m = 0.0f;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, fabsf(__uint_as_float(staged[i].w)));
    sh[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] = fmaxf(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = sh[0];
}

cudaError_t launch_absmax_f(const uint4* staged, int64_t n, float* out, cudaStream_t s) {
    note_launch();
    k_absmax_f<<<1, 256, 0, s>>>(staged, n, out);
    return cudaGetLastError();
}

// clusters of k_lattice_i8 resident at once on the current device (one wave); sm_count / 2 if the query fails
int i8_stage_atoms() { return ti8::KS; }

int i8_cluster_slots() {
    using namespace ti8;
    static int cached[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return std::max(1, sm_count() / 2);
    if (cached[dev] > 0) return cached[dev];
    int n = 0;
    if (cudaFuncSetAttribute(k_lattice_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * 256, 1, 1);
        cfg.blockDim = dim3(NTHREADS, 1, 1);
        cfg.dynamicSmemBytes = SMEM_BYTES;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, (void*)k_lattice_i8, &cfg) != cudaSuccess) n = 0;
    }
    (void)cudaGetLastError();
    cached[dev] = n > 0 ? n : std::max(1, sm_count() / 2);
    return cached[dev];
}

cudaError_t launch_lattice_i8(const uint4* staged, int64_t N, int64_t frames, const LatticeGeom& g, int64_t chunk_atoms,
                              int64_t n_chunks, float* fmax_scratch, int uniform_f, float2* partial, cudaStream_t s,
                              void* direct_out, int out_f64, int mode, const BrightSink* bright) {
    if (direct_out && n_chunks != 1) return cudaErrorInvalidValue;
    using namespace ti8;
    if (chunk_atoms > kI8MaxChunk) return cudaErrorInvalidValue;
    const int tiles_h = (int)((g.n_h + PAIR_H - 1) / PAIR_H), tiles_k = (int)((g.n_k + TN - 1) / TN);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_lattice_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        attr = true;
    }
    const float* fm = nullptr;
    if (!uniform_f) {
        // W scale F = max |f_j| over the staged atoms of frame 0 (f is per atom, the same in every frame)
        note_launch();
        k_absmax_f<<<1, 256, 0, s>>>(staged, N, fmax_scratch);
        fm = fmax_scratch;
    }
    static int dbg = -1;
    if (dbg < 0) { const char* e = getenv("XPCS_I8_DEBUG"); dbg = e ? atoi(e) : 0; }
    dim3 grid(2 * tiles_h * tiles_k, (unsigned)n_chunks, (unsigned)frames);
    note_launch();
    k_lattice_i8<<<grid, NTHREADS, SMEM_BYTES, s>>>(staged, N, g, chunk_atoms, tiles_k, partial, frames, fm, dbg,
                                                    direct_out, out_f64, mode,
                                                    bright ? *bright : BrightSink{nullptr, nullptr, 0.0, nullptr});
    return cudaGetLastError();
}

}  // namespace xpcs
