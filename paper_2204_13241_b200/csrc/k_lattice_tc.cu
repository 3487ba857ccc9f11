// k_lattice_tc.cu -- K3: lattice-plane amplitude on the 5th-generation tensor cores (tcgen05, TMEM accumulators),
// split-FP16 operands: the precise tensor engine (per-atom form factors and the heavy kinds of species calls).
//
// The per-axis factorisation of Eq.(7) on a reciprocal-lattice plane makes the
// amplitude a matrix product over atoms.  CONJUGATE ROW PAIRS (as k_lattice_i8.cu): a cluster of 2 CTAs (one per SM)
// owns 256 consecutive rows h = c +- d around the tile centre c = H0 + 127.5 and 128 k of one frame and a chunk of
// atoms (split-K; chunks are folded in FP64 by k_amp_reduce / k_species_combine).  With X_d = e^{2 pi i d Th_a} =
// a + i b and W_k = f e^{2 pi i (Th_0 + k Th_b + c Th_a)} = wr + i wi, ONE real product [a; b] x [wr | wi]^T gives both
// rows of a pair: q(c + d) = (AR - BI) + i (AI + BR), q(c - d) = (AR + BI) + i (AI - BR), q = conj(p) (R1).
// tcgen05.mma.cta_group::2.kind::f16, M = 256 (each CTA rows [a | b] of its 64 d), N = 256 (each CTA B rows [wr | wi]
// of its 64 k), K = 16, FP32 accumulators in TMEM.
// Precision: every phasor component v is split v = hi + lo (hi on a 2^-10 grid, exact in fp16; lo = fp16(v - hi)) and
// each real product uses three MMAs (hi.hi + hi.lo + lo.hi; the dropped lo.lo term is < 2^-22 per term), i.e.
// FP32-class products (a single fp16/tf32 pass fails the 1e-3 N gate).
//
// Accumulation: the tcgen05 FP32 accumulator is not round-to-nearest (measured: the error of a TMEM accumulation
// grows linearly with its length, SURVEY A.8 / DESIGN.md "tensor accumulator"), so no TMEM accumulator ever sums
// more than SUB_STAGES * 16 = 256 atoms: two TMEM accumulators (2 x 256 columns) alternate, and while the MMA
// fills one, four drain warps add the other into round-to-nearest FP32 running sums in shared memory; at the end the
// drain warps combine the a/b rows of the sums into the conjugate pair and write the tile.
//
// One CTA per SM (TMEM 512 columns): NGROUPS producer groups of 2 warps (1 X warp, 1 W warp; group g fills stages
// g, g + NGROUPS, ... of a STAGES-deep ring of 16-atom stages; a thread owns 4 atoms x 8 rows and walks the rows
// with the angle-addition recurrence), 4 drain warps, and one warp that allocates TMEM and whose lane 0
// issues the 3 MMAs per stage.  Producer -> MMA: mbarrier full[s] (2 x 2 warp arrivals of the pair after
// fence.proxy.async); MMA -> producer: tcgen05.commit -> empty[s]; MMA -> drain: tcgen05.commit -> tfull[b];
// drain -> MMA: tempty[b] (8 arrivals).
#include "common.cuh"
#include <cuda_fp16.h>
#include <type_traits>

namespace xpcs {

namespace tc {
constexpr int HD = 64;                            // d values per CTA (the pair covers 128 d = 256 h rows)
constexpr int TM = 2 * HD, TN = 128, KS = 16;     // A rows per CTA ([a | b]), pair tile cols (k), atoms per stage
constexpr int PAIR_M = 2 * TM;                    // MMA M = 256
constexpr int PAIR_H = 4 * HD;                    // 256 output rows h per pair tile
constexpr int BN = TN / 2;                        // k per CTA; B rows per CTA: [wr | wi] = 128
#ifndef XPCS_TC_STAGES
#define XPCS_TC_STAGES 4
#endif
constexpr int STAGES = XPCS_TC_STAGES;
#ifndef XPCS_TC_SUB_STAGES
#define XPCS_TC_SUB_STAGES 16
#endif
constexpr int SUB_STAGES = XPCS_TC_SUB_STAGES;    // stages per TMEM accumulator (16 stages = 256 atoms)
constexpr int APLANE = TM * KS * 2;               // bytes per fp16 plane (128 rows x 16 atoms), A and B alike
constexpr int BPLANE = APLANE;
constexpr int HALF_ROWS = HD / 8 * 256;           // byte offset of row 64 in a plane (8-row core groups of 256 B)
constexpr int STAGE_BYTES = 2 * APLANE + 2 * BPLANE;   // A_hi A_lo | B_hi B_lo = 16 KB
constexpr int MMA_N = 2 * TN;                     // N = 256: [wr | wi] of 64 k per CTA half
#ifndef XPCS_TC_GROUPS
#define XPCS_TC_GROUPS 4
#endif
constexpr int RPT = 8, XWARPS = 1, WWARPS = 1;    // rows per producer thread; X / W warps per group
constexpr int NGROUPS = XPCS_TC_GROUPS, GROUP_WARPS = XWARPS + WWARPS;
static_assert(NGROUPS <= STAGES, "mbarrier parity: producer groups must not exceed the stage count");
constexpr int NPROD_WARPS = NGROUPS * GROUP_WARPS, NDRAIN_WARPS = 4;
// per-warp records of a stage (16 atoms); record r sits in 16-B unit r ^ ((r & 8) >> 2): conflict-free cp.async
// writes (8 lanes per phase) and per-field 32-bit reads of records {u, 4 + u, 8 + u, 12 + u}
constexpr int WREC = 16, WSLOT = WREC;
constexpr int MMA_WARP = NPROD_WARPS + NDRAIN_WARPS;
constexpr int NTHREADS = (MMA_WARP + 1) * 32;
constexpr int TMEM_COLS = 512;                    // buffer b: cols [256b, 256b+256) = [wr k<64 | wi k<64 | wr k>=64 | wi k>=64]
constexpr int SUM_LD = 129;                       // running sums [256 cols][129] fp32 (padded: conflict-free)
constexpr int SUM_BYTES = 256 * SUM_LD * 4;
#ifndef XPCS_TC_ASLOTS
#define XPCS_TC_ASLOTS 4
#endif
constexpr int ASLOTS = XPCS_TC_ASLOTS;            // cp.async prefetch ring depth (distance ASLOTS - 1 stages)
constexpr int ASLOT_BYTES = NPROD_WARPS * ASLOTS * WSLOT * 16;   // per producer warp: its stage's 16 atoms, padded
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + SUM_BYTES + ASLOT_BYTES + 1024 + 256;
static_assert(SMEM_BYTES <= 227 * 1024, "k_lattice_tc: shared memory over the 227 KB opt-in limit");
}  // namespace tc

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle: core matrix = 8 rows x 16 B contiguous (128 B);
// LBO = byte distance between the two K-adjacent core matrices, SBO = between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                      // descriptor version for tcgen05
    return d;                                     // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// kind::f16 instruction descriptor: D fp32, A/B fp16, K-major both, N = MMA_N, M = PAIR_M (cta_group::2).
__host__ __device__ constexpr uint32_t idesc_f16(bool neg_a) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((neg_a ? 1u : 0u) << 13) | ((uint32_t)(tc::MMA_N >> 3) << 17) |
           ((uint32_t)(tc::PAIR_M >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// ---- CTA-pair (cluster of 2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    // CTA-scope release (as CUTLASS's ClusterBarrier::arrive(cta_id)): a .cluster scope would emit CCTL.IVALL
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void umma2_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// warp-uniform issue of one stage: the whole warp executes it, elect.sync picks the issuing lane (always lane 0, so
// the commits track that lane's MMAs); D += A_hi.B_hi (+ A_hi.B_lo + A_lo.B_hi), commit to empty[s] (and to
// tfull[b] when bar2 != 0); operands stay warp-uniform (no per-instruction ELECT loops)
__device__ __forceinline__ void umma2_tc_stage(uint32_t d, uint64_t a_h, uint64_t a_l, uint64_t b_h, uint64_t b_l,
                                               uint32_t idesc, uint32_t first, uint32_t mma_on, uint32_t lo_on,
                                               uint32_t bar, uint32_t bar2) {
    asm volatile(
        "{\n\t.reg .pred p, e, q, l, t;\n\t.reg .b16 m;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "setp.ne.and.b32 q, %7, 0, e;\n\t"
        "setp.ne.and.b32 l, %8, 0, q;\n\t"
        "setp.ne.and.b32 t, %10, 0, e;\n\t"
        "mov.b16 m, 3;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %3, %5, p;\n\t"
        "@l tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %4, %5, 1;\n\t"
        "@l tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, 1;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%9], m;\n\t"
        "@t tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%10], m;\n\t}"
        ::"r"(d), "l"(a_h), "l"(a_l), "l"(b_h), "l"(b_l), "r"(idesc), "r"(first), "r"(mma_on), "r"(lo_on), "r"(bar),
          "r"(bar2)
        : "memory");
}
// commit to the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}

#define TMEM_LD32(taddr, r)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                            \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),         \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),   \
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), \
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])  \
        : "r"(taddr))

// byte offset of element (row m, atom a) inside one plane: [m/8][a/8][m%8][a%8] fp16
__device__ __forceinline__ uint32_t plane_off(int m, int a) {
    return (uint32_t)((m >> 3) * 256 + (a >> 3) * 128 + (m & 7) * 16 + (a & 7) * 2);
}

// ---- split-precision operand generation -------------------------------------------------------------
// hi = v rounded to the grid 2^(e-10) with the magic constant M = 1.5 * 2^(13+e) (|v| <= 2^e: hi has <= 11
// significant bits, so fp16(hi) is exact); lo = v - hi exactly (|lo| <= 2^(e-11)), then fp16(lo): the pair
// represents v to ~2^(e-22).  For W = f * cos the residual comes from one FMA of the exact product f * cos.
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint32_t pack_half2(unsigned long long v) {   // (lo, hi) fp32 -> half2 bits
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi2(v)), "f"(lo2(v)));
    return r;
}
template <int OFF>
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.b32 [%0+%2], %1;" ::"r"(addr), "r"(v), "n"(OFF));
}
// v = (v0, v1) for atoms (a, a+1); M2 = (M, M); hi -> plane P, lo -> plane P + 1
template <int OFF_HI, int OFF_LO>
__device__ __forceinline__ void split_store(uint32_t addr, unsigned long long v, unsigned long long M2) {
    const unsigned long long hi = fsub2(fadd2(v, M2), M2);
    const unsigned long long lo = fsub2(v, hi);
    sts32<OFF_HI>(addr, pack_half2(hi));
    sts32<OFF_LO>(addr, pack_half2(lo));
}
// v = f * c (pairwise) with the residual taken from the exact products
template <int OFF_HI, int OFF_LO>
__device__ __forceinline__ void split_store_f(uint32_t addr, unsigned long long f2, unsigned long long c2,
                                              unsigned long long M2) {
    const unsigned long long t = ffma2(f2, c2, M2);
    const unsigned long long hi = fsub2(t, M2);
    const unsigned long long nhi = fsub2(M2, t);                  // -hi
    unsigned long long lo;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(lo) : "l"(f2), "l"(c2), "l"(nhi));
    sts32<OFF_HI>(addr, pack_half2(hi));
    sts32<OFF_LO>(addr, pack_half2(lo));
}
// value-only variant: hi / lo half2 words of f * c (residual from the exact products)
__device__ __forceinline__ void split_vals_f(unsigned long long f2, unsigned long long c2, unsigned long long M2,
                                             uint32_t& h, uint32_t& l) {
    const unsigned long long t = ffma2(f2, c2, M2);
    const unsigned long long hi = fsub2(t, M2);
    const unsigned long long nhi = fsub2(M2, t);
    unsigned long long lo;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(lo) : "l"(f2), "l"(c2), "l"(nhi));
    h = pack_half2(hi);
    l = pack_half2(lo);
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long swap2(unsigned long long v) { return (v >> 32) | (v << 32); }
// (upper, lower) fp32 -> half2 bits, lower at the lower address
__device__ __forceinline__ uint32_t pack_h2(float upper, float lower) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(upper), "f"(lower));
    return r;
}
#ifndef XPCS_TC_ACC_TWIDDLE
#define XPCS_TC_ACC_TWIDDLE 0        // 1: accurate twiddle (error 1.4e-5 -> 9.3e-6 rms |dI|/N, 7 % slower)
#endif
// the row-step twiddle e^{-2 pi i 8 Th} of the angle-addition recurrence: its error drifts coherently along the
// rows it generates, so it is evaluated accurately (sincospif: FMA-pipe polynomial with exact reduction, ~1 ulp)
// rather than on the SFU (~2^-21)
__device__ __forceinline__ void twiddle8(uint32_t th, float& s, float& c) {
#if XPCS_TC_ACC_TWIDDLE
    // T = T_hi + T_lo (high 16 bits signed, low 16 bits): sincospif of the exactly representable 2 T_hi / 2^32,
    // then the rotation by the small angle t = 2 pi T_lo / 2^32 < 1e-4 rad (cos t = 1 - t^2 / 2, sin t = t; the
    // dropped terms are < 2e-13)
    const uint32_t T = 8u * th;
    float sh, ch;
    sincospif((float)(int32_t)(T & 0xFFFF0000u) * 4.656612873077393e-10f, &sh, &ch);   // 2^-31
    const float t = (float)(T & 0xFFFFu) * 1.4629180792671596e-09f;                      // 2 pi / 2^32
    const float cl = fmaf(-0.5f * t, t, 1.0f);
    c = fmaf(ch, cl, -sh * t);
    s = fmaf(sh, cl, ch * t);
#else
    __sincosf(turns_to_radians(8u * th), &s, &c);
#endif
}
template <int OFF>
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.b32 [%0+%3], {%1, %2};" ::"r"(addr), "r"(a), "r"(b), "n"(OFF));
}
// M = 1.5 * 2^(13 + e), e = max(0, exponent bound of |f|) so that |f| <= 2^e
__device__ __forceinline__ float split_magic(float f) {
    const int ef = (int)((__float_as_uint(f) >> 23) & 0xFF);
    const int e = max(0, ef - 126);
    return __uint_as_float(((uint32_t)(140 + e) << 23) | 0x00400000u);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc::NTHREADS, 1)
k_lattice_tc(const uint4* __restrict__ staged, int64_t N, LatticeGeom g, int64_t chunk_atoms, int tiles_k,
             float2* __restrict__ partial, int64_t frames, int dbg_flags) {
    using namespace tc;
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* sums = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);
    uint4* aslot = reinterpret_cast<uint4*>(smem + STAGES * STAGE_BYTES + SUM_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + SUM_BYTES + ASLOT_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();                  // 0 = leader (issues the pair's MMAs)
    const int ptile = blockIdx.x >> 1;                     // pair tile: 256 h x 128 k
    const int tile_h = ptile / tiles_k;
    const int64_t H0 = g.h0 + (int64_t)tile_h * PAIR_H;    // first row h of the pair tile; centre c = H0 + 127.5
    const int tk0 = (ptile % tiles_k) * TN;                // the pair's 128 k columns
    const int bk0 = tk0 + (int)rank * BN;                  // this CTA's 64 k rows of B
    const int64_t chunk = blockIdx.y, t = blockIdx.z;
    const int64_t a_begin = chunk * chunk_atoms, a_end = min(N, a_begin + chunk_atoms);
    const int n_stages = (int)((a_end - a_begin + KS - 1) / KS);
    const int n_sub = (n_stages + SUB_STAGES - 1) / SUB_STAGES;
    const uint4* S = staged + t * N;

    if (threadIdx.x == 0) {
        // in the leader: full[s] counts the producer warps of one group in both CTAs, tempty[b] the drain warps
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 2 * GROUP_WARPS); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 2 * NDRAIN_WARPS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == MMA_WARP) {
        // ================= MMA issuer: the leader CTA's MMA warp drives the pair (one elected lane issues) ==========
        if (rank == 0) {
            const uint32_t idesc = idesc_f16(false);
            const uint32_t lo_on = dbg_flags & 1 ? 0u : 1u;   // experiments: bit 0 drops the hi.lo / lo.hi products
            // descriptors of stage slot 0; slot s adds s * STAGE_BYTES / 16 to the 14-bit address field
            const uint64_t d0 = umma_desc(smem_u32(smem), 128, 256);
            constexpr uint64_t dP = (uint64_t)(APLANE >> 4), dS = (uint64_t)(STAGE_BYTES >> 4);
            for (int i = 0; i < n_stages; ++i) {
                const int s = i % STAGES;
                const int u = i / SUB_STAGES, b = u & 1;
                const bool sub_first = (i % SUB_STAGES) == 0;
                if (sub_first && !(dbg_flags & 8)) {   // accumulator b must have been drained by both CTAs (use u - 2)
                    mbar_wait_cluster(&tempty[b], (uint32_t)(((u >> 1) + 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                mbar_wait_cluster(&full[s], (uint32_t)((i / STAGES) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t a_h = d0 + (uint64_t)s * dS;
                const uint32_t d = tmem + (uint32_t)(b * 256);
                const uint32_t first = sub_first ? 0u : 1u;
                const bool last_sub = (i % SUB_STAGES) == SUB_STAGES - 1 || i == n_stages - 1;
                // experiments: bit 2 skips the MMAs (producer/drain cost alone)
                umma2_tc_stage(d, a_h, a_h + dP, a_h + 2 * dP, a_h + 3 * dP, idesc, first, (dbg_flags & 4) ? 0u : 1u,
                               lo_on, smem_u32(&empty[s]), last_sub ? smem_u32(&tfull[b]) : 0u);
            }
        }
        __syncwarp();
    } else if (warp < NPROD_WARPS) {
        // ================= phasor producers: group g fills stages g, g + NGROUPS, ...  A thread owns 4 atoms (one
        // 8-byte half2 pair per row and plane, STS.64) and 8 rows spaced 8 apart, walked with the angle-addition
        // recurrence (2 sincos per atom per stage, 2 packed ops per phasor); split into fp16 hi/lo with magic
        // numbers (3 packed ops per phasor) and packed with cvt.f16x2.  Lanes (quad qq, row mr): conflict-free.
        const int grp = warp / GROUP_WARPS, wi = warp % GROUP_WARPS;
        // lanes: each half-warp owns one 128-B K half of a row group (qq in {0,1} | {2,3}, mr 0..7), so the
        // STS.64 of a half-warp phase covers 128 contiguous bytes (no bank conflict between the K halves)
        const int qq = (lane & 1) | ((lane >> 4) << 1), mr = (lane >> 1) & 7;
        const bool is_x = wi < XWARPS;
        const uint32_t slot0 = smem_u32(aslot) + (uint32_t)(warp * ASLOTS * WSLOT * 16);
        const uint32_t full0 = mapa(smem_u32(full), 0);
        // X rows: d = i + 1/2, i = 64 rank + mr + 8 r, phase d Th_a = i Th_a + Th_a / 2 turns; W rows: k = bk0 + mr + 8 r,
        // phase Th_0 + k Th_b + c Th_a, c Th_a = (H0 + 127) Th_a + Th_a / 2 (Th_a / 2 taken as Th_a >> 1 on both sides:
        // the pair's phases sum to h Th_a exactly or to within one 2^-32 unit)
        const uint32_t i0 = (uint32_t)((int)rank * HD + mr);
        const uint32_t cH = (uint32_t)(H0 + PAIR_H / 2 - 1);
        const uint32_t kk = (uint32_t)(g.k0 + bk0 + mr);
        auto prefetch = [&](int li) {
            const int i = grp + li * NGROUPS;
            if (i < n_stages && lane < WREC) {
                const int64_t j = a_begin + (int64_t)i * KS + lane;
                const bool ok = j < a_end;
                cp_async16(slot0 + (uint32_t)(((li % ASLOTS) * WSLOT + (lane ^ ((lane & 8) >> 2))) * 16), S + (ok ? j : 0),
                           ok ? 16u : 0u);
            }
            cp_async_commit();
        };
#pragma unroll
        for (int k = 0; k < ASLOTS - 1; ++k) prefetch(k);
        const unsigned long long MX2 = pack2(12288.0f, 12288.0f);             // |X| <= 1: hi on the 2^-10 grid
        // byte offset of (row m, quad qq) in a plane: [m/8][qq/2][m%8][qq%2 * 8 B]
        const uint32_t qoff = (uint32_t)((qq >> 1) * 128 + mr * 16 + (qq & 1) * 8);
        // the stage loop, specialised per warp role (no per-stage branch between the X and W paths)
        auto produce = [&](auto role) {
            constexpr bool X = decltype(role)::value;
            for (int li = 0;; ++li) {
                const int i = grp + li * NGROUPS;
                if (i >= n_stages) break;
                const int s = i % STAGES;
                cp_async_wait<ASLOTS - 2>();
                __syncwarp();
                prefetch(li + ASLOTS - 1);
                unsigned long long v[4], st[4], f2[4];
                float fm = 0.f;
                const uint32_t ra = slot0 + (uint32_t)((li % ASLOTS) * WSLOT * 16);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t a = ra + (uint32_t)((((4 * qq + u) ^ (qq & 2))) * 16);   // record 4 qq + u
                    float s0, c0, s1, c1;
                    if (X) {
                        uint32_t tha;
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tha) : "r"(a));
                        __sincosf(turns_to_radians(i0 * tha + (tha >> 1)), &s0, &c0);
                        twiddle8(tha, s1, c1);
                    } else {
                        uint32_t tha, thb, th0, fw;
                        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(tha), "=r"(thb), "=r"(th0), "=r"(fw) : "r"(a));
                        __sincosf(turns_to_radians(kk * thb + th0 + cH * tha + (tha >> 1)), &s0, &c0);
                        twiddle8(thb, s1, c1);
                        const float fj = __uint_as_float(fw);             // padding atoms: f = 0 -> W = 0
                        f2[u] = pack2(fj, fj);
                        fm = fmaxf(fm, fabsf(fj));
                    }
                    v[u] = pack2(c0, s0);
                    st[u] = pack2(c1, s1);
                }
                mbar_wait(&empty[s], (uint32_t)(((i / STAGES) + 1) & 1));
                const uint32_t sbase = smem_u32(smem) + (uint32_t)(s * STAGE_BYTES);
                {
                    // rows m = mr + 8 r: real parts (a | wr) into rows m of the hi/lo planes, imaginary parts (b | wi)
                    // into rows 64 + m
                    const uint32_t a0 = sbase + (X ? 0u : (uint32_t)(2 * APLANE)) + qoff;
                    const unsigned long long M2 = X ? MX2 : pack2(split_magic(fm), split_magic(fm));
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        unsigned long long hi[4], lo[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (X) {
                                hi[u] = fsub2(fadd2(v[u], M2), M2);               // (c_hi, s_hi), exact in fp16
                                lo[u] = fsub2(v[u], hi[u]);                        // (c_lo, s_lo)
                            } else {
                                const unsigned long long tt = ffma2(f2[u], v[u], M2);
                                hi[u] = fsub2(tt, M2);                             // f (c, s) hi
                                lo[u] = ffma2(f2[u], v[u], fsub2(M2, tt));         // f (c, s) - hi, from the exact product
                            }
                            const unsigned long long cd = pack2(lo2(st[u]), lo2(st[u]));
                            const unsigned long long sd = pack2(-hi2(st[u]), hi2(st[u]));
                            v[u] = ffma2(swap2(v[u]), sd, fmul2(v[u], cd));
                        }
                        const uint32_t ad = a0 + (uint32_t)(r * 256);
                        sts64<0>(ad, pack_h2(lo2(hi[1]), lo2(hi[0])), pack_h2(lo2(hi[3]), lo2(hi[2])));                    // re hi
                        sts64<APLANE>(ad, pack_h2(lo2(lo[1]), lo2(lo[0])), pack_h2(lo2(lo[3]), lo2(lo[2])));               // re lo
                        sts64<HALF_ROWS>(ad, pack_h2(hi2(hi[1]), hi2(hi[0])), pack_h2(hi2(hi[3]), hi2(hi[2])));            // im hi
                        sts64<APLANE + HALF_ROWS>(ad, pack_h2(hi2(lo[1]), hi2(lo[0])), pack_h2(hi2(lo[3]), hi2(lo[2])));   // im lo
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> async proxy
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(full0 + (uint32_t)(s * 8));   // the leader's full[s]
            }
        };
        if (is_x) produce(std::true_type{});
        else produce(std::false_type{});
        cp_async_wait<0>();
    } else {
        // ================= drain warps: TMEM accumulator -> RN fp32 running sums (smem) -> tile =================
        const int quarter = warp & 3;               // TMEM lanes 32*quarter .. +31 = rows of this CTA's half
        const int r = quarter * 32 + lane;
        const uint32_t tempty0 = mapa(smem_u32(tempty), 0);
        for (int c = 0; c < 256; ++c) sums[c * SUM_LD + r] = 0.f;
        for (int u = 0; u < ((dbg_flags & 8) ? 0 : n_sub); ++u) {   // experiments: bit 3 skips the drain
            const int b = u & 1;
            mbar_wait_cluster(&tfull[b], (uint32_t)((u >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * 256);
            uint32_t v[2][32];
#pragma unroll
            for (int blk = 0; blk < 8; blk += 2) {
#pragma unroll
                for (int q = 0; q < 2; ++q) TMEM_LD32(tb + (uint32_t)((blk + q) * 32), v[q]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (blk == 6) {   // all of accumulator b has been read: hand it back to the leader's MMA
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty0 + (uint32_t)(b * 8));
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    float* col = sums + ((blk + q) * 32) * SUM_LD + r;
                    float acc[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) acc[c] = col[c * SUM_LD];
#pragma unroll
                    for (int c = 0; c < 32; ++c) col[c * SUM_LD] = acc[c] + __uint_as_float(v[q][c]);
                }
            }
        }
        // ---- conjugate-pair combination and the tile write: this CTA's 64 d give output rows h = c + d and c - d
        // (partial[chunk][t][ih][ik] = q, coalesced along k).  sums column of (k, comp): 128 (k / 64) + 64 comp + k % 64
        asm volatile("bar.sync 1, 128;" ::: "memory");   // the four drain warps' running sums are complete
        const int64_t n_q = g.n_h * g.n_k;
        float2* P = partial + (chunk * frames + t) * n_q;
        const int64_t ih_base = (int64_t)tile_h * PAIR_H + PAIR_H / 2;   // output row of h = c + 1/2
        for (int dl = quarter; dl < HD; dl += 4) {
            const int di = (int)rank * HD + dl;
            const int64_t ihp = ih_base + di, ihm = ih_base - 1 - di;
#pragma unroll
            for (int j = 0; j < TN / 32; ++j) {
                const int c = lane + 32 * j;
                const int64_t ik = tk0 + c;
                const int cr = 128 * (c >> 6) + (c & 63), ci = cr + 64;
                const float AR = sums[cr * SUM_LD + dl], AI = sums[ci * SUM_LD + dl];
                const float BR = sums[cr * SUM_LD + HD + dl], BI = sums[ci * SUM_LD + HD + dl];
                if (ik < g.n_k) {
                    if (ihp < g.n_h) P[ihp * g.n_k + ik] = make_float2(AR - BI, AI + BR);
                    if (ihm < g.n_h) P[ihm * g.n_k + ik] = make_float2(AR + BI, AI - BR);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    }
}

bool lattice_tc_supported(const LatticeGeom& g) {
    static int ok = -1;
    if (ok < 0) {
        int dev = 0, major = 0, minor = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        ok = (major == 10 && minor == 0) ? 1 : 0;
        const char* env = getenv("XPCS_DISABLE_TC");
        if (env && env[0] == '1') ok = 0;
    }
    (void)g;
    return ok == 1;
}

cudaError_t launch_lattice_tc(const uint4* staged, int64_t N, int64_t frames, const LatticeGeom& g,
                              int64_t chunk_atoms, int64_t n_chunks, float2* partial, cudaStream_t s) {
    using namespace tc;
    const int tiles_h = (int)((g.n_h + PAIR_H - 1) / PAIR_H), tiles_k = (int)((g.n_k + TN - 1) / TN);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_lattice_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        attr = true;
    }
    dim3 grid(2 * tiles_h * tiles_k, (unsigned)n_chunks, (unsigned)frames);   // 2 CTAs (one cluster) per pair tile
    note_launch();
    static int dbg = -1;
    if (dbg < 0) { const char* e = getenv("XPCS_TC_DEBUG"); dbg = e ? atoi(e) : 0; }
    k_lattice_tc<<<grid, NTHREADS, SMEM_BYTES, s>>>(staged, N, g, chunk_atoms, tiles_k, partial, frames, dbg);
    return cudaGetLastError();
}

}  // namespace xpcs
