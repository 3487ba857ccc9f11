// k_lattice_i8.cu -- K3b: lattice-plane amplitude on the tcgen05 INTEGER tensor cores (kind::i8, exact int32
// accumulation in TMEM), the fast engine for uniform form factors.
//
// Same factorisation as k_lattice_tc.cu (Eq. 7, on a reciprocal-lattice plane):
//     p^e(h,k) = sum_j X_h(j) W_k(j),  X_h = e^{-2 pi i h Th_a(j)},  W_k = (f_j / F) e^{-2 pi i (Th_0 + k Th_b)(j)}
// with F = max_j |f_j|.  Every phasor component v in [-1, 1] is written as two int8 limbs (Q16, the default):
//     x = rint(32512 v) = 256 hi + lo,  hi = round(x / 256) in [-127, 127],  lo in [-128, 127]
// (|v - x / 32512| <= 1 / 65024 = 1.54e-5).  One FFMA t = fma(v, 32512, 1.5 * 2^23 + 128) leaves y = x + 128 in the
// low 16 bits of t: byte 1 = hi, byte 0 = lo + 128, so both limbs come from one instruction and two byte permutes.
// Each real product is
//     v w ~ [65536 hi.hi' + 256 (hi.lo' + lo.hi')] / 32512^2      (the dropped lo.lo' term is <= 1.55e-5, zero-mean)
// i.e. three int8 MMAs into two TMEM accumulators, HH = sum hi.hi' and X = sum (hi.lo' + lo.hi').  The integer
// accumulation is EXACT (no TMEM rounding, unlike the FP32 accumulator of the split-FP16 engine), so
// a chunk of up to 32768 atoms (int32 overflow bound: 4 x 127 x 128 x 32768 < 2^31) accumulates in TMEM and is
// drained once; the result carries only the limb quantisation error (rms |dI| ~ 3e-5 N per pixel for f = 1,
// DESIGN.md 6.3).  XPCS_I8_Q16=0 builds the previous base-254 limbs (hi = rint(127 v), lo = rint(254 (127 v - hi)),
// v ~ (254 hi + lo) / 32258, three magic-number FFMAs per component; kept for comparison).
// The int8 tensor rate is twice the fp16 rate on sm_100a (measured 8192 vs 4096 MAC/clk/SM, tools/mma_rate.cu).
//
// CTA pair (cluster of 2, cta_group::2): 256 (h) x 128 (k) pixel tile, M = 256, N = 256 ([Re | Im'] of 64 k per CTA
// half, B rows [-Ws | Wr | Ws]), K = 32 atoms per stage, 6 MMAs per stage:
//     HH += Xr_hi.B1_hi + Xs_hi.B2_hi,   X += Xr_hi.B1_lo + Xr_lo.B1_hi + Xs_hi.B2_lo + Xs_lo.B2_hi
// (B1 = [Wr | Ws], B2 = [-Ws | Wr]: D = [Re | Im'], Im' = -Im; the partials hold conj(p) like the fp16 engine).
//
// Producers: 5 groups of 6 warps; group g fills stages i = g mod 5 (6-stage ring, 28 KB per stage; the group count
// must not exceed the stage count, see the empty-barrier parity note in DESIGN.md 6.1).  A warp thread
// owns 4 consecutive atoms (one 32-bit word per row and limb plane) and 8 rows spaced 8 apart (X or W), and walks
// the rows with the angle-addition recurrence X_{m+8} = X_m X_8 (packed FP32x2, 2 ops per phasor; 2 SFU sincos per
// atom per thread), quantises with one packed magic-number FFMA per phasor (Q16) and packs limb bytes with PRMT.
// Lanes (quad qq, row mr) write 32 distinct banks per store.  After the last stage, warps 0-7 (two per TMEM lane
// quarter, splitting the columns) wait for the final MMA commit and drain both accumulators,
// p = (65536 HH + 256 X) F / 32512^2 (Q16), through a shared-memory tile into row-contiguous global writes: the
// partial amplitude, or with a single atom chunk the final I = |p|^2 (or p) itself.
#include "common.cuh"

namespace xpcs {

namespace ti8 {
constexpr int TM = 128, TN = 128, KS = 32;          // rows (h) per CTA, pair tile cols (k), atoms per stage
constexpr int PAIR_M = 2 * TM;
constexpr int BN = TN / 2;                          // k rows of B per CTA
constexpr int APLANE = TM * KS;                     // int8 A plane: 128 rows x 32 atoms = 4 KB
constexpr int BROWS = 3 * BN;                       // [-Ws | Wr | Ws]
constexpr int BPLANE = BROWS * KS;                  // 6 KB
constexpr int STAGE_BYTES = 4 * APLANE + 2 * BPLANE;   // Xr_hi Xr_lo Xs_hi Xs_lo | B_hi B_lo = 28 KB
#ifndef XPCS_I8_STAGES
#define XPCS_I8_STAGES 6
#endif
constexpr int STAGES = XPCS_I8_STAGES;
#ifndef XPCS_I8_GROUPS
#define XPCS_I8_GROUPS 5
#endif
constexpr int NGROUPS = XPCS_I8_GROUPS, GROUP_WARPS = 6;   // per group: 4 X warps (2 quad halves x 2 row halves), 2 W warps
constexpr int NPROD_WARPS = NGROUPS * GROUP_WARPS;  // 30
constexpr int MMA_WARP = NPROD_WARPS;               // producer warps 0-7 (two per TMEM lane quarter) also drain the tile
constexpr int NTHREADS = (MMA_WARP + 1) * 32;       // 992
constexpr int MMA_N = 2 * TN;                       // 256
constexpr int TMEM_COLS = 512;                      // HH cols [0, 256), X cols [256, 512)
constexpr int ASL = 4;                              // atom-record slots per warp (cp.async prefetch distance ASL - 1)
constexpr int WREC = 16;                            // records a producer warp needs per stage (its 4 atom quads)
// record r of a warp's stage sits in 16-B unit r ^ ((r & 8) >> 2) of its slot: the cp.async writes (8 lanes per
// phase, records 0-7 / 8-15) and the per-field 32-bit reads of records {u, 4 + u, 8 + u, 12 + u} (one per quad)
// both hit distinct banks, one wavefront per instruction
constexpr int WSLOT = WREC;
constexpr int ASLOT_BYTES = NPROD_WARPS * ASL * WSLOT * 16;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + ASLOT_BYTES + 1024 + 256;
constexpr float MAGIC = 12582912.0f;                // 1.5 * 2^23
#ifndef XPCS_I8_Q16
#define XPCS_I8_Q16 1
#endif
// Q16 limbs: x = rint(QS v) in [-QS, QS], x = 256 hi + lo with hi in [-127, 127], lo in [-128, 127]; one FFMA
// t = fma(v, QS, M + 128) holds y = x + 128 in its low 16 bits: byte 1 = hi, byte 0 = lo + 128 (= lo ^ 0x80)
constexpr float QS = 32512.0f;
constexpr float QMAGIC = MAGIC + 128.0f;
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
    d |= (uint64_t)((256u >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
// kind::i8 instruction descriptor: D s32 (2), A/B signed int8 (1), K-major, N = 256, M = 256 (cta_group::2)
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(ti8::MMA_N >> 3) << 17) |
                              ((uint32_t)(ti8::PAIR_M >> 4) << 24);
__device__ __forceinline__ void umma2_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdescI8), "r"(acc));
}
__device__ __forceinline__ void i8_commit_both(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            su32(bar))
        : "memory");
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

#if !XPCS_I8_Q16
// (c, s) -> limb magic floats: t1 = M + hi (low byte = hi), t2 = M + lo (low byte = lo), element-wise on (c, s).
// u = M - 254 hi is exact (an integer < 2^24); t2 = fl(32258 v + u) rounds once to the integer grid of M, so
// t2 = M + rint(32258 v - 254 hi) = M + lo with |lo| <= 127 (|32258 v - 254 hi| = 254 |127 v - hi| <= 127).
__device__ __forceinline__ void quantise(unsigned long long v, unsigned long long& t1, unsigned long long& t2) {
    t1 = ffma2(v, pack2(127.0f, 127.0f), pack2(ti8::MAGIC, ti8::MAGIC));          // M + rint(127 v)
    const unsigned long long u = ffma2(t1, pack2(-254.0f, -254.0f),
                                       pack2(255.0f * ti8::MAGIC, 255.0f * ti8::MAGIC));   // = M - 254 hi (exact)
    t2 = ffma2(v, pack2(32258.0f, 32258.0f), u);                                  // M + lo
}
// low bytes of four 32-bit words -> one word (byte t = atom t)
__device__ __forceinline__ uint32_t pack_bytes(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
#endif
// Q16: four magic words (atoms 0..3) -> (hi bytes, lo bytes) words, byte t = atom t
__device__ __forceinline__ void q16_pack(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, uint32_t& hi, uint32_t& lo) {
    const uint32_t p01 = __byte_perm(t0, t1, 0x5140), p23 = __byte_perm(t2, t3, 0x5140);   // [b0 b0' b1 b1']
    hi = __byte_perm(p01, p23, 0x7632);
    lo = __byte_perm(p01, p23, 0x5410) ^ 0x80808080u;
}
#if !XPCS_I8_Q16
// per-byte two's-complement negation of four int8 in [-127, 127]
__device__ __forceinline__ uint32_t neg_bytes(uint32_t w) {
    const uint32_t n = ~w;
    return ((n & 0x7F7F7F7Fu) + 0x01010101u) ^ (n & 0x80808080u);
}
#endif
template <int OFF>
__device__ __forceinline__ void i8_sts(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.b32 [%0+%2], %1;" ::"r"(addr), "r"(v), "n"(OFF));
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
             void* __restrict__ direct_out, int out_f64, int mode) {
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
    const int th0 = (ptile / tiles_k) * PAIR_M + (int)rank * TM;
    const int tk0 = (ptile % tiles_k) * TN;
    const int bk0 = tk0 + (int)rank * BN;
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
        // ================= MMA issuer: one lane of the leader CTA drives the pair =================
        if (rank == 0 && lane == 0) {
            const uint32_t base = su32(smem);
            for (int i = 0; i < n_stages; ++i) {
                const int s = i % STAGES;
                i8_mbar_wait(&full[s], (uint32_t)((i / STAGES) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t sb = base + s * STAGE_BYTES;
                const uint64_t xr_h = i8_desc(sb), xr_l = i8_desc(sb + APLANE);
                const uint64_t xs_h = i8_desc(sb + 2 * APLANE), xs_l = i8_desc(sb + 3 * APLANE);
                const uint32_t bh = sb + 4 * APLANE, bl = bh + BPLANE;
                const uint64_t b1_h = i8_desc(bh + BN * KS), b1_l = i8_desc(bl + BN * KS);
                const uint64_t b2_h = i8_desc(bh), b2_l = i8_desc(bl);
                const uint32_t acc = i > 0 ? 1u : 0u;
                if (!(dbg_flags & 4)) {
                    umma2_i8(tmem, xr_h, b1_h, acc);
                    umma2_i8(tmem, xs_h, b2_h, 1);
                    umma2_i8(tmem + 256, xr_h, b1_l, acc);
                    umma2_i8(tmem + 256, xr_l, b1_h, 1);
                    umma2_i8(tmem + 256, xs_h, b2_l, 1);
                    umma2_i8(tmem + 256, xs_l, b2_h, 1);
                }
                i8_commit_both(&empty[s]);
            }
            i8_commit_both(done);
        }
        __syncwarp();
    } else if (warp < NPROD_WARPS) {
        // ================= producers: group g fills stages g, g + NGROUPS, g + 2 NGROUPS, ... =================
        const int grp = warp / GROUP_WARPS, wi = warp % GROUP_WARPS;
        const int qq = lane & 3, mr = lane >> 2;
        const bool is_x = wi < 4;
        const int qh = is_x ? (wi & 1) : wi - 4;              // quad half (K bytes 0-15 or 16-31 of the stage)
        const int rh = wi >> 1;                               // X warps: row half (rows mr + 8 r, r in [8 rh, 8 rh + 8))
        const uint32_t full0 = i8_mapa(su32(full), 0);
        // every warp prefetches its own 16 atom records (atoms 16 qh .. 16 qh + 15 of each of its stages) with
        // cp.async into a private ring: no cross-warp barrier per stage
        const uint32_t slot0 = su32(aslot) + (uint32_t)(warp * ASL * WSLOT * 16);
        const float invF = 1.0f / F;
        auto prefetch = [&](int li) {   // local stage li of this group -> slot li % ASL of this warp
            const int i = grp + li * NGROUPS;
            if (i < n_stages && lane < WREC) {
                const int64_t j = a_begin + (int64_t)i * KS + WREC * qh + lane;
                const bool ok = j < a_end;
                i8_cp_async16(slot0 + (uint32_t)(((li % ASL) * WSLOT + (lane ^ ((lane & 8) >> 2))) * 16), S + (ok ? j : 0),
                              ok ? 16u : 0u);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
#pragma unroll
        for (int k = 0; k < ASL - 1; ++k) prefetch(k);
        for (int li = 0;; ++li) {
            const int i = grp + li * NGROUPS;
            if (i >= n_stages) break;
            const int s = i % STAGES;
            asm volatile("cp.async.wait_group %0;" ::"n"(ti8::ASL - 2) : "memory");
            __syncwarp();                 // the warp's records of stage i are visible to all its lanes; every lane has
            prefetch(li + ASL - 1);       // finished reading slot (li - 1) % ASL, which is refilled now
            uint4 at[4];
            {
                // only the fields this warp uses: X warps Th_a, W warps (Th_b, Th_0, f)
                const uint32_t ra = slot0 + (uint32_t)((li % ASL) * WSLOT * 16);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t a = ra + (uint32_t)((((4 * qq + u) ^ (qq & 2))) * 16);   // record 4 qq + u
                    if (is_x) {
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(at[u].x) : "r"(a));
                        at[u].y = at[u].z = at[u].w = 0u;
                    } else {
                        at[u].x = 0u;
                        asm volatile("ld.shared.u32 %0, [%1+4];" : "=r"(at[u].y) : "r"(a));
                        asm volatile("ld.shared.u32 %0, [%1+8];" : "=r"(at[u].z) : "r"(a));
                        asm volatile("ld.shared.u32 %0, [%1+12];" : "=r"(at[u].w) : "r"(a));
                    }
                }
            }
            i8_mbar_wait(&empty[s], (uint32_t)(((i / STAGES) + 1) & 1));
            const uint32_t sbase = su32(smem) + (uint32_t)(s * STAGE_BYTES);
            if (!(dbg_flags & 2)) {
                if (is_x) {
                    // X rows m = mr + 8 r (8 rh <= r < 8 rh + 8) of this CTA's 128: X_m = e^{-2 pi i h Th_a}, h = h0 + th0 + m
                    const uint32_t h = (uint32_t)(g.h0 + th0 + mr + 64 * rh);
                    unsigned long long v[4], st[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float s0, c0, s1, c1;
                        __sincosf(turns_to_radians(h * at[u].x), &s0, &c0);
                        __sincosf(turns_to_radians(8u * at[u].x), &s1, &c1);
                        v[u] = pack2(c0, s0);
                        st[u] = pack2(c1, s1);
                    }
                    const uint32_t a0 = sbase + (uint32_t)(qh * 128 + mr * 16 + qq * 4 + rh * 8 * 256);
#if XPCS_I8_Q16
                    const unsigned long long QS2 = pack2(QS, QS), QM2 = pack2(QMAGIC, QMAGIC);
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        uint32_t tc[4], ts[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const unsigned long long tq = ffma2(v[u], QS2, QM2);
                            tc[u] = (uint32_t)tq; ts[u] = (uint32_t)(tq >> 32);
                            const unsigned long long cd = pack2(lo2(st[u]), lo2(st[u]));
                            const unsigned long long sd = pack2(-hi2(st[u]), hi2(st[u]));
                            v[u] = ffma2(swap2(v[u]), sd, f2mul(v[u], cd));
                        }
                        uint32_t xrh, xrl, xsh, xsl;
                        q16_pack(tc[0], tc[1], tc[2], tc[3], xrh, xrl);
                        q16_pack(ts[0], ts[1], ts[2], ts[3], xsh, xsl);
                        const uint32_t ad = a0 + (uint32_t)(r * 256);
                        i8_sts<0 * APLANE>(ad, xrh);
                        i8_sts<1 * APLANE>(ad, xrl);
                        i8_sts<2 * APLANE>(ad, xsh);
                        i8_sts<3 * APLANE>(ad, xsl);
                    }
#else
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        uint32_t hc[4], lc[4], hs[4], ls[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            unsigned long long t1, t2;
                            quantise(v[u], t1, t2);
                            hc[u] = (uint32_t)t1; hs[u] = (uint32_t)(t1 >> 32);
                            lc[u] = (uint32_t)t2; ls[u] = (uint32_t)(t2 >> 32);
                            // angle addition: (c, s) <- (c cd - s sd, s cd + c sd)
                            const unsigned long long cd = pack2(lo2(st[u]), lo2(st[u]));
                            const unsigned long long sd = pack2(-hi2(st[u]), hi2(st[u]));
                            v[u] = ffma2(swap2(v[u]), sd, f2mul(v[u], cd));
                        }
                        const uint32_t ad = a0 + (uint32_t)(r * 256);
                        i8_sts<0 * APLANE>(ad, pack_bytes(hc[0], hc[1], hc[2], hc[3]));
                        i8_sts<1 * APLANE>(ad, pack_bytes(lc[0], lc[1], lc[2], lc[3]));
                        i8_sts<2 * APLANE>(ad, pack_bytes(hs[0], hs[1], hs[2], hs[3]));
                        i8_sts<3 * APLANE>(ad, pack_bytes(ls[0], ls[1], ls[2], ls[3]));
                    }
#endif
                } else {
                    // W rows k = mr + 8 r (r < 8) of this CTA's 64: W_k = (f / F) e^{-2 pi i (Th_0 + kk Th_b)}
                    const uint32_t kk = (uint32_t)(g.k0 + bk0 + mr);
                    unsigned long long v[4], st[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float s0, c0, s1, c1;
                        __sincosf(turns_to_radians(at[u].z + kk * at[u].y), &s0, &c0);
                        __sincosf(turns_to_radians(8u * at[u].y), &s1, &c1);
                        const float fs = __uint_as_float(at[u].w) * invF;
                        v[u] = pack2(fs * c0, fs * s0);
                        st[u] = pack2(c1, s1);
                    }
                    const uint32_t a0 = sbase + (uint32_t)(4 * APLANE + qh * 128 + mr * 16 + qq * 4);
#if XPCS_I8_Q16
                    const unsigned long long QS2 = pack2(QS, QS), QM2 = pack2(QMAGIC, QMAGIC);
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        uint32_t tc[4], ts[4], tn[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const unsigned long long tq = ffma2(v[u], QS2, QM2);
                            tc[u] = (uint32_t)tq; ts[u] = (uint32_t)(tq >> 32);
                            // -Ws limbs from rint(-QS s) = -rint(QS s) (lo = -128 has no int8 negation)
                            tn[u] = __float_as_uint(fmaf(hi2(v[u]), -QS, QMAGIC));
                            const unsigned long long cd = pack2(lo2(st[u]), lo2(st[u]));
                            const unsigned long long sd = pack2(-hi2(st[u]), hi2(st[u]));
                            v[u] = ffma2(swap2(v[u]), sd, f2mul(v[u], cd));
                        }
                        uint32_t whr, wlr, whs, wls, nhs, nls;
                        q16_pack(tc[0], tc[1], tc[2], tc[3], whr, wlr);
                        q16_pack(ts[0], ts[1], ts[2], ts[3], whs, wls);
                        q16_pack(tn[0], tn[1], tn[2], tn[3], nhs, nls);
                        const uint32_t ad = a0 + (uint32_t)(r * 256);
                        // B rows: -Ws at k, Wr at BN + k, Ws at 2 BN + k  (BN rows = 8 groups of 256 B)
                        i8_sts<0>(ad, nhs);
                        i8_sts<BPLANE>(ad, nls);
                        i8_sts<8 * 256>(ad, whr);
                        i8_sts<BPLANE + 8 * 256>(ad, wlr);
                        i8_sts<16 * 256>(ad, whs);
                        i8_sts<BPLANE + 16 * 256>(ad, wls);
                    }
#else
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        uint32_t hc[4], lc[4], hs[4], ls[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            unsigned long long t1, t2;
                            quantise(v[u], t1, t2);
                            hc[u] = (uint32_t)t1; hs[u] = (uint32_t)(t1 >> 32);
                            lc[u] = (uint32_t)t2; ls[u] = (uint32_t)(t2 >> 32);
                            const unsigned long long cd = pack2(lo2(st[u]), lo2(st[u]));
                            const unsigned long long sd = pack2(-hi2(st[u]), hi2(st[u]));
                            v[u] = ffma2(swap2(v[u]), sd, f2mul(v[u], cd));
                        }
                        const uint32_t whr = pack_bytes(hc[0], hc[1], hc[2], hc[3]);
                        const uint32_t wlr = pack_bytes(lc[0], lc[1], lc[2], lc[3]);
                        const uint32_t whs = pack_bytes(hs[0], hs[1], hs[2], hs[3]);
                        const uint32_t wls = pack_bytes(ls[0], ls[1], ls[2], ls[3]);
                        const uint32_t ad = a0 + (uint32_t)(r * 256);
                        // B rows: -Ws at k, Wr at BN + k, Ws at 2 BN + k  (BN rows = 8 groups of 256 B)
                        i8_sts<0>(ad, neg_bytes(whs));
                        i8_sts<BPLANE>(ad, neg_bytes(wls));
                        i8_sts<8 * 256>(ad, whr);
                        i8_sts<BPLANE + 8 * 256>(ad, wlr);
                        i8_sts<16 * 256>(ad, whs);
                        i8_sts<BPLANE + 16 * 256>(ad, wls);
                    }
#endif
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) i8_arrive_cluster(full0 + (uint32_t)(s * 8));
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    if (warp < 8) {
        // ================= drain (warps 0-7 after production): exact int32 accumulators -> fp32 partial tile ======
        // warp w reads TMEM lane quarter w % 4 (the tcgen05.ld lane restriction) and column half w / 4
        const int quarter = warp & 3, half = warp >> 2;
        i8_mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16);
        const int row = quarter * 32 + lane;
        const int64_t n_q = g.n_h * g.n_k;
        float2* P = partial + (chunk * frames + t) * n_q;
        // p = (64516 HH + 254 X) F / 32258^2 in FP32 (the partial is fp32; |rounding| <= 2^-23 |p|).  The tile goes
        // through shared memory (the stage ring is free once `done` fired: every MMA has read its operands) so that
        // the global writes are row-contiguous: TMEM lane = pixel row, so direct stores would touch 32 rows per
        // instruction.  Layout [128 rows][64 float4 + 1 pad] (pixel pairs; the pad makes the float4 writes of a
        // warp's 32 rows conflict-free).
#if XPCS_I8_Q16
        const float c_hh = (float)(65536.0 * (double)F / (32512.0 * 32512.0));   // p = (65536 HH + 256 X) F / QS^2
        const float c_x = (float)(256.0 * (double)F / (32512.0 * 32512.0));
#else
        const float c_hh = (float)(64516.0 * (double)F / (32258.0 * 32258.0));
        const float c_x = (float)(254.0 * (double)F / (32258.0 * 32258.0));
#endif
        float4* tile = reinterpret_cast<float4*>(smem);
        constexpr int TLD = TN / 2 + 1;
#pragma unroll 1
        for (int kb = 8 * half; kb < 8 * half + 8; ++kb) {     // 8 pixel columns per step (32 registers of TMEM data)
            const uint32_t cre = (uint32_t)(kb < 8 ? 8 * kb : 8 * kb + 64);   // [Re k<64 | Im' k<64 | Re k>=64 | Im' k>=64]
            uint32_t hre[8], him[8], xre[8], xim[8];
            I8_TMEM_LD8(tb + cre, hre);
            I8_TMEM_LD8(tb + cre + 64, him);
            I8_TMEM_LD8(tb + 256 + cre, xre);
            I8_TMEM_LD8(tb + 256 + cre + 64, xim);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                float4 v;
                v.x = fmaf((float)(int32_t)hre[j], c_hh, (float)(int32_t)xre[j] * c_x);
                v.y = fmaf((float)(int32_t)him[j], c_hh, (float)(int32_t)xim[j] * c_x);
                v.z = fmaf((float)(int32_t)hre[j + 1], c_hh, (float)(int32_t)xre[j + 1] * c_x);
                v.w = fmaf((float)(int32_t)him[j + 1], c_hh, (float)(int32_t)xim[j + 1] * c_x);
                tile[row * TLD + 4 * kb + j / 2] = v;
            }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");   // drain warps 0-7 only
        const int tid = threadIdx.x;                     // 0..255
        const int rows = (int)min((int64_t)TM, g.n_h - th0), cols = (int)min((int64_t)TN, g.n_k - tk0);
        const bool vec = (g.n_k & 1) == 0;               // 16-B aligned pixel pairs
        if (direct_out == nullptr) {
            for (int e = tid; e < TM * (TN / 2); e += 256) {
                const int r = e / (TN / 2), c2 = e % (TN / 2);
                if (r >= rows || 2 * c2 >= cols) continue;
                const float4 v = tile[r * TLD + c2];
                float2* dst = P + (int64_t)(th0 + r) * g.n_k + tk0 + 2 * c2;
                if (vec && 2 * c2 + 1 < cols) *reinterpret_cast<float4*>(dst) = v;
                else {
                    dst[0] = make_float2(v.x, v.y);
                    if (2 * c2 + 1 < cols) dst[1] = make_float2(v.z, v.w);
                }
            }
        } else {
            // single atom chunk: the final result straight from the tile, with the arithmetic of k_amp_reduce for
            // C = 1 (FP64 |p|^2 of the fp32 amplitude, Eq. 8; or the amplitude p = conj of the accumulated value)
            for (int e = tid; e < TM * (TN / 2); e += 256) {
                const int r = e / (TN / 2), c2 = e % (TN / 2);
                if (r >= rows || 2 * c2 >= cols) continue;
                const float4 v = tile[r * TLD + c2];
                const bool two = 2 * c2 + 1 < cols;
                const int64_t i0 = t * n_q + (int64_t)(th0 + r) * g.n_k + tk0 + 2 * c2;
                if (mode == 0) {
                    const double I0 = (double)v.x * (double)v.x + (double)v.y * (double)v.y;
                    const double I1 = (double)v.z * (double)v.z + (double)v.w * (double)v.w;
                    if (out_f64) {
                        double* o = (double*)direct_out + i0;
                        o[0] = I0;
                        if (two) o[1] = I1;
                    } else {
                        float* o = (float*)direct_out + i0;
                        if (two && vec) *reinterpret_cast<float2*>(o) = make_float2((float)I0, (float)I1);
                        else { o[0] = (float)I0; if (two) o[1] = (float)I1; }
                    }
                } else {
                    if (out_f64) {
                        double* o = (double*)direct_out + 2 * i0;
                        o[0] = (double)v.x; o[1] = -(double)v.y;
                        if (two) { o[2] = (double)v.z; o[3] = -(double)v.w; }
                    } else {
                        float* o = (float*)direct_out + 2 * i0;
                        if (two && vec) *reinterpret_cast<float4*>(o) = make_float4(v.x, -v.y, v.z, -v.w);
                        else { o[0] = v.x; o[1] = -v.y; if (two) { o[2] = v.z; o[3] = -v.w; } }
                    }
                }
            }
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

// clusters of k_lattice_i8 resident at once on the current device (one wave); sm_count / 2 if the query fails
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
                              void* direct_out, int out_f64, int mode) {
    if (direct_out && n_chunks != 1) return cudaErrorInvalidValue;
    using namespace ti8;
    if (chunk_atoms > kI8MaxChunk) return cudaErrorInvalidValue;
    const int tiles_h = (int)((g.n_h + PAIR_M - 1) / PAIR_M), tiles_k = (int)((g.n_k + TN - 1) / TN);
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
                                                    direct_out, out_f64, mode);
    return cudaGetLastError();
}

}  // namespace xpcs
