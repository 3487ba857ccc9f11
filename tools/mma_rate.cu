// mma_rate.cu -- tcgen05 MMA issue rate per SM (clock64, so per clock and independent of DVFS): kind::f16 vs
// kind::i8, cta_group::1, M = 128, N = 256, back-to-back on fixed shared-memory operands.  Decides whether an
// integer-limb engine (exact int32 accumulation) can beat the split-FP16 engine.  One JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_rate tools/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

template <int KIND>   // 0 = f16, 1 = i8
__global__ void __launch_bounds__(128, 1) k_rate(int reps, unsigned long long* cyc) {
    __shared__ __align__(1024) char sm[4096 + 8192];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < (4096 + 8192) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t base = smem_u32(sm);
        const uint64_t a = desc(base, 128, 256), b = desc(base + 4096, 128, 256);
        const uint32_t idesc = KIND == 0 ? ((1u << 4) | ((256u >> 3) << 17) | ((128u >> 4) << 24))
                                         : ((2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24));
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            const uint32_t d = tmem + (uint32_t)((r & 1) * 256);
            if (KIND == 0)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(r > 1 ? 1 : 0));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(r > 1 ? 1 : 0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        const long long t1 = clock64();
        cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    unsigned long long h[512];
    const int reps = 8192;
    double rate[2];
    float ms[2];
    for (int kind = 0; kind < 2; ++kind) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int w = 0; w < 2; ++w) {
            cudaEventRecord(e0);
            if (kind == 0) k_rate<0><<<sms, 128>>>(reps, d); else k_rate<1><<<sms, 128>>>(reps, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms[kind], e0, e1);
        cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        const double macs = 128.0 * 256.0 * (kind == 0 ? 16.0 : 32.0) * reps;
        rate[kind] = macs / mx;
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"sms\": %d, \"f16_mac_per_clk_per_sm\": %.1f, \"i8_mac_per_clk_per_sm\": %.1f, \"f16_ms\": %.3f, "
           "\"i8_ms\": %.3f, \"f16_tflops_wall\": %.1f, \"i8_tops_wall\": %.1f, \"err\": \"%s\"}\n", sms, rate[0], rate[1],
           ms[0], ms[1], 2.0 * 128 * 256 * 16.0 * reps * sms / (ms[0] * 1e-3) / 1e12,
           2.0 * 128 * 256 * 32.0 * reps * sms / (ms[1] * 1e-3) / 1e12, cudaGetErrorString(e));
    return 0;
}
