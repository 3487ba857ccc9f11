// microbench.cu -- C4 roofline microbenchmarks on the B200 (per-SM issue rates measured with clock64, so the
// numbers are per clock and independent of the DVFS state).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o build/microbench tools/microbench.cu ; run on the GPU box.  Prints one JSON line.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int CH = 8;

__device__ unsigned long long g_sink;

__global__ void __launch_bounds__(1024) k_mufu(float seed, unsigned long long* cyc) {
    float x[CH];
    for (int i = 0; i < CH; ++i) x[i] = seed + threadIdx.x * 1e-3f + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) { float s, c; __sincosf(x[i], &s, &c); x[i] = s + c; }
    }
    __syncthreads();
    long long t1 = clock64();
    float acc = 0; for (int i = 0; i < CH; ++i) acc += x[i];
    if (acc == 12345.f) g_sink = 1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(1024) k_ffma(float seed, unsigned long long* cyc) {
    float x[CH], y = seed * 0.999f, z = seed * 1e-7f;
    for (int i = 0; i < CH; ++i) x[i] = seed + threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], y, z);
    }
    __syncthreads();
    long long t1 = clock64();
    float acc = 0; for (int i = 0; i < CH; ++i) acc += x[i];
    if (acc == 12345.f) g_sink = 1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(1024) k_ffma2(float seed, unsigned long long* cyc) {
    unsigned long long x[CH], y, z;
    float a = seed * 0.999f, b = seed * 1e-7f;
    y = (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(a) << 32);
    z = (unsigned long long)__float_as_uint(b) | ((unsigned long long)__float_as_uint(b) << 32);
    for (int i = 0; i < CH; ++i) { float v = seed + threadIdx.x + i; x[i] = (unsigned long long)__float_as_uint(v) * 0x100000001ull; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(y), "l"(z));
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned long long acc = 0; for (int i = 0; i < CH; ++i) acc ^= x[i];
    if (acc == 12345) g_sink = 1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(1024) k_dfma(double seed, unsigned long long* cyc) {
    double x[CH], y = seed * 0.999, z = seed * 1e-7;
    for (int i = 0; i < CH; ++i) x[i] = seed + threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fma(x[i], y, z);
    }
    __syncthreads();
    long long t1 = clock64();
    double acc = 0; for (int i = 0; i < CH; ++i) acc += x[i];
    if (acc == 12345.0) g_sink = 1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(1024) k_imad(unsigned seed, unsigned long long* cyc) {
    unsigned x[CH], y = seed | 1, z = seed * 7;
    for (int i = 0; i < CH; ++i) x[i] = seed + threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = x[i] * y + z;
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned acc = 0; for (int i = 0; i < CH; ++i) acc ^= x[i];
    if (acc == 12345) g_sink = 1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K, typename A>
double run(K kern, A seed, double ops_per_thread_iter, int iters, int sms, unsigned long long* d) {
    kern<<<sms, 1024>>>(seed, d);
    cudaDeviceSynchronize();
    kern<<<sms, 1024>>>(seed, d);
    cudaDeviceSynchronize();
    unsigned long long h[1024];
    cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    return 1024.0 * iters * CH * ops_per_thread_iter / mx;   // ops per clock per SM
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * 1024);
    double mufu = run(k_mufu, 0.3f, 2.0, ITERS, sms, d);        // MUFU.SIN + MUFU.COS per sincos
    double ffma = run(k_ffma, 1.0f, 1.0, ITERS, sms, d);
    double ffma2 = run(k_ffma2, 1.0f, 2.0, ITERS, sms, d);      // 2 FMA lanes per FFMA2
    double dfma = run(k_dfma, 1.0, 1.0, ITERS / 8, sms, d);
    double imad = run(k_imad, 3u, 1.0, ITERS, sms, d);
    printf("{\"sms\": %d, \"mufu_per_clk_sm\": %.2f, \"ffma_per_clk_sm\": %.2f, \"ffma2_fma_per_clk_sm\": %.2f, "
           "\"dfma_per_clk_sm\": %.2f, \"imad_per_clk_sm\": %.2f, \"err\": \"%s\"}\n",
           sms, mufu, ffma, ffma2, dfma, imad, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
