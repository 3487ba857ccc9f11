// How many clusters of 2 / 4 / 8 CTAs (one CTA per SM: ~200 KB of dynamic shared memory) fit at once on this GPU:
// cluster sizes above 2 lose the SMs a GPC cannot fill with whole clusters.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_probe(int* o) { extern __shared__ int s[]; s[threadIdx.x] = 0; if (o) o[0] = s[0]; }
int main() {
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("{\"sms\": %d", sms);
    for (int cl : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl * 64, 1, 1); cfg.blockDim = dim3(704, 1, 1); cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k_probe, &cfg);
        printf(", \"cl%d\": {\"clusters\": %d, \"ctas\": %d, \"err\": \"%s\"}", cl, n, n * cl, cudaGetErrorString(e));
    }
    printf("}\n");
}
