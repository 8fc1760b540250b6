// How many clusters of 2/3/4/6/8 CTAs (one CTA per SM, ~160 KB shared memory) can be resident
// at once on this device: the GPC granularity that bounds cluster-shaped persistent grids.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; s[threadIdx.x] = 0; }
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 167 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    for (int cl : {1, 2, 3, 4, 6, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cl * 64);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = 167 * 1024;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %2d: max active clusters %d (%d SMs) %s\n", cl, n, n * cl, cudaGetErrorString(e));
    }
}
