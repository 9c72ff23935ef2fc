// Development probe: how many thread-block clusters of a 1-CTA-per-SM kernel
// (1024-thread launch bounds, large dynamic shared memory, like the sweep kernel)
// can be co-resident on this GPU, per cluster size and block size.
#include <cstdio>
#include <cuda_runtime.h>
extern __shared__ unsigned char sm[];
__global__ void __launch_bounds__(1024, 1) k(int *o) { if (o) o[threadIdx.x] = sm[threadIdx.x]; }
int main() {
    int smem = 180 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("sms %d\n", sms);
    const int blocks[] = {1024, 928, 832, 768, 704, 640, 512};
    for (int b : blocks)
        for (int cs = 1; cs <= 16; cs++) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs); cfg.blockDim = dim3(b); cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
            cfg.attrs = a; cfg.numAttrs = 1;
            int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
            printf("block %4d cluster %2d -> %3d clusters, %3d SMs %s\n", b, cs, n, n * cs, e ? cudaGetErrorString(e) : "");
        }
    return 0;
}
