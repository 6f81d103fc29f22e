// How many 2-CTA clusters of a 1-CTA-per-SM kernel (200 KB dynamic smem) the
// device holds at once (cudaOccupancyMaxActiveClusters), vs SMs / 2.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int *p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) p[0] = s[0]; }
int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int cs : {1, 2, 4}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sms / cs * cs);
        cfg.blockDim = dim3(448);
        cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int mc = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&mc, k, &cfg);
        printf("SMs %d cluster %d: max active clusters %d (%s) -> %d CTAs\n", sms, cs, mc,
               cudaGetErrorString(e), mc * cs);
    }
    return 0;
}
