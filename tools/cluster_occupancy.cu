// How many 2-CTA clusters of a 384-thread, 227 KB-shared-memory kernel can be
// co-resident on this GPU (the persistent attention grid needs 74 for 148 CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/co tools/cluster_occupancy.cu && /tmp/co
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* x) { extern __shared__ int s[]; if (x) x[0] = s[0]; }
int main() {
    const int smem = 232448;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148 / cs * cs);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
    }
}
