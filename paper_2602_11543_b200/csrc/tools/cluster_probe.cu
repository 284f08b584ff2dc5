// How many thread-block clusters of size 2 / 4 / 8 (one 214 KB-smem CTA per SM, the grouped
// GEMM's footprint) can be co-resident on this GPU: the SM budget a multicast GEMM would get.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe_k(int* out) {
    extern __shared__ int s[];
    if (threadIdx.x == 0) s[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && out) out[blockIdx.x] = s[0];
}

int main() {
    const int smem = 214 * 1024;
    cudaFuncSetAttribute(probe_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_k, &cfg);
        printf("cluster %2d: max active clusters %d -> %d CTAs (%s)\n", cs, n, n * cs,
               cudaGetErrorString(e));
    }
    return 0;
}
