// How many clusters of each size fit at one 200 KB / 512-thread CTA per SM (GPC packing).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o cluster_fit cluster_fit.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* p) {
    extern __shared__ int s[];
    s[threadIdx.x] = threadIdx.x;
    if (s[threadIdx.x ^ 1] == -1) p[0] = 1;
}

int main() {
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.blockDim = dim3(512);
        cfg.gridDim = dim3(cs);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %2d: %3d clusters -> %3d SMs %s\n", cs, n, n * cs, e ? cudaGetErrorString(e) : "");
    }
    return 0;
}
