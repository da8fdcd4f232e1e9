// Probe: how many 2-CTA clusters can be co-resident on a B200 for a kernel shaped like the fused
// conv kernels (320 threads, ~100 KB dynamic shared memory, 96 registers) — i.e. whether
// cta_group::2 pairs can keep 2 CTAs per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_occ cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(320, 2) k_dummy(int* p) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0 && p) sm[0] = p[blockIdx.x];
}

int main() {
    for (int smem_kb : {60, 80, 100, 104, 110}) {
        for (int cs : {1, 2}) {
            cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
            cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(296);
            cfg.blockDim = dim3(320);
            cfg.dynamicSmemBytes = smem_kb * 1024;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
            int blocks = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_dummy, 320, smem_kb * 1024);
            printf("smem %3d KB cluster %d: max active clusters %d (%s), blocks/SM %d\n", smem_kb, cs, n,
                   cudaGetErrorString(e), blocks);
        }
    }
    return 0;
}
