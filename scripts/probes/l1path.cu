// Probe: does a register-destined global load (LDG.128, L1 no-allocate) cost the same L1/shared
// data-bank traffic as a cp.async (LDGSTS) into shared memory? Both kernels stream the same
// L2-resident 64 MiB buffer with 16-byte accesses, 8 rows of 128 B per warp instruction pair.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l1path l1path.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__global__ void k_ldg(const int4* __restrict__ src, size_t n16, int iters, int* out) {
    int acc = 0;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int it = 0; it < iters; ++it)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride * 4) {
            int4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                size_t j = i + u * stride;
                if (j < n16) asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + j));
                else v[u] = make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    if (acc == 0x12345678) out[0] = acc;
}

__global__ void k_ldgsts(const int4* __restrict__ src, size_t n16, int iters, int* out) {
    __shared__ __align__(16) int4 buf[4][256];
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int it = 0; it < iters; ++it)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride * 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                size_t j = i + u * stride;
                uint32_t d = (uint32_t)__cvta_generic_to_shared(&buf[u][threadIdx.x]);
                int sz = j < n16 ? 16 : 0;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src + (j < n16 ? j : 0)), "r"(sz));
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
    if (buf[0][threadIdx.x].x == 0x12345678) out[0] = 1;
}

int main() {
    size_t bytes = 64ull << 20, n16 = bytes / 16;
    int4* src;
    int* out;
    cudaMalloc(&src, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(src, 1, bytes);
    int iters = 20;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int k = 0; k < 2; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (k == 0) k_ldg<<<148 * 8, 256>>>(src, n16, iters, out);
            else k_ldgsts<<<148 * 8, 256>>>(src, n16, iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%s: %.3f ms, %.1f GB/s (L2-resident, %.1f B/clk/SM at 1.965 GHz)\n", k ? "ldgsts" : "ldg", ms,
               bytes * (double)iters / ms / 1e6, bytes * (double)iters / (ms * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
