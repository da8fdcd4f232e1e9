// Probe: tcgen05.mma issue rate from shared memory (SS) and with A in TMEM (TS), M = 128, bf16,
// N = 64 / 128 / 256, one CTA per SM, no producers — and the same with W warps streaming
// 16-byte cp.async copies of an L2-resident buffer into another shared region (the gather's
// shared-memory writes) to measure how the two share the SM's shared-memory bandwidth.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1803_11385_b200/csrc -o mma_rate mma_rate.cu
#include <cstdio>
#include <cuda_bf16.h>
#include "tc_common.cuh"
using namespace hcb::tc;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, int acc) {
    asm volatile(
        "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}

template <int N, bool TS, bool MN = false>
__global__ void __launch_bounds__(256, 1) k_rate(int iters, const int4* __restrict__ src, size_t n16, int copy_warps, int* flag) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    // A: 4 stages x 16 KB, B: 4 stages x N*128 B, copy region 64 KB
    uint8_t* A = sm;
    uint8_t* B = sm + 4 * 16384;
    uint8_t* Cp = B + 4 * N * 128;
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ int stop;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (4 * 16384 + 4 * N * 128) / 16; i += blockDim.x)
        reinterpret_cast<int4*>(sm)[i] = make_int4(0x3f803f80, 0x3f803f80, 0, 0);
    if (tid == 0) { mbar_init(smem_u32(&bar), 1); mbar_init_fence(); stop = 0; }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(128, N, MN, MN);
        // K-major: 16-byte LBO, 8-row atoms of 1 KB; MN-major (the dW kernel's layout): 64-wide MN
        // blocks 8 KB apart (64 K rows of 128 B), K16 = 16 rows = 2 KB
        const uint64_t a0 = MN ? sw128_desc(smem_u32(A), 8192, 1024) : sw128_desc(smem_u32(A), 16, 1024);
        const uint64_t b0 = MN ? sw128_desc(smem_u32(B), 8192, 1024) : sw128_desc(smem_u32(B), 16, 1024);
        const uint32_t kstep = MN ? 128 : 2;  // descriptor units (16 B) per K16
        if (elect_one()) {
            for (int it = 0; it < iters; ++it) {
                const int s = it & 3;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    if (TS) mma_ts(tmem + 256, tmem + s * 32 + kk * 8, b0 + ((s * N * 128) >> 4) + 2 * kk, idesc, 1);
                    else mma_bf16(tmem + (N <= 128 ? 256 : 0), a0 + ((s * 16384) >> 4) + kstep * kk, b0 + ((s * N * 128) >> 4) + kstep * kk, idesc, 1);
                }
            }
            mma_commit(smem_u32(&bar));
        }
        __syncwarp();
        mbar_wait(smem_u32(&bar), 0);
        if (lane_id() == 0) atomicExch(&stop, 1);
    } else if (warp <= copy_warps) {
        // stream 16-byte copies into a 64 KB region until the MMAs finish
        const size_t stride = (size_t)gridDim.x * copy_warps * 32;
        size_t i = ((size_t)blockIdx.x * copy_warps + (warp - 1)) * 32 + lane_id();
        uint32_t dst = smem_u32(Cp) + ((warp - 1) * 32 + lane_id()) * 16;
        int k = 0;
        while (!*(volatile int*)&stop) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + ((k + u) & 7) * 8192), "l"(src + i));
                i += stride;
                if (i >= n16) i -= n16;
            }
            k += 8;
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 2;" ::: "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        atomicAdd(reinterpret_cast<unsigned long long*>(flag), (unsigned long long)k);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS, bool MN = false>
void run(int copy_warps, const int4* src, size_t n16, int* flag) {
    auto k = k_rate<N, TS, MN>;
    const int smem = 1024 + 4 * 16384 + 4 * N * 128 + 65536;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<148, 256, smem>>>(100, src, n16, copy_warps, flag);
    cudaDeviceSynchronize();
    cudaMemset(flag, 0, 8);
    cudaEventRecord(a);
    k<<<148, 256, smem>>>(iters, src, n16, copy_warps, flag);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double cyc = ms * 1e-3 * 1.965e9;  // at max clock
    const double mmas = (double)iters * 4;
    const double floor_cyc = 128.0 * N / 256;
    unsigned long long copies = 0;
    cudaMemcpy(&copies, flag, 8, cudaMemcpyDeviceToHost);
    printf("%s%s N=%3d copy_warps=%d: %.3f ms, %.1f cycles per MMA (floor %.0f) -> %.0f%% of tensor floor; MMA smem reads %.0f B/clk/SM; cp.async writes %.0f B/clk/SM\n",
           TS ? "TS" : "SS", MN ? "-MN" : "", N, copy_warps, ms, cyc / mmas, floor_cyc, 100 * floor_cyc * mmas / cyc,
           mmas * ((TS ? 0 : 4096) + N * 32) / cyc / 148, copies * 32.0 * 16 / cyc / 148);
}

int main() {
    size_t bytes = 64ull << 20, n16 = bytes / 16;
    int4* src;
    int* flag;
    cudaMalloc(&src, bytes);
    cudaMalloc(&flag, 8);
    cudaMemset(src, 0, bytes);
    for (int cw : {0, 4}) {
        run<64, false>(cw, src, n16, flag);
        run<128, false>(cw, src, n16, flag);
        run<64, false, true>(cw, src, n16, flag);
        run<128, false, true>(cw, src, n16, flag);
        run<64, true>(cw, src, n16, flag);
        run<128, true>(cw, src, n16, flag);
    }
    return 0;
}
