// Probe: tcgen05.mma with the A operand in tensor memory (TS form), kind::f16 (bf16 in, fp32 acc).
// A (128 x 64) is written into TMEM by the 4 warps with tcgen05.st.32x32b.x32 (thread = lane = row m,
// 32-bit column j = elements k = 2j (low half) and 2j+1); B (N x 64) sits in shared memory in the
// K-major SWIZZLE_128B layout. D = A . B^T is checked against a host reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1803_11385_b200/csrc -o ts_mma ts_mma.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_bf16.h>
#include "tc_common.cuh"
using namespace hcb::tc;

constexpr int N = 64;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, int acc) {
    asm volatile(
        "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}

__global__ void k_probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
    __shared__ __align__(1024) uint8_t bs[N * 128 + 1024];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    uint8_t* b = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(bs) + 1023) & ~uintptr_t(1023));
    for (int e = tid; e < N * 8; e += 128) {  // row n, chunk c (8 bf16)
        const int n = e / 8, c = e % 8;
        *reinterpret_cast<int4*>(b + sw128_offset(n, c)) = *reinterpret_cast<const int4*>(B + n * 64 + c * 8);
    }
    if (tid == 0) { mbar_init(smem_u32(&bar), 1); mbar_init_fence(); }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // A rows -> TMEM columns [0, 32)
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) {
        __nv_bfloat162 p = __halves2bfloat162(A[tid * 64 + 2 * j], A[tid * 64 + 2 * j + 1]);
        v[j] = *reinterpret_cast<uint32_t*>(&p);
    }
    tmem_st32(tmem + ((uint32_t)(warp * 32) << 16), v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(128, N, false, false);
        const uint64_t b0 = sw128_desc(smem_u32(b), 16, 1024);
        for (int kk = 0; kk < 4; ++kk) mma_ts(tmem + 64, tmem + kk * 8, b0 + 2 * kk, idesc, kk != 0);
        mma_commit(smem_u32(&bar));
    }
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + 64 + c0, r);
        tmem_ld_wait();
        for (int e = 0; e < 16; ++e) D[tid * N + c0 + e] = __uint_as_float(r[e]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 128); }
}

int main() {
    __nv_bfloat16 *hA = new __nv_bfloat16[128 * 64], *hB = new __nv_bfloat16[N * 64];
    float* hD = new float[128 * N];
    srand(1);
    for (int i = 0; i < 128 * 64; ++i) hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
    for (int i = 0; i < N * 64; ++i) hB[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
    __nv_bfloat16 *dA, *dB;
    float* dD;
    cudaMalloc(&dA, 128 * 64 * 2); cudaMalloc(&dB, N * 64 * 2); cudaMalloc(&dD, 128 * N * 4);
    cudaMemcpy(dA, hA, 128 * 64 * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, N * 64 * 2, cudaMemcpyHostToDevice);
    k_probe<<<1, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < 64; ++k) s += (double)__bfloat162float(hA[m * 64 + k]) * __bfloat162float(hB[n * 64 + k]);
            maxerr = fmax(maxerr, fabs(s - hD[m * N + n]));
        }
    printf("TS-form MMA (A in TMEM, 32x32b.x32 store): max abs err %.3g -> %s\n", maxerr, maxerr < 1e-3 ? "OK" : "MISMATCH");
    return 0;
}
