// gemm_fast.cu — HC_MATH_FAST contraction for the reference-layout operators:
// a register-tiled FFMA GEMM (128x128 CTA tile, 8x8 per thread) with a
// deterministic split-K (partials reduced in fixed split order by a second
// kernel) for the long-K product matmul_trans_b (dW, K = N voxels).
// Tolerance-level parity only (FMA contraction and a different summation order
// than src/gemm.cpp). The tensor-core path lives in conv_tc.cu.
#include <cuda_runtime.h>

#include "hc_launch.cuh"

namespace hcb {

namespace {

constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8, NT = 256;

// C[M x N] (+)= opA(A)[M x K] * opB(B)[K x N] over k in [k_begin, k_end)
//   TA: A stored K x M (lda = M), else M x K (lda = K)
//   TB: B stored N x K (ldb = K), else K x N (ldb = N)
template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) k_gemm(const float* __restrict__ A, const float* __restrict__ B,
                                             float* __restrict__ Cout, long long M, long long N, long long K,
                                             long long k_chunk) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const long long m0 = (long long)blockIdx.y * BM, n0 = (long long)blockIdx.x * BN;
    const long long kb = (long long)blockIdx.z * k_chunk;
    const long long ke = min(K, kb + k_chunk);
    float* C = Cout + (long long)blockIdx.z * M * N;
    const int tid = threadIdx.x;
    const int tm = (tid / (BN / TN)) * TM, tn = (tid % (BN / TN)) * TN;
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

    for (long long k0 = kb; k0 < ke; k0 += BK) {
        // stage A tile (BM x BK) and B tile (BK x BN): 1024 elements each, 4 per thread
#pragma unroll
        for (int e = 0; e < (BM * BK) / NT; ++e) {
            const int idx = tid + e * NT;
            int mm, kk;
            if (TA) { mm = idx % BM; kk = idx / BM; }   // coalesced along m
            else    { kk = idx % BK; mm = idx / BK; }   // along k
            const long long gm = m0 + mm, gk = k0 + kk;
            float v = 0.0f;
            if (gm < M && gk < ke) v = TA ? __ldg(A + gk * M + gm) : __ldg(A + gm * K + gk);
            As[kk][mm] = v;
        }
#pragma unroll
        for (int e = 0; e < (BN * BK) / NT; ++e) {
            const int idx = tid + e * NT;
            int nn, kk;
            if (TB) { kk = idx % BK; nn = idx / BK; }
            else    { nn = idx % BN; kk = idx / BN; }
            const long long gn = n0 + nn, gk = k0 + kk;
            float v = 0.0f;
            if (gn < N && gk < ke) v = TB ? __ldg(B + gn * K + gk) : __ldg(B + gk * N + gn);
            Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float ar[TM], br[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) ar[i] = As[kk][tm + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) br[j] = Bs[kk][tn + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const long long gm = m0 + tm + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const long long gn = n0 + tn + j;
            if (gn < N) C[gm * N + gn] = acc[i][j];
        }
    }
}

// fixed-order reduction of split partials: c = sum_z P[z] (z ascending)
__global__ void k_reduce_splits(const float* __restrict__ P, float* __restrict__ C, long long MN, int splits) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= MN) return;
    float s = 0.0f;
    for (int z = 0; z < splits; ++z) s += P[(long long)z * MN + i];
    C[i] = s;
}

template <bool TA, bool TB>
void run(const float* A, const float* B, float* C, long long M, long long N, long long K, cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0) {
        cuda_check(cudaMemsetAsync(C, 0, sizeof(float) * M * N, s), "memset");
        return;
    }
    const long long tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    int splits = 1;
    // long-K products with few output tiles: split K so ~2 waves fill 148 SMs
    while (tiles * splits < 296 && K / (splits * 2) >= 4096 && splits < 256) splits *= 2;
    const long long chunk = ((K + splits - 1) / splits + BK - 1) / BK * BK;
    dim3 g((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)splits);
    if (splits == 1) {
        k_gemm<TA, TB><<<g, NT, 0, s>>>(A, B, C, M, N, K, chunk);
    } else {
        Scratch part(sizeof(float) * M * N * splits, s);
        k_gemm<TA, TB><<<g, NT, 0, s>>>(A, B, part.as<float>(), M, N, K, chunk);
        k_reduce_splits<<<grid_for(M * N, 256), 256, 0, s>>>(part.as<float>(), C, M * N, splits);
    }
    launched("gemm (fast)", splits == 1 ? 1 : 2);
}

}  // namespace

// matmul: c[ra x cb] = a[ra x k] * b[k x cb]
void fast_gemm_nn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, cudaStream_t s) {
    run<false, false>(a, b, c, ra, cb, k, s);
}
// matmul_trans_a: c[k x cb] = a[ra x k]^T * b[ra x cb]
void fast_gemm_tn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, cudaStream_t s) {
    run<true, false>(a, b, c, k, cb, ra, s);
}
// matmul_trans_b: c[ra x rb] = a[ra x k] * b[rb x k]^T
void fast_gemm_nt(const float* a, const float* b, float* c, long long ra, long long k, long long rb, cudaStream_t s) {
    run<false, true>(a, b, c, ra, rb, k, s);
}

}  // namespace hcb
