// gemm_exact.cu — order-exact products (HC_MATH_EXACT; fp32 and fp64, the reference's two
// instantiations gemm.cpp:117-118), bit-identical to src/gemm.cpp: every output element
// accumulates k strictly ascending with a separately rounded multiply and add
// (mul_rn/add_rn = __fmul_rn/__fadd_rn or __dmul_rn/__dadd_rn: no FMA contraction),
// and matmul / matmul_trans_a skip zero a-entries exactly like row_axpy_product
// (gemm.cpp:14-26) and matmul_trans_a (gemm.cpp:37-52).
//
// These kernels are the parity path. They keep the reference's serial
// reduction per output element, so matmul_trans_b (a dot over N voxels) is
// latency-bound by design; the throughput path is HC_MATH_FAST / the native
// implicit-GEMM conv (conv_tc.cu).
#include <cuda_runtime.h>

#include "hc_launch.cuh"

namespace hcb {

namespace {

constexpr int kRows = 32;   // output rows per thread (register block)
constexpr int kKTile = 32;  // k-slice of `a` staged in shared memory
constexpr int kThreads = 128;

// gemm.cpp:14-35: c[i,j] = sum_k a[i,k]*b[k,j] (k ascending, a==0 skipped)
template <typename T>
__global__ void k_nn_exact(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ c,
                           long long ra, long long k, long long cb) {
    __shared__ T as[kRows][kKTile];
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long i0 = (long long)blockIdx.y * kRows;
    T acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = T(0);
    for (long long k0 = 0; k0 < k; k0 += kKTile) {
        for (int e = threadIdx.x; e < kRows * kKTile; e += blockDim.x) {
            const int r = e / kKTile, kk = e % kKTile;
            as[r][kk] = (i0 + r < ra && k0 + kk < k) ? a[(i0 + r) * k + k0 + kk] : T(0);
        }
        __syncthreads();
        const int kt = (int)(k - k0 < kKTile ? k - k0 : kKTile);
        for (int kk = 0; kk < kt; ++kk) {
            const T bv = j < cb ? __ldg(b + (k0 + kk) * cb + j) : T(0);
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                const T av = as[r][kk];
                if (av != T(0)) acc[r] = add_rn(acc[r], mul_rn(av, bv));
            }
        }
        __syncthreads();
    }
    if (j < cb)
#pragma unroll
        for (int r = 0; r < kRows; ++r)
            if (i0 + r < ra) c[(i0 + r) * cb + j] = acc[r];
}

// gemm.cpp:37-52: c[r,j] = sum_i a[i,r]*b[i,j] (i ascending, a==0 skipped)
template <typename T>
__global__ void k_tn_exact(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ c,
                           long long ra, long long k, long long cb) {
    __shared__ T as[kKTile][kRows];
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long r0 = (long long)blockIdx.y * kRows;
    T acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = T(0);
    for (long long i0 = 0; i0 < ra; i0 += kKTile) {
        for (int e = threadIdx.x; e < kRows * kKTile; e += blockDim.x) {
            const int ii = e / kRows, r = e % kRows;
            as[ii][r] = (i0 + ii < ra && r0 + r < k) ? a[(i0 + ii) * k + r0 + r] : T(0);
        }
        __syncthreads();
        const int it = (int)(ra - i0 < kKTile ? ra - i0 : kKTile);
        for (int ii = 0; ii < it; ++ii) {
            const T bv = j < cb ? __ldg(b + (i0 + ii) * cb + j) : T(0);
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                const T av = as[ii][r];
                if (av != T(0)) acc[r] = add_rn(acc[r], mul_rn(av, bv));
            }
        }
        __syncthreads();
    }
    if (j < cb)
#pragma unroll
        for (int r = 0; r < kRows; ++r)
            if (r0 + r < k) c[(r0 + r) * cb + j] = acc[r];
}

// gemm.cpp:54-69: c[i,j] = a[i,:] . b[j,:], a strictly sequential dot.
// One thread per output; 32 threads of a warp share i (broadcast a loads).
template <typename T>
__global__ void k_nt_exact(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ c,
                           long long ra, long long k, long long rb) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= ra * rb) return;
    const long long i = t / rb, j = t % rb;
    const T* ar = a + i * k;
    const T* br = b + j * k;
    T acc = T(0);
    long long kk = 0;
    for (; kk + 8 <= k; kk += 8) {
        T av[8], bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            av[u] = __ldg(ar + kk + u);
            bv[u] = __ldg(br + kk + u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = add_rn(acc, mul_rn(av[u], bv[u]));
    }
    for (; kk < k; ++kk) acc = add_rn(acc, mul_rn(__ldg(ar + kk), __ldg(br + kk)));
    c[i * rb + j] = acc;
}

template <typename T>
void nn_exact(const T* a, const T* b, T* c, long long ra, long long k, long long cb,
                   cudaStream_t s) {
    if (ra <= 0 || cb <= 0) return;
    if (k <= 0) {
        cuda_check(cudaMemsetAsync(c, 0, sizeof(T) * ra * cb, s), "memset");
        return;
    }
    dim3 g(grid_for(cb, kThreads), (unsigned)((ra + kRows - 1) / kRows));
    k_nn_exact<T><<<g, kThreads, 0, s>>>(a, b, c, ra, k, cb);
    launched("matmul (exact)");
}

template <typename T>
void tn_exact(const T* a, const T* b, T* c, long long ra, long long k, long long cb,
                   cudaStream_t s) {
    if (k <= 0 || cb <= 0) return;
    if (ra <= 0) {
        cuda_check(cudaMemsetAsync(c, 0, sizeof(T) * k * cb, s), "memset");
        return;
    }
    dim3 g(grid_for(cb, kThreads), (unsigned)((k + kRows - 1) / kRows));
    k_tn_exact<T><<<g, kThreads, 0, s>>>(a, b, c, ra, k, cb);
    launched("matmul_trans_a (exact)");
}

template <typename T>
void nt_exact(const T* a, const T* b, T* c, long long ra, long long k, long long rb,
                   cudaStream_t s) {
    if (ra <= 0 || rb <= 0) return;
    k_nt_exact<T><<<grid_for(ra * rb, kThreads), kThreads, 0, s>>>(a, b, c, ra, k, rb);
    launched("matmul_trans_b (exact)");
}


}  // namespace

#define HC_EXACT_OVERLOADS(T)                                                                                   \
    void gemm_nn_exact(const T* a, const T* b, T* c, long long ra, long long k, long long cb, cudaStream_t s) {  \
        nn_exact<T>(a, b, c, ra, k, cb, s);                                                                     \
    }                                                                                                           \
    void gemm_tn_exact(const T* a, const T* b, T* c, long long ra, long long k, long long cb, cudaStream_t s) {  \
        tn_exact<T>(a, b, c, ra, k, cb, s);                                                                     \
    }                                                                                                           \
    void gemm_nt_exact(const T* a, const T* b, T* c, long long ra, long long k, long long rb, cudaStream_t s) {  \
        nt_exact<T>(a, b, c, ra, k, rb, s);                                                                     \
    }
HC_EXACT_OVERLOADS(float)
HC_EXACT_OVERLOADS(double)
#undef HC_EXACT_OVERLOADS

}  // namespace hcb
