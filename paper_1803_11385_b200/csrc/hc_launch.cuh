// hc_launch.cuh — small launch helpers shared by the .cu files (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "hashconv_b200.h"

namespace hcb {

void cuda_check(cudaError_t e, const char* what);
void* dev_alloc(size_t bytes);
hc_math current_math();

// Kernel-launch accounting (hc_launch_count): every launch site reports how many
// kernels it enqueued, then checks the launch.
void count_launches(long long n);
inline void launched(const char* what, long long n = 1) {
    count_launches(n);
    cuda_check(cudaGetLastError(), what);
}

inline cudaStream_t as_stream(hc_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// The dynamic shared-memory opt-in is a per-device-context attribute: set it once per
// (kernel, device), so a process driving several GPUs sets it on each.
bool smem_optin_needed(const void* kern, int dev);  // records (kern, dev) on first query
template <typename K>
void smem_optin(K kern, int bytes) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (!smem_optin_needed(reinterpret_cast<const void*>(kern), dev)) return;
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem attr");
}

inline unsigned grid_for(long long n, int threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

// The default stream-ordered pool releases freed memory to the OS at every synchronisation
// (release threshold 0), so a multi-GB scratch (a materialised column matrix, lo planes)
// would be re-mapped on every call. Keep up to HCB_POOL_KEEP_GB (default 48) GB cached.
void scratch_pool_init();

// Stream-ordered scratch buffer (cudaMallocAsync / cudaFreeAsync).
struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    Scratch(size_t bytes, cudaStream_t st) : s(st) {
        scratch_pool_init();
        cuda_check(cudaMallocAsync(&p, bytes ? bytes : 16, st), "cudaMallocAsync");
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Reference-signature conv in HC_MATH_FAST on the fused split-precision tensor-core path
// (conv_tc.cu): eligible for a stride-1 field over one structure with <= 128 channels.
bool fused_x2_eligible(const hc_psh* in, const hc_psh* out, hc_conv_spec sp, int taps);
long long fused_route_count(long long add);  // hc_fused_route_count
int* deferred_flag_device();                  // hc_deferred_status's word (device alias)
void fused_conv_forward_f32(const hc_psh* in, const float* data, const float* w, hc_conv_spec sp, int taps,
                            long long N, float* result, cudaStream_t s);
void fused_conv_backward_f32(const float* dy, const float* w, const float* cols, const hc_psh* in, hc_conv_spec sp,
                             int taps, long long N, float* dw, float* dx, cudaStream_t s);

// Exact GEMMs (gemm_exact.cu) — reference accumulation order, fp32 and fp64.
void gemm_nn_exact(const float* a, const float* b, float* c, long long ra, long long k, long long cb, cudaStream_t s);
void gemm_tn_exact(const float* a, const float* b, float* c, long long ra, long long k, long long cb, cudaStream_t s);
void gemm_nt_exact(const float* a, const float* b, float* c, long long ra, long long k, long long rb, cudaStream_t s);
void gemm_nn_exact(const double* a, const double* b, double* c, long long ra, long long k, long long cb,
                   cudaStream_t s);
void gemm_tn_exact(const double* a, const double* b, double* c, long long ra, long long k, long long cb,
                   cudaStream_t s);
void gemm_nt_exact(const double* a, const double* b, double* c, long long ra, long long k, long long rb,
                   cudaStream_t s);

// Separately rounded arithmetic (the reference is built without FMA contraction,
// SURVEY.md §0.3), for both instantiations.
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

}  // namespace hcb
