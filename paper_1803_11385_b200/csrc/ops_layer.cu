// ops_layer.cu — the rest of the reference's cnn_ops.hpp operator surface, in its layout
// (channel-major C x N feature matrices, fp32 and fp64): batch norm (cnn_ops.cpp:437-507),
// scale (509-546), ReLU (548-573) and inverted dropout (575-608). The native net has fused
// voxel-major versions of BN/ReLU (net_ops.cu); these serve callers of the reference API.
//
// Numerics follow the reference build (no FMA contraction: every product and sum is a
// separately rounded __*_rn): per-channel statistics are double sums — in a fixed tree
// order here instead of the reference's sequential loop, so the double sums can differ in
// their last bits; after the cast to float the results are identical except in vanishingly
// rare rounding ties (tests/test_layer_ops_gpu.py asserts equality for fp32). ReLU, scale
// forward and dropout (the reference's mt19937_64 stream, regenerated on the device) are
// bit-exact.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <stdexcept>

#include "hc_internal.h"
#include "hc_launch.cuh"

namespace hcb {
namespace {

constexpr int kBnThreads = 512;
constexpr int kT = 256;

__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// fixed-shape tree over the block (deterministic for a given launch shape)
template <int NT>
__device__ double block_sum(double v, double* red) {
    red[threadIdx.x] = v;
    __syncthreads();
#pragma unroll
    for (int w = NT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// cnn_ops.cpp:450-480: one block per channel — statistics (training) or running stats
// (inference), the running-stat update, inv_std, then y = (x - T(mean)) * inv_std.
template <typename T>
__global__ void __launch_bounds__(kBnThreads) k_bn_forward(const T* __restrict__ x, long long n, T* rmean, T* rvar,
                                                           T eps, T momentum, int training, T* __restrict__ y,
                                                           T* __restrict__ inv_std_out) {
    __shared__ double red[kBnThreads];
    const int c = blockIdx.x;
    const T* xr = x + (long long)c * n;
    double mean, var;
    if (training) {
        double s = 0;
        for (long long j = threadIdx.x; j < n; j += kBnThreads) s = __dadd_rn(s, (double)xr[j]);
        mean = __ddiv_rn(block_sum<kBnThreads>(s, red), (double)n);
        double s2 = 0;
        for (long long j = threadIdx.x; j < n; j += kBnThreads) {
            const double d = __dsub_rn((double)xr[j], mean);
            s2 = __dadd_rn(s2, __dmul_rn(d, d));
        }
        var = __ddiv_rn(block_sum<kBnThreads>(s2, red), (double)n);
        if (threadIdx.x == 0) {  // cnn_ops.cpp:468-469, T arithmetic
            const T keep = sub_rn(T(1), momentum);
            rmean[c] = add_rn(mul_rn(keep, rmean[c]), mul_rn(momentum, static_cast<T>(mean)));
            rvar[c] = add_rn(mul_rn(keep, rvar[c]), mul_rn(momentum, static_cast<T>(var)));
        }
    } else {
        mean = (double)rmean[c];
        var = (double)rvar[c];
    }
    const T inv_std = static_cast<T>(__ddiv_rn(1.0, sqrt(__dadd_rn(var, (double)eps))));
    const T m = static_cast<T>(mean);
    T* yr = y + (long long)c * n;
    for (long long j = threadIdx.x; j < n; j += kBnThreads) yr[j] = mul_rn(sub_rn(xr[j], m), inv_std);
    if (threadIdx.x == 0 && inv_std_out) inv_std_out[c] = inv_std;
}

// cnn_ops.cpp:484-507
template <typename T>
__global__ void __launch_bounds__(kBnThreads) k_bn_backward(const T* __restrict__ dy, const T* __restrict__ xh,
                                                            const T* __restrict__ inv_std, long long n,
                                                            T* __restrict__ dx) {
    __shared__ double red[kBnThreads];
    const int c = blockIdx.x;
    const T* dyr = dy + (long long)c * n;
    const T* xr = xh + (long long)c * n;
    double s1 = 0, s2 = 0;
    for (long long j = threadIdx.x; j < n; j += kBnThreads) {
        s1 = __dadd_rn(s1, (double)dyr[j]);
        s2 = __dadd_rn(s2, __dmul_rn((double)dyr[j], (double)xr[j]));
    }
    s1 = block_sum<kBnThreads>(s1, red);
    s2 = block_sum<kBnThreads>(s2, red);
    const double inv_n = __ddiv_rn(1.0, (double)n);
    const double istd = (double)inv_std[c];
    T* dxr = dx + (long long)c * n;
    for (long long j = threadIdx.x; j < n; j += kBnThreads) {
        // istd * (dy - s1 * inv_n - xh * s2 * inv_n), left to right, each step rounded
        const double a = __dsub_rn((double)dyr[j], __dmul_rn(s1, inv_n));
        const double b = __dmul_rn(__dmul_rn((double)xr[j], s2), inv_n);
        dxr[j] = static_cast<T>(__dmul_rn(istd, __dsub_rn(a, b)));
    }
}

// cnn_ops.cpp:509-522: y = g * x + b (separate rounding)
template <typename T>
__global__ void k_scale_forward(const T* __restrict__ x, long long rows, long long cols, const T* __restrict__ g,
                                const T* __restrict__ b, T* __restrict__ y) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= rows * cols) return;
    const long long r = i / cols;
    y[i] = add_rn(mul_rn(g[r], x[i]), b[r]);
}

// cnn_ops.cpp:525-546: per channel double sums -> T; dx = gamma * dy
template <typename T>
__global__ void __launch_bounds__(kBnThreads) k_scale_backward(const T* __restrict__ dy, const T* __restrict__ x,
                                                               const T* __restrict__ gamma, long long cols,
                                                               T* __restrict__ dgamma, T* __restrict__ dbeta,
                                                               T* __restrict__ dx) {
    __shared__ double red[kBnThreads];
    const int r = blockIdx.x;
    const T* dyr = dy + (long long)r * cols;
    const T* xr = x + (long long)r * cols;
    T* dxr = dx + (long long)r * cols;
    const T g = gamma[r];
    double sg = 0, sb = 0;
    for (long long j = threadIdx.x; j < cols; j += kBnThreads) {
        sg = __dadd_rn(sg, __dmul_rn((double)dyr[j], (double)xr[j]));
        sb = __dadd_rn(sb, (double)dyr[j]);
        dxr[j] = mul_rn(g, dyr[j]);
    }
    sg = block_sum<kBnThreads>(sg, red);
    sb = block_sum<kBnThreads>(sb, red);
    if (threadIdx.x == 0) {
        dgamma[r] = static_cast<T>(sg);
        dbeta[r] = static_cast<T>(sb);
    }
}

// cnn_ops.cpp:548-573: std::max(T(0), x) == (0 < x ? x : 0); backward passes dy where out > 0
template <typename T>
__global__ void k_relu_forward(const T* __restrict__ x, long long total, T* __restrict__ y) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < total) y[i] = T(0) < x[i] ? x[i] : T(0);
}
template <typename T>
__global__ void k_relu_backward(const T* __restrict__ dy, const T* __restrict__ out, long long total,
                                T* __restrict__ dx) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < total) dx[i] = out[i] > T(0) ? dy[i] : T(0);
}

// ----------------------------------------------------------------- mt19937_64 (rng.hpp:11-24)
// The reference draws its dropout mask from std::mt19937_64(seed), one uniform_float per
// element in order (cnn_ops.cpp:585-592). One CTA regenerates that exact stream: the state
// is seeded by thread 0, each 312-word twist runs in three dependency phases across the
// threads, and every word of a twist is tempered and consumed by one thread.
constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull, kMtUpper = 0xFFFFFFFF80000000ull, kMtLower = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t mt_mix(uint64_t hi_src, uint64_t lo_src, uint64_t far) {
    const uint64_t y = (hi_src & kMtUpper) | (lo_src & kMtLower);
    return far ^ (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}
__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= (y >> 43);
    return y;
}

template <typename T>
__global__ void __launch_bounds__(320) k_dropout_forward(const T* __restrict__ x, long long total, uint64_t seed,
                                                         float ratio_f, T scale, T* __restrict__ y,
                                                         uint8_t* __restrict__ keep) {
    __shared__ uint64_t mt[kMtN];
    const int t = threadIdx.x;
    if (t == 0) {  // std::mersenne_twister_engine::seed
        uint64_t v = seed;
        mt[0] = v;
        for (int i = 1; i < kMtN; ++i) {
            v = 6364136223846793005ull * (v ^ (v >> 62)) + (uint64_t)i;
            mt[i] = v;
        }
    }
    __syncthreads();
    for (long long base = 0; base < total; base += kMtN) {
        // twist (libstdc++ _M_gen_rand order): k < n-m from old words; n-m <= k < n-1 from the
        // new mt[k-(n-m)]; k = n-1 from the new mt[0] and mt[m-1]
        uint64_t nv = 0;
        if (t < kMtN - kMtM) nv = mt_mix(mt[t], mt[t + 1], mt[t + kMtM]);
        __syncthreads();
        if (t < kMtN - kMtM) mt[t] = nv;
        __syncthreads();
        if (t >= kMtN - kMtM && t < kMtN - 1) nv = mt_mix(mt[t], mt[t + 1], mt[t - (kMtN - kMtM)]);
        __syncthreads();
        if (t >= kMtN - kMtM && t < kMtN - 1) mt[t] = nv;
        __syncthreads();
        if (t == kMtN - 1) mt[t] = mt_mix(mt[kMtN - 1], mt[0], mt[kMtM - 1]);
        __syncthreads();
        const long long i = base + t;
        if (t < kMtN && i < total) {
            const uint64_t u = mt_temper(mt[t]);
            const float uf = static_cast<float>(static_cast<uint32_t>(u >> 40)) * 0x1.0p-24f;  // uniform_float
            const bool k = uf >= ratio_f;
            keep[i] = k ? 1 : 0;
            y[i] = k ? mul_rn(x[i], scale) : T(0);
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void k_dropout_backward(const T* __restrict__ dy, const uint8_t* __restrict__ keep, long long total, T scale,
                                   T* __restrict__ dx) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < total) dx[i] = keep[i] ? mul_rn(dy[i], scale) : T(0);
}

__global__ void k_fill_u8(uint8_t* p, long long n, uint8_t v) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// ----------------------------------------------------------------- host
template <typename T>
hc_status bn_forward(const T* x, int64_t c, int64_t n, T* rmean, T* rvar, int64_t stats_channels, T eps, T momentum,
                     int32_t training, T* y, T* inv_std, hc_stream stream) {
    return guard([&] {
        if (stats_channels != c) throw std::invalid_argument("batch_norm: stats channel mismatch");
        if (n == 0) throw std::invalid_argument("batch_norm: empty input");
        if (c == 0) return;
        k_bn_forward<T><<<(unsigned)c, kBnThreads, 0, as_stream(stream)>>>(x, n, rmean, rvar, eps, momentum,
                                                                           training, y, inv_std);
        launched("batch_norm_forward");
    });
}

template <typename T>
hc_status bn_backward(const T* dy, int64_t c, int64_t n, const T* normalized, int64_t nrows, int64_t ncols,
                      const T* inv_std, T* dx, hc_stream stream) {
    return guard([&] {
        if (nrows != c || ncols != n) throw std::invalid_argument("batch_norm_backward: cache shape mismatch");
        if (c == 0 || n == 0) return;
        k_bn_backward<T><<<(unsigned)c, kBnThreads, 0, as_stream(stream)>>>(dy, normalized, inv_std, n, dx);
        launched("batch_norm_backward");
    });
}

template <typename T>
hc_status scale_fwd(const T* x, int64_t rows, int64_t cols, const T* gamma, int64_t ng, const T* beta, int64_t nb,
                    T* y, hc_stream stream) {
    return guard([&] {
        if (ng != rows || ng != nb) throw std::invalid_argument("scale: parameter channel mismatch");
        if (rows * cols == 0) return;
        k_scale_forward<T><<<grid_for(rows * cols, kT), kT, 0, as_stream(stream)>>>(x, rows, cols, gamma, beta, y);
        launched("scale_forward");
    });
}

template <typename T>
hc_status scale_bwd(const T* dy, const T* x, int64_t rows, int64_t cols, const T* gamma, T* dgamma, T* dbeta, T* dx,
                    hc_stream stream) {
    return guard([&] {
        if (rows == 0) return;
        k_scale_backward<T><<<(unsigned)rows, kBnThreads, 0, as_stream(stream)>>>(dy, x, gamma, cols, dgamma, dbeta,
                                                                                  dx);
        launched("scale_backward");
    });
}

template <typename T>
hc_status relu_fwd(const T* x, int64_t total, T* y, hc_stream stream) {
    return guard([&] {
        if (total <= 0) return;
        k_relu_forward<T><<<grid_for(total, kT), kT, 0, as_stream(stream)>>>(x, total, y);
        launched("relu_forward");
    });
}

template <typename T>
hc_status relu_bwd(const T* dy, int64_t dr, int64_t dc, const T* out, int64_t orows, int64_t ocols, T* dx,
                   hc_stream stream) {
    return guard([&] {
        if (dr != orows || dc != ocols) throw std::invalid_argument("relu_backward: shape mismatch");
        if (dr * dc == 0) return;
        k_relu_backward<T><<<grid_for(dr * dc, kT), kT, 0, as_stream(stream)>>>(dy, out, dr * dc, dx);
        launched("relu_backward");
    });
}

template <typename T>
T dropout_scale(T ratio) {  // T(1) / (T(1) - ratio), in T
    return T(1) / (T(1) - ratio);
}

template <typename T>
hc_status dropout_fwd(const T* x, int64_t total, T ratio, uint64_t seed, int32_t training, T* y, uint8_t* keep,
                      hc_stream stream) {
    return guard([&] {
        if (ratio < T(0) || ratio >= T(1)) throw std::invalid_argument("dropout ratio must be in [0,1)");
        cudaStream_t s = as_stream(stream);
        if (total <= 0) return;
        if (!training || ratio == T(0)) {  // identity, mask all ones (cnn_ops.cpp:580-583)
            if (y != x) cuda_check(cudaMemcpyAsync(y, x, sizeof(T) * total, cudaMemcpyDeviceToDevice, s), "copy");
            if (keep) {
                k_fill_u8<<<grid_for(total, kT), kT, 0, s>>>(keep, total, 1);
                launched("dropout mask");
            }
            return;
        }
        if (!keep) throw std::invalid_argument("dropout: training mode needs a mask buffer");
        k_dropout_forward<T><<<1, 320, 0, s>>>(x, total, seed, static_cast<float>(ratio), dropout_scale(ratio), y, keep);
        launched("dropout_forward");
    });
}

template <typename T>
hc_status dropout_bwd(const T* dy, int64_t total, const uint8_t* keep, int64_t keep_size, T ratio, T* dx,
                      hc_stream stream) {
    return guard([&] {
        if (keep_size != total) throw std::invalid_argument("dropout_backward: mask size mismatch");
        if (total <= 0) return;
        k_dropout_backward<T><<<grid_for(total, kT), kT, 0, as_stream(stream)>>>(dy, keep, total,
                                                                                dropout_scale(ratio), dx);
        launched("dropout_backward");
    });
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

#define HC_LAYER_ABI(T, S)                                                                                           \
    hc_status hc_batch_norm_forward_##S(const T* x, int64_t c, int64_t n, T* running_mean, T* running_var,          \
                                        int64_t stats_channels, T eps, T momentum, int32_t training, T* y,          \
                                        T* inv_std, hc_stream stream) {                                             \
        return bn_forward<T>(x, c, n, running_mean, running_var, stats_channels, eps, momentum, training, y,        \
                             inv_std, stream);                                                                      \
    }                                                                                                                \
    hc_status hc_batch_norm_backward_##S(const T* dy, int64_t c, int64_t n, const T* normalized, int64_t nrows,    \
                                         int64_t ncols, const T* inv_std, T* dx, hc_stream stream) {                \
        return bn_backward<T>(dy, c, n, normalized, nrows, ncols, inv_std, dx, stream);                             \
    }                                                                                                                \
    hc_status hc_scale_forward_##S(const T* x, int64_t rows, int64_t cols, const T* gamma, int64_t n_gamma,        \
                                   const T* beta, int64_t n_beta, T* y, hc_stream stream) {                         \
        return scale_fwd<T>(x, rows, cols, gamma, n_gamma, beta, n_beta, y, stream);                                \
    }                                                                                                                \
    hc_status hc_scale_backward_##S(const T* dy, const T* x, int64_t rows, int64_t cols, const T* gamma,           \
                                    T* d_gamma, T* d_beta, T* dx, hc_stream stream) {                               \
        return scale_bwd<T>(dy, x, rows, cols, gamma, d_gamma, d_beta, dx, stream);                                 \
    }                                                                                                                \
    hc_status hc_relu_forward_##S(const T* x, int64_t total, T* y, hc_stream stream) {                             \
        return relu_fwd<T>(x, total, y, stream);                                                                    \
    }                                                                                                                \
    hc_status hc_relu_backward_##S(const T* dy, int64_t rows, int64_t cols, const T* forward_out, int64_t o_rows,  \
                                   int64_t o_cols, T* dx, hc_stream stream) {                                       \
        return relu_bwd<T>(dy, rows, cols, forward_out, o_rows, o_cols, dx, stream);                                \
    }                                                                                                                \
    hc_status hc_dropout_forward_##S(const T* x, int64_t total, T ratio, uint64_t seed, int32_t training, T* y,    \
                                     uint8_t* keep, hc_stream stream) {                                             \
        return dropout_fwd<T>(x, total, ratio, seed, training, y, keep, stream);                                    \
    }                                                                                                                \
    hc_status hc_dropout_backward_##S(const T* dy, int64_t total, const uint8_t* keep, int64_t keep_size, T ratio, \
                                      T* dx, hc_stream stream) {                                                    \
        return dropout_bwd<T>(dy, total, keep, keep_size, ratio, dx, stream);                                       \
    }

HC_LAYER_ABI(float, f32)
HC_LAYER_ABI(double, f64)
#undef HC_LAYER_ABI

}  // extern "C"
