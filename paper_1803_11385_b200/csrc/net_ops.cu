// net_ops.cu — the native (voxel-major) layers around the hash conv: max pooling with
// switches and its unpooling, batch norm + ReLU (forward and backward), and the final
// 2^3 dense pool of the classification head. These are the net.cpp:181-323 block
// operators (conv -> batch_norm -> relu -> max_pool, cnn_ops.cpp:234-284, 336-372,
// 437-489, 542-561; final_dense_pool net.cpp:69-122) on [N][C] feature rows, so every
// thread moves whole 16-byte channel chunks (8 bf16 or 4 fp32 channels) instead of
// the reference layout's strided single channels.
//
// Pool maps come from hc_field_map (row-major [N_coarse][F^3], F = S = 2): field row t of
// coarse voxel p is the fine column pmap[p][t] or -1. Pooling fields with F == S tile the
// fine level, so every fine voxel has at most one parent; hc_native_pool_parents inverts
// the map once per level pair (parent column + field row), which makes unpooling a
// coalesced pull instead of a scatter.
//
// Batch statistics are reduced in a fixed order (per-block double partials, then one
// ordered pass) -> deterministic; mean/var/inv_std follow cnn_ops.cpp:455-474 (two-pass,
// biased variance, double accumulation, inv_std = 1/sqrt(var + eps)).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "hashconv_b200_native.h"
#include "hc_internal.h"
#include "hc_launch.cuh"
#include "x2_layout.cuh"

namespace hcb {
namespace {

using bf16 = __nv_bfloat16;
constexpr int kT = 256;

// 8 channels of one row as floats (bf16: one 16-byte load; fp32: two)
__device__ __forceinline__ void load8(const bf16* p, float (&v)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}
__device__ __forceinline__ void store8(bf16* p, const float (&v)[8]) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

// ---------------------------------------------------------------------- pooling
__global__ void k_pool_parents(const int* __restrict__ pmap, long long nc, int fd, int* __restrict__ parent,
                               signed char* __restrict__ prow) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // over nc * fd
    if (i >= nc * fd) return;
    const int g = pmap[i];
    if (g < 0) return;
    parent[g] = (int)(i / fd);
    prow[g] = (signed char)(i % fd);
}

// cnn_ops.cpp:234-284: per channel, the first present field row seeds the max and a
// later row replaces it only if strictly greater; an empty field gives 0 and switch -1.
// OT: the output element type (T, or bf16 with SPLIT: the split-precision rows [nc][2C] the next
// conv consumes, so no separate split pass).
template <typename T, int FD, typename OT = T, bool SPLIT = false>
__global__ void __launch_bounds__(kT) k_nmax_pool(const int* __restrict__ pmap, long long nc, const T* __restrict__ x,
                                                 int C, OT* __restrict__ y, signed char* __restrict__ sw) {
    const int chunks = C >> 3;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // over nc * chunks
    if (i >= nc * chunks) return;
    const long long p = i / chunks;
    const int c0 = (int)(i - p * chunks) * 8;
    float best[8];
    int arg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        best[e] = 0.0f;
        arg[e] = -1;
    }
#pragma unroll
    for (int t = 0; t < FD; ++t) {
        const int g = __ldg(pmap + p * FD + t);
        if (g < 0) continue;
        float v[8];
        load8(x + (long long)g * C + c0, v);
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (arg[e] < 0 || v[e] > best[e]) {
                best[e] = v[e];
                arg[e] = t;
            }
    }
    if constexpr (SPLIT) store8_split(y + p * 2 * C, c0, C, best);
    else store8(y + p * C + c0, best);
    char4 s0 = make_char4(arg[0], arg[1], arg[2], arg[3]), s1 = make_char4(arg[4], arg[5], arg[6], arg[7]);
    *reinterpret_cast<int2*>(sw + p * C + c0) = make_int2(*reinterpret_cast<int*>(&s0), *reinterpret_cast<int*>(&s1));
}

// cnn_ops.cpp:336-372 with one covering output per fine voxel (F == S): the fine
// voxel takes the coarse gradient where the coarse switch names its field row.
template <typename T>
__global__ void __launch_bounds__(kT) k_nmax_unpool(const int* __restrict__ parent, const signed char* __restrict__ prow,
                                                   long long nf, const T* __restrict__ dy,
                                                   const signed char* __restrict__ sw, int C, T* __restrict__ dx,
                                                   float* __restrict__ acc = nullptr) {
    const int chunks = C >> 3;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // over nf * chunks
    if (i >= nf * chunks) return;
    const long long g = i / chunks;
    const int c0 = (int)(i - g * chunks) * 8;
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = 0.0f;
    const int p = __ldg(parent + g);
    if (p >= 0) {
        const int r = __ldg(prow + g);
        float v[8];
        load8(dy + (long long)p * C + c0, v);
        const int2 s = __ldg(reinterpret_cast<const int2*>(sw + (long long)p * C + c0));
        const signed char* sc = reinterpret_cast<const signed char*>(&s);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = sc[e] == r ? 0.0f + v[e] : 0.0f;
    }
    if (acc) {  // acc += the unpooled row (o is exact in T: what acc.add_(unpooled row) computes)
        float a[8];
        load8(acc + g * C + c0, a);
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] = __fadd_rn(a[e], o[e]);
        store8(acc + g * C + c0, a);
        return;
    }
    store8(dx + g * C + c0, o);
}

// Adjoint of max_unpool (= the max pool's forward selection applied to a gradient):
// out[p][c] = fine[pmap[p][sw[p][c]]][c], 0 where the switch is -1.
template <typename T>
__global__ void __launch_bounds__(kT) k_switch_gather(const int* __restrict__ pmap, long long nc, int fd,
                                                     const T* __restrict__ fine, const signed char* __restrict__ sw,
                                                     int C, T* __restrict__ out) {
    const int chunks = C >> 3;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nc * chunks) return;
    const long long p = i / chunks;
    const int c0 = (int)(i - p * chunks) * 8;
    const int2 s = __ldg(reinterpret_cast<const int2*>(sw + p * C + c0));
    const signed char* sc = reinterpret_cast<const signed char*>(&s);
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        o[e] = 0.0f;
        if (sc[e] >= 0) {
            const int g = __ldg(pmap + p * fd + sc[e]);
            if (g >= 0) {
                if constexpr (sizeof(T) == 2) o[e] = __bfloat162float(fine[(long long)g * C + c0 + e]);
                else o[e] = fine[(long long)g * C + c0 + e];
            }
        }
    }
    store8(out + p * C + c0, o);
}

// ---------------------------------------------------------------------- batch norm + ReLU
// Column partial sums over row blocks: thread (r, q) owns channel quad q of rows
// r, r + R, ... inside the block's row range; partials [block][C] in double.
// MODE 0: sum x; 1: sum (x - mean)^2; 2: (sum dyb, sum dyb*xhat) with dyb = dy*(xhat > 0).
// Rows per partial block: enough blocks for ~4 per SM (the statistics of a small level are
// otherwise a few long serial chains), at most 1024; fixed for a given n -> deterministic.
inline int bn_rows_per_block(long long n) {
    long long r = (n + 591) / 592;
    r = (r + 63) / 64 * 64;
    return (int)(r < 64 ? 64 : r > 1024 ? 1024 : r);
}
inline int bn_blocks(long long n) { return (int)((n + bn_rows_per_block(n) - 1) / bn_rows_per_block(n)); }

template <int MODE, typename DT>
__global__ void __launch_bounds__(kT) k_col_partials(const float* __restrict__ a, const DT* __restrict__ b, long long n,
                                                    int C, const double* __restrict__ mean, double* __restrict__ part,
                                                    int rpb) {
    const int quads = C >> 2;
    const int R = kT / quads;  // rows in flight per block step
    const int q = threadIdx.x % quads, r = threadIdx.x / quads;
    __shared__ double red[2][kT * 4];
    double s[4] = {0, 0, 0, 0}, t[4] = {0, 0, 0, 0};
    if (r < R) {
        const long long r0 = (long long)blockIdx.x * rpb;
        const long long r1 = min(n, r0 + rpb);
        double mu[4] = {0, 0, 0, 0};
        if (MODE == 1)
#pragma unroll
            for (int e = 0; e < 4; ++e) mu[e] = mean[q * 4 + e];
#pragma unroll 4
        for (long long row = r0 + r; row < r1; row += R) {  // unrolled: 4 row loads in flight per thread
            const float4 x = __ldg(reinterpret_cast<const float4*>(a + row * C + q * 4));
            const float xv[4] = {x.x, x.y, x.z, x.w};
            if (MODE == 2) {
                float dv[4];
                if constexpr (sizeof(DT) == 2) {
                    const uint2 u = __ldg(reinterpret_cast<const uint2*>(b + row * C + q * 4));
                    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
                    const float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
                    dv[0] = f0.x, dv[1] = f0.y, dv[2] = f1.x, dv[3] = f1.y;
                } else {
                    const float4 d = __ldg(reinterpret_cast<const float4*>(b + row * C + q * 4));
                    dv[0] = d.x, dv[1] = d.y, dv[2] = d.z, dv[3] = d.w;
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double g = xv[e] > 0.0f ? (double)dv[e] : 0.0;
                    s[e] += g;
                    t[e] += g * xv[e];
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double d = MODE == 1 ? (double)xv[e] - mu[e] : (double)xv[e];
                    s[e] += MODE == 1 ? d * d : d;
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        red[0][threadIdx.x * 4 + e] = s[e];
        red[1][threadIdx.x * 4 + e] = t[e];
    }
    __syncthreads();
    if (threadIdx.x < C) {  // fixed-order fold over the R row lanes of channel c
        const int c = threadIdx.x, cq = c >> 2, ce = c & 3;
        double u = 0, v = 0;
        for (int rr = 0; rr < R; ++rr) {
            u += red[0][(rr * quads + cq) * 4 + ce];
            v += red[1][(rr * quads + cq) * 4 + ce];
        }
        part[((long long)blockIdx.x * 2 + 0) * C + c] = u;
        part[((long long)blockIdx.x * 2 + 1) * C + c] = v;
    }
}

// Fold the per-block partials in block order; MODE 0 -> mean, MODE 1 -> var and the
// running-stat update (cnn_ops.cpp:463-470), MODE 2 -> backward sums.
template <int MODE>
__global__ void k_col_fold(const double* __restrict__ part, int blocks, long long n, int C, double* __restrict__ out0,
                           double* __restrict__ out1, float* __restrict__ run_mean, float* __restrict__ run_var,
                           float momentum, float eps, const double* __restrict__ mean, float* __restrict__ inv_std) {
    // one block per channel: thread j folds partial blocks j, j + kT, ..., then a fixed-shape
    // tree over the kT lanes (deterministic for a given partial count)
    const int c = blockIdx.x;
    __shared__ double su[kT], sv[kT];
    double u = 0, v = 0;
    for (int b = threadIdx.x; b < blocks; b += kT) {
        u += part[((long long)b * 2 + 0) * C + c];
        v += part[((long long)b * 2 + 1) * C + c];
    }
    su[threadIdx.x] = u;
    sv[threadIdx.x] = v;
    __syncthreads();
    for (int w = kT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            su[threadIdx.x] += su[threadIdx.x + w];
            sv[threadIdx.x] += sv[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    u = su[0];
    v = sv[0];
    if (MODE == 0) {
        out0[c] = u / (double)n;
    } else if (MODE == 1) {
        const double var = u / (double)n;
        out1[c] = var;
        if (run_mean) {
            run_mean[c] = (1.0f - momentum) * run_mean[c] + momentum * (float)mean[c];
            run_var[c] = (1.0f - momentum) * run_var[c] + momentum * (float)var;
        }
        inv_std[c] = (float)(1.0 / sqrt(var + (double)eps));
    } else {
        out0[c] = u;
        out1[c] = v;
    }
}

// Batch-norm statistics from the conv epilogue's per-tile {sum, centred sum of squares}
// (hc_native_gather_gemm*_stats): one block per channel, two passes in double over the
// tiles, each a per-thread sum over a contiguous tile range (4 loads in flight) and a
// fixed-shape tree: the mean S / n, then the exact decomposition
//   M2 = sum_t [ M2_t + n_t (s_t / n_t - mean)^2 ]
// (no division per tile: n_t = 128 except the last tile), -> biased variance
// (cnn_ops.cpp:455-466), running stats and inv_std as k_col_fold MODE 1 forms them.
// Deterministic; replaces a serial Chan merge (a double division chain per tile).
__device__ __forceinline__ double block_sum_fixed(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int w = kT / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kT) k_bn_fold_tiles(const float2* __restrict__ st, long long tiles, long long n,
                                                     int C, float* __restrict__ run_mean, float* __restrict__ run_var,
                                                     float momentum, float eps, double* __restrict__ mean_out,
                                                     float* __restrict__ inv_std) {
    const int c = blockIdx.x;
    __shared__ double sh[kT];
    const long long t0 = tiles * threadIdx.x / kT, t1 = tiles * (threadIdx.x + 1) / kT;
    double s = 0.0;
    long long t = t0;
    for (; t + 4 <= t1; t += 4) {
        const float a = st[t * C + c].x, b = st[(t + 1) * C + c].x, d = st[(t + 2) * C + c].x,
                    e = st[(t + 3) * C + c].x;
        s += (double)a;
        s += (double)b;
        s += (double)d;
        s += (double)e;
    }
    for (; t < t1; ++t) s += (double)st[t * C + c].x;
    const double mu = block_sum_fixed(s, sh) / (double)n;
    double m2 = 0.0;
    const long long full = n / 128;  // tiles [0, full) hold 128 voxels
    for (t = t0; t < t1; ++t) {
        const float2 v = st[t * C + c];
        const double nt = t < full ? 128.0 : (double)(n - t * 128);
        const double d = (double)v.x * (t < full ? 0.0078125 : 1.0 / nt) - mu;
        m2 += (double)v.y + nt * d * d;
    }
    const double var = block_sum_fixed(m2, sh) / (double)n;
    if (threadIdx.x != 0) return;
    mean_out[c] = mu;
    run_mean[c] = (1.0f - momentum) * run_mean[c] + momentum * (float)mu;
    run_var[c] = (1.0f - momentum) * run_var[c] + momentum * (float)var;
    inv_std[c] = (float)(1.0 / sqrt(var + (double)eps));
}

// Synchronised (data-parallel) batch norm: statistics from sums taken over the GLOBAL batch
// (all-reduced by the caller). sum_sq == nullptr: mean = sum_x / n_total; otherwise
// var = sum_sq / n_total (biased, cnn_ops.cpp:463-466), running stats, inv_std — the same
// arithmetic as k_col_fold MODE 0 / 1, so one rank reproduces the fused call bit for bit.
__global__ void k_bn_finalize(const double* __restrict__ sum_x, const double* __restrict__ sum_sq, long long n_total,
                              int C, float* __restrict__ run_mean, float* __restrict__ run_var, float momentum,
                              float eps, double* __restrict__ mean, float* __restrict__ inv_std) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    if (!sum_sq) {
        mean[c] = sum_x[c] / (double)n_total;
        return;
    }
    const double var = sum_sq[c] / (double)n_total;
    if (run_mean) {
        run_mean[c] = (1.0f - momentum) * run_mean[c] + momentum * (float)mean[c];
        run_var[c] = (1.0f - momentum) * run_var[c] + momentum * (float)var;
    }
    inv_std[c] = (float)(1.0 / sqrt(var + (double)eps));
}

// xhat = (x - mean) * inv_std (float, cnn_ops.cpp:472); out = relu(xhat) (bf16 for the
// next layer); xhat kept (fp32) for the backward pass.
template <typename OT>
__global__ void __launch_bounds__(kT) k_bn_relu_apply(const float* __restrict__ x, long long n, int C,
                                                     const double* __restrict__ mean,
                                                     const float* __restrict__ inv_std, float* __restrict__ xhat,
                                                     OT* __restrict__ out) {
    const int chunks = C >> 3;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n * chunks) return;
    const long long row = i / chunks;
    const int c0 = (int)(i - row * chunks) * 8;
    float v[8], h[8], o[8];
    load8(x + row * C + c0, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        h[e] = (v[e] - (float)mean[c0 + e]) * inv_std[c0 + e];
        o[e] = fmaxf(0.0f, h[e]);
    }
    if (xhat) store8(xhat + row * C + c0, h);
    store8(out + row * C + c0, o);
}

// Inference batch norm + ReLU (cnn_ops.cpp:470-475 with training = false): the running
// statistics stand in for the batch's, inv_std = T(1 / sqrt(double(var) + eps)),
// y = (x - T(mean)) * inv_std, out = max(0, y) (bf16 for the next layer).
template <typename OT>
__global__ void __launch_bounds__(kT) k_bn_relu_infer(const float* __restrict__ x, long long n, int C,
                                                     const float* __restrict__ rmean, const float* __restrict__ rvar,
                                                     float eps, OT* __restrict__ out) {
    const int chunks = C >> 3;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n * chunks) return;
    const long long row = i / chunks;
    const int c0 = (int)(i - row * chunks) * 8;
    float v[8], o[8];
    load8(x + row * C + c0, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float inv = (float)(1.0 / sqrt((double)rvar[c0 + e] + (double)eps));
        o[e] = fmaxf(0.0f, __fmul_rn(__fsub_rn(v[e], rmean[c0 + e]), inv));
    }
    store8(out + row * C + c0, o);
}

// dx = inv_std * (dyb - s1/n - xhat * s2/n), dyb = dy * (xhat > 0)  (cnn_ops.cpp:476-489
// after relu_backward cnn_ops.cpp:553-561); bf16 out = the conv layer's output gradient.
template <typename DT, typename OT, bool SPLIT = false>
__global__ void __launch_bounds__(kT) k_bn_relu_bwd_apply(const DT* __restrict__ dy, const float* __restrict__ xhat,
                                                         long long n, int C, const double* __restrict__ s1,
                                                         const double* __restrict__ s2,
                                                         const float* __restrict__ inv_std, OT* __restrict__ dx,
                                                         long long n_total) {
    const int chunks = C >> 3;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n * chunks) return;
    const long long row = i / chunks;
    const int c0 = (int)(i - row * chunks) * 8;
    float d[8], h[8], o[8];
    load8(dy + row * C + c0, d);
    load8(xhat + row * C + c0, h);
    const double inv_n = 1.0 / (double)n_total;  // the (global) batch the sums were taken over
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const double g = h[e] > 0.0f ? (double)d[e] : 0.0;
        o[e] = (float)((double)inv_std[c0 + e] * (g - s1[c0 + e] * inv_n - (double)h[e] * s2[c0 + e] * inv_n));
    }
    if constexpr (SPLIT) store8_split(dx + row * 2 * C, c0, C, o);
    else store8(dx + row * C + c0, o);
}

// ---------------------------------------------------------------------- final dense pool
// net.cpp:69-106: per model v and dense parent cell q of the 2^3 grid, max over the present
// resolution-4 children (first hit seeds, strict '>'); head_in[(c*8 + cell)][v], src = the
// winning fine column (-1 when the cell's field is empty). cmap: [b][8][8] child columns.
__device__ __forceinline__ float to_f(bf16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }

template <typename T>
__global__ void k_dense_pool(const int* __restrict__ cmap, int b, const T* __restrict__ x, int C,
                             float* __restrict__ head, int* __restrict__ src) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over b * 8 * C
    if (i >= b * 8 * C) return;
    const int c = i % C, cell = (i / C) % 8, v = i / (8 * C);
    const int* kids = cmap + (v * 8 + cell) * 8;
    float best = 0.0f;
    int col = -1;
    for (int k = 0; k < 8; ++k) {
        const int g = kids[k];
        if (g < 0) continue;
        const float val = to_f(x[(long long)g * C + c]);
        if (col < 0 || val > best) {
            best = val;
            col = g;
        }
    }
    head[(long long)(c * 8 + cell) * b + v] = col < 0 ? 0.0f : best;
    src[(c * 8 + cell) * b + v] = col;
}

// net.cpp:108-122: dx[c][src] += d_head (each fine column is the source of at most one
// (c, cell, v) entry per channel, so this is a plain scatter; dx pre-zeroed).
__global__ void k_dense_pool_bwd(const float* __restrict__ dhead, const int* __restrict__ src, int b, int C,
                                 float* __restrict__ dx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over C * 8 * b
    if (i >= C * 8 * b) return;
    const int col = src[i];
    if (col < 0) return;
    const int c = i / (8 * b);
    dx[(long long)col * C + c] += dhead[i];
}

// net.cpp:339-346 sgd_update: v = momentum*v + lr*(g + wd*w); w -= v (separate fp32
// roundings, as the reference's non-FMA build).
// Multi-tensor SGD: up to kSgdMax (w, v, g, n) tensors in one launch (a training step updates every
// conv and FC tensor; one launch instead of one per tensor). Tensor k owns blocks
// [first[k], first[k+1]); the per-element arithmetic is k_sgd's.
constexpr int kSgdMax = 32;
struct SgdList {
    float* w[kSgdMax];
    float* v[kSgdMax];
    const float* g[kSgdMax];
    long long n[kSgdMax];
    int first[kSgdMax + 1];
    int count;
};

__global__ void __launch_bounds__(kT) k_sgd_multi(const SgdList L, float lr, float momentum, float wd) {
    int k = 0;
    while (k + 1 < L.count && (int)blockIdx.x >= L.first[k + 1]) ++k;
    const long long i = (long long)(blockIdx.x - L.first[k]) * blockDim.x + threadIdx.x;
    if (i >= L.n[k]) return;
    float* w = L.w[k];
    float* v = L.v[k];
    const float vi = __fadd_rn(__fmul_rn(momentum, v[i]), __fmul_rn(lr, __fadd_rn(L.g[k][i], __fmul_rn(wd, w[i]))));
    v[i] = vi;
    w[i] = __fsub_rn(w[i], vi);
}

__global__ void k_sgd(float* __restrict__ w, float* __restrict__ v, const float* __restrict__ g, long long n, float lr,
                      float momentum, float wd) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float vi = __fadd_rn(__fmul_rn(momentum, v[i]), __fmul_rn(lr, __fadd_rn(g[i], __fmul_rn(wd, w[i]))));
    v[i] = vi;
    w[i] = __fsub_rn(w[i], vi);
}

void check_c8(int c) {
    if (c <= 0 || c % 8 != 0) throw std::invalid_argument("native net ops: channels must be a multiple of 8");
}

void check_out_dtype(hc_dtype t) {
    if (t != HC_DTYPE_BF16 && t != HC_DTYPE_F32) throw std::invalid_argument("native net op: output dtype must be bf16 or f32");
}
// the batch-norm backward may also write the split-precision rows its conv's dW / dX consume
void check_grad_out_dtype(hc_dtype t) {
    if (t != HC_DTYPE_BF16 && t != HC_DTYPE_F32 && t != HC_DTYPE_SPLIT)
        throw std::invalid_argument("native batch norm backward: output dtype must be bf16, f32 or split");
}

// out = relu(xhat) as bf16 or fp32 (the split-precision net keeps fp32 activations)
void bn_relu_apply_out(const float* x, long long n, int c, const double* mean, const float* inv_std, float* xhat,
                              void* out, hc_dtype out_dtype, cudaStream_t s) {
    const long long m = n * (c / 8);
    if (out_dtype == HC_DTYPE_F32)
        k_bn_relu_apply<float><<<grid_for(m, kT), kT, 0, s>>>(x, n, c, mean, inv_std, xhat, static_cast<float*>(out));
    else
        k_bn_relu_apply<bf16><<<grid_for(m, kT), kT, 0, s>>>(x, n, c, mean, inv_std, xhat, static_cast<bf16*>(out));
    launched("batch-norm + relu");
}

template <typename DT>
void bn_bwd_apply_out(const DT* d, const float* xhat, long long n, int c, const double* s1, const double* s2,
                             const float* inv_std, void* out, hc_dtype out_dtype, long long n_total, cudaStream_t s) {
    const long long m = n * (c / 8);
    if (out_dtype == HC_DTYPE_SPLIT)
        k_bn_relu_bwd_apply<DT, bf16, true><<<grid_for(m, kT), kT, 0, s>>>(d, xhat, n, c, s1, s2, inv_std,
                                                                           static_cast<bf16*>(out), n_total);
    else if (out_dtype == HC_DTYPE_F32)
        k_bn_relu_bwd_apply<DT, float><<<grid_for(m, kT), kT, 0, s>>>(d, xhat, n, c, s1, s2, inv_std,
                                                                      static_cast<float*>(out), n_total);
    else
        k_bn_relu_bwd_apply<DT, bf16><<<grid_for(m, kT), kT, 0, s>>>(d, xhat, n, c, s1, s2, inv_std,
                                                                     static_cast<bf16*>(out), n_total);
}

// Dropout (net.cpp:236-251) from uniform draws u: mask = (u < keep) / keep, out = x * mask — the
// same fp32 operations as the torch composition it replaces, in one pass.
__global__ void k_dropout_apply(const float* __restrict__ u, const float* __restrict__ x, long long n, float keep,
                                float* __restrict__ mask, float* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float m = u[i] < keep ? 1.0f / keep : 0.0f;
    mask[i] = m;
    out[i] = x[i] * m;
}

// Softmax cross-entropy of the net's scores [classes][b] (net.cpp:260-283) in one launch: warp
// w takes columns w, w + 32, ...; per column the class max, sum of exp (double), log-sum-exp, the
// label's negative log-probability and the scores' gradient (softmax - onehot) * inv_b. The loss
// is summed per warp over its columns in order, then over the warps in order (deterministic).
__global__ void __launch_bounds__(1024) k_softmax_xent(const float* __restrict__ scores, int classes, int b,
                                                       const long long* __restrict__ labels, double inv_b,
                                                       double* __restrict__ loss, float* __restrict__ dscores) {
    __shared__ double part[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double lsum = 0.0;
    for (int j = w; j < b; j += 32) {
        double m = -INFINITY;
        for (int k = lane; k < classes; k += 32) m = fmax(m, (double)scores[(long long)k * b + j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        double se = 0.0;
        for (int k = lane; k < classes; k += 32) se += exp((double)scores[(long long)k * b + j] - m);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const double lse = m + log(se);
        const long long lab = labels[j];
        for (int k = lane; k < classes; k += 32) {
            const double p = exp((double)scores[(long long)k * b + j] - lse);
            dscores[(long long)k * b + j] = (float)((p - (k == lab ? 1.0 : 0.0)) * inv_b);
        }
        if (lane == 0) lsum += lse - (double)scores[lab * b + j];
    }
    if (lane == 0) part[w] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < 32; ++q) t += part[q];
        loss[0] = t * inv_b;
    }
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

hc_status hc_native_pool_parents(const int32_t* pmap, int64_t n_coarse, int32_t fd, int64_t n_fine, int32_t* parent,
                                 int8_t* prow, hc_stream stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        if (n_fine > 0) cuda_check(cudaMemsetAsync(parent, 0xFF, sizeof(int32_t) * n_fine, s), "memset");
        if (n_coarse <= 0) return;
        k_pool_parents<<<grid_for(n_coarse * fd, kT), kT, 0, s>>>(pmap, n_coarse, fd, parent,
                                                                  reinterpret_cast<signed char*>(prow));
        launched("pool parents");
    });
}

hc_status hc_native_max_pool(const int32_t* pmap, int64_t n_coarse, int32_t fd, const void* x, hc_dtype dtype,
                             int32_t c, void* y, int8_t* switches, hc_stream stream) {
    return guard([&] {
        check_c8(c);
        if (fd != 8) throw std::invalid_argument("native max_pool: 2x2x2 fields (F = S = 2) only");
        if (n_coarse <= 0) return;
        cudaStream_t s = as_stream(stream);
        const long long n = n_coarse * (c / 8);
        signed char* sw = reinterpret_cast<signed char*>(switches);
        if (dtype == HC_DTYPE_BF16)
            k_nmax_pool<bf16, 8><<<grid_for(n, kT), kT, 0, s>>>(pmap, n_coarse, static_cast<const bf16*>(x), c,
                                                                static_cast<bf16*>(y), sw);
        else if (dtype == HC_DTYPE_SPLIT)  // fp32 input, split-precision output rows
            k_nmax_pool<float, 8, bf16, true><<<grid_for(n, kT), kT, 0, s>>>(
                pmap, n_coarse, static_cast<const float*>(x), c, static_cast<bf16*>(y), sw);
        else
            k_nmax_pool<float, 8><<<grid_for(n, kT), kT, 0, s>>>(pmap, n_coarse, static_cast<const float*>(x), c,
                                                                 static_cast<float*>(y), sw);
        launched("native max_pool");
    });
}

hc_status hc_native_max_unpool(const int32_t* parent, const int8_t* prow, int64_t n_fine, const void* dy,
                               hc_dtype dtype, int32_t c, const int8_t* switches, void* dx, hc_stream stream) {
    return guard([&] {
        check_c8(c);
        if (n_fine <= 0) return;
        cudaStream_t s = as_stream(stream);
        const long long n = n_fine * (c / 8);
        const signed char* pr = reinterpret_cast<const signed char*>(prow);
        const signed char* sw = reinterpret_cast<const signed char*>(switches);
        if (dtype == HC_DTYPE_BF16)
            k_nmax_unpool<bf16><<<grid_for(n, kT), kT, 0, s>>>(parent, pr, n_fine, static_cast<const bf16*>(dy), sw,
                                                               c, static_cast<bf16*>(dx));
        else
            k_nmax_unpool<float><<<grid_for(n, kT), kT, 0, s>>>(parent, pr, n_fine, static_cast<const float*>(dy), sw,
                                                                c, static_cast<float*>(dx));
        launched("native max_unpool");
    });
}

hc_status hc_native_max_unpool_add(const int32_t* parent, const int8_t* prow, int64_t n_fine, const void* dy,
                                   hc_dtype dtype, int32_t c, const int8_t* switches, float* acc,
                                   hc_stream stream) {
    return guard([&] {
        check_c8(c);
        if (!acc) throw std::invalid_argument("native max_unpool_add: null accumulator");
        if (n_fine <= 0) return;
        cudaStream_t s = as_stream(stream);
        const long long n = n_fine * (c / 8);
        const signed char* pr = reinterpret_cast<const signed char*>(prow);
        const signed char* sw = reinterpret_cast<const signed char*>(switches);
        if (dtype == HC_DTYPE_BF16)
            k_nmax_unpool<bf16><<<grid_for(n, kT), kT, 0, s>>>(parent, pr, n_fine, static_cast<const bf16*>(dy), sw,
                                                               c, nullptr, acc);
        else
            k_nmax_unpool<float><<<grid_for(n, kT), kT, 0, s>>>(parent, pr, n_fine, static_cast<const float*>(dy), sw,
                                                                c, nullptr, acc);
        launched("native max_unpool (accumulating)");
    });
}

hc_status hc_native_switch_gather(const int32_t* pmap, int64_t n_coarse, int32_t fd, const void* fine, hc_dtype dtype,
                                  int32_t c, const int8_t* switches, void* out, hc_stream stream) {
    return guard([&] {
        check_c8(c);
        if (n_coarse <= 0) return;
        cudaStream_t s = as_stream(stream);
        const long long n = n_coarse * (c / 8);
        const signed char* sw = reinterpret_cast<const signed char*>(switches);
        if (dtype == HC_DTYPE_BF16)
            k_switch_gather<bf16><<<grid_for(n, kT), kT, 0, s>>>(pmap, n_coarse, fd, static_cast<const bf16*>(fine), sw,
                                                                 c, static_cast<bf16*>(out));
        else
            k_switch_gather<float><<<grid_for(n, kT), kT, 0, s>>>(pmap, n_coarse, fd, static_cast<const float*>(fine),
                                                                  sw, c, static_cast<float*>(out));
        launched("switch gather");
    });
}

size_t hc_native_bn_workspace(int64_t n, int32_t c) {
    const long long blocks = bn_blocks(n);
    return (size_t)(blocks * 2 * c + 4 * c) * sizeof(double);
}

hc_status hc_native_bn_relu_forward(const float* x, int64_t n, int32_t c, int32_t training, float momentum, float eps,
                                    float* running_mean, float* running_var, float* inv_std, float* xhat,
                                    void* out_bf16, void* workspace, size_t ws_bytes, hc_stream stream) {
    return hc_native_bn_relu_forward_dt(x, n, c, training, momentum, eps, running_mean, running_var, inv_std, xhat,
                                        out_bf16, HC_DTYPE_BF16, workspace, ws_bytes, stream);
}

hc_status hc_native_bn_relu_forward_dt(const float* x, int64_t n, int32_t c, int32_t training, float momentum,
                                       float eps, float* running_mean, float* running_var, float* inv_std, float* xhat,
                                       void* out, hc_dtype out_dtype, void* workspace, size_t ws_bytes,
                                       hc_stream stream) {
    return guard([&] {
        check_out_dtype(out_dtype);
        check_c8(c);
        if (c > kT) throw std::invalid_argument("native batch norm: at most 256 channels");
        if (n <= 0) throw std::invalid_argument("batch_norm: empty input");
        if (ws_bytes < hc_native_bn_workspace(n, c)) throw std::invalid_argument("native batch norm: workspace too small");
        cudaStream_t s = as_stream(stream);
        const int blocks = bn_blocks(n);
        const int rpb = bn_rows_per_block(n);
        double* part = static_cast<double*>(workspace);
        double* mean = part + (long long)blocks * 2 * c;
        double* var = mean + c;
        if (training) {
            k_col_partials<0, float><<<blocks, kT, 0, s>>>(x, nullptr, n, c, nullptr, part, rpb);
            k_col_fold<0><<<c, kT, 0, s>>>(part, blocks, n, c, mean, nullptr, nullptr, nullptr, 0, 0, nullptr, nullptr);
            k_col_partials<1, float><<<blocks, kT, 0, s>>>(x, nullptr, n, c, mean, part, rpb);
            k_col_fold<1><<<c, kT, 0, s>>>(part, blocks, n, c, nullptr, var, running_mean, running_var, momentum, eps,
                                          mean, inv_std);
            launched("batch-norm statistics", 4);
        } else {
            throw std::invalid_argument("native batch norm: inference mode uses the reference-layout path");
        }
        bn_relu_apply_out(x, n, c, mean, inv_std, xhat, out, out_dtype, s);
    });
}

hc_status hc_native_bn_relu_backward(const void* d_relu, hc_dtype dtype, const float* xhat, const float* inv_std,
                                     int64_t n, int32_t c, void* d_conv_bf16, void* workspace, size_t ws_bytes,
                                     hc_stream stream) {
    return hc_native_bn_relu_backward_dt(d_relu, dtype, xhat, inv_std, n, c, d_conv_bf16, HC_DTYPE_BF16, workspace,
                                         ws_bytes, stream);
}

hc_status hc_native_bn_relu_backward_dt(const void* d_relu, hc_dtype dtype, const float* xhat, const float* inv_std,
                                        int64_t n, int32_t c, void* d_conv, hc_dtype out_dtype, void* workspace,
                                        size_t ws_bytes, hc_stream stream) {
    return guard([&] {
        check_grad_out_dtype(out_dtype);
        check_c8(c);
        if (c > kT) throw std::invalid_argument("native batch norm: at most 256 channels");
        if (n <= 0) return;
        if (ws_bytes < hc_native_bn_workspace(n, c)) throw std::invalid_argument("native batch norm: workspace too small");
        cudaStream_t s = as_stream(stream);
        const int blocks = bn_blocks(n);
        const int rpb = bn_rows_per_block(n);
        double* part = static_cast<double*>(workspace);
        double* s1 = part + (long long)blocks * 2 * c;
        double* s2 = s1 + c;
        if (dtype == HC_DTYPE_BF16) {
            const bf16* d = static_cast<const bf16*>(d_relu);
            k_col_partials<2, bf16><<<blocks, kT, 0, s>>>(xhat, d, n, c, nullptr, part, rpb);
            k_col_fold<2><<<c, kT, 0, s>>>(part, blocks, n, c, s1, s2, nullptr, nullptr, 0, 0, nullptr, nullptr);
            bn_bwd_apply_out(d, xhat, n, c, s1, s2, inv_std, d_conv, out_dtype, n, s);
        } else {
            const float* d = static_cast<const float*>(d_relu);
            k_col_partials<2, float><<<blocks, kT, 0, s>>>(xhat, d, n, c, nullptr, part, rpb);
            k_col_fold<2><<<c, kT, 0, s>>>(part, blocks, n, c, s1, s2, nullptr, nullptr, 0, 0, nullptr, nullptr);
            bn_bwd_apply_out(d, xhat, n, c, s1, s2, inv_std, d_conv, out_dtype, n, s);
        }
        launched("batch-norm + relu backward", 3);
    });
}

hc_status hc_native_bn_relu_inference(const float* x, int64_t n, int32_t c, const float* running_mean,
                                      const float* running_var, float eps, void* out_bf16, hc_stream stream) {
    return hc_native_bn_relu_inference_dt(x, n, c, running_mean, running_var, eps, out_bf16, HC_DTYPE_BF16, stream);
}

hc_status hc_native_bn_relu_inference_dt(const float* x, int64_t n, int32_t c, const float* running_mean,
                                         const float* running_var, float eps, void* out, hc_dtype out_dtype,
                                         hc_stream stream) {
    return guard([&] {
        check_c8(c);
        check_out_dtype(out_dtype);
        if (n <= 0) return;
        const long long m = n * (c / 8);
        cudaStream_t s = as_stream(stream);
        if (out_dtype == HC_DTYPE_F32)
            k_bn_relu_infer<float><<<grid_for(m, kT), kT, 0, s>>>(x, n, c, running_mean, running_var, eps,
                                                                  static_cast<float*>(out));
        else
            k_bn_relu_infer<bf16><<<grid_for(m, kT), kT, 0, s>>>(x, n, c, running_mean, running_var, eps,
                                                                 static_cast<bf16*>(out));
        launched("batch-norm (inference) + relu");
    });
}

hc_status hc_native_bn_relu_forward_tiles(const float* tile_stats, int64_t n, int32_t c, float momentum, float eps,
                                          float* running_mean, float* running_var, float* inv_std, const float* x,
                                          float* xhat, void* out, hc_dtype out_dtype, void* workspace,
                                          size_t ws_bytes, hc_stream stream) {
    return guard([&] {
        check_c8(c);
        check_out_dtype(out_dtype);
        if (c > kT) throw std::invalid_argument("native batch norm: at most 256 channels");
        if (n <= 0) throw std::invalid_argument("batch_norm: empty input");
        if (ws_bytes < (size_t)c * sizeof(double)) throw std::invalid_argument("native batch norm: workspace too small");
        cudaStream_t s = as_stream(stream);
        double* mean = static_cast<double*>(workspace);
        const long long tiles = (n + 127) / 128;
        k_bn_fold_tiles<<<c, kT, 0, s>>>(reinterpret_cast<const float2*>(tile_stats), tiles, n, c, running_mean,
                                        running_var, momentum, eps, mean, inv_std);
        launched("batch-norm statistics from conv tiles");
        bn_relu_apply_out(x, n, c, mean, inv_std, xhat, out, out_dtype, s);
    });
}

hc_status hc_native_bn_stat(int32_t mode, const float* x, const void* d, hc_dtype dtype, int64_t n, int32_t c,
                            const double* mean, double* sums, void* workspace, size_t ws_bytes, hc_stream stream) {
    return guard([&] {
        check_c8(c);
        if (c > kT) throw std::invalid_argument("native batch norm: at most 256 channels");
        if (mode < 0 || mode > 2) throw std::invalid_argument("native batch norm: bad statistics mode");
        if (mode == 1 && !mean) throw std::invalid_argument("native batch norm: mode 1 needs the mean");
        if (mode == 2 && !d) throw std::invalid_argument("native batch norm: mode 2 needs the gradient");
        cudaStream_t s = as_stream(stream);
        if (n <= 0) {  // an empty shard contributes zeros to the global sums
            cuda_check(cudaMemsetAsync(sums, 0, sizeof(double) * 2 * c, s), "memset");
            return;
        }
        if (ws_bytes < hc_native_bn_workspace(n, c)) throw std::invalid_argument("native batch norm: workspace too small");
        const int blocks = bn_blocks(n);
        const int rpb = bn_rows_per_block(n);
        double* part = static_cast<double*>(workspace);
        if (mode == 0) k_col_partials<0, float><<<blocks, kT, 0, s>>>(x, nullptr, n, c, nullptr, part, rpb);
        else if (mode == 1) k_col_partials<1, float><<<blocks, kT, 0, s>>>(x, nullptr, n, c, mean, part, rpb);
        else if (dtype == HC_DTYPE_BF16)
            k_col_partials<2, bf16><<<blocks, kT, 0, s>>>(x, static_cast<const bf16*>(d), n, c, nullptr, part, rpb);
        else k_col_partials<2, float><<<blocks, kT, 0, s>>>(x, static_cast<const float*>(d), n, c, nullptr, part, rpb);
        k_col_fold<2><<<c, kT, 0, s>>>(part, blocks, n, c, sums, sums + c, nullptr, nullptr, 0, 0, nullptr, nullptr);
        launched("batch-norm partial sums", 2);
    });
}

hc_status hc_native_bn_finalize(const double* sum_x, const double* sum_sq, int64_t n_total, int32_t c, float momentum,
                                float eps, float* running_mean, float* running_var, double* mean, float* inv_std,
                                hc_stream stream) {
    return guard([&] {
        if (n_total <= 0) throw std::invalid_argument("batch_norm: empty input");
        if (c <= 0 || c > kT) throw std::invalid_argument("native batch norm: 1..256 channels");
        k_bn_finalize<<<1, kT, 0, as_stream(stream)>>>(sum_x, sum_sq, n_total, c, running_mean, running_var, momentum,
                                                      eps, mean, inv_std);
        launched("batch-norm finalize");
    });
}

hc_status hc_native_bn_relu_apply(const float* x, int64_t n, int32_t c, const double* mean, const float* inv_std,
                                  float* xhat, void* out_bf16, hc_stream stream) {
    return hc_native_bn_relu_apply_dt(x, n, c, mean, inv_std, xhat, out_bf16, HC_DTYPE_BF16, stream);
}

hc_status hc_native_bn_relu_apply_dt(const float* x, int64_t n, int32_t c, const double* mean, const float* inv_std,
                                     float* xhat, void* out, hc_dtype out_dtype, hc_stream stream) {
    return guard([&] {
        check_c8(c);
        check_out_dtype(out_dtype);
        if (n <= 0) return;
        bn_relu_apply_out(x, n, c, mean, inv_std, xhat, out, out_dtype, as_stream(stream));
    });
}

hc_status hc_native_bn_relu_backward_apply(const void* d_relu, hc_dtype dtype, const float* xhat, const float* inv_std,
                                           int64_t n, int32_t c, const double* s1, const double* s2, int64_t n_total,
                                           void* d_conv_bf16, hc_stream stream) {
    return hc_native_bn_relu_backward_apply_dt(d_relu, dtype, xhat, inv_std, n, c, s1, s2, n_total, d_conv_bf16,
                                               HC_DTYPE_BF16, stream);
}

hc_status hc_native_bn_relu_backward_apply_dt(const void* d_relu, hc_dtype dtype, const float* xhat,
                                              const float* inv_std, int64_t n, int32_t c, const double* s1,
                                              const double* s2, int64_t n_total, void* d_conv, hc_dtype out_dtype,
                                              hc_stream stream) {
    return guard([&] {
        check_c8(c);
        check_grad_out_dtype(out_dtype);
        if (n <= 0) return;
        if (n_total <= 0) throw std::invalid_argument("batch_norm: empty input");
        cudaStream_t s = as_stream(stream);
        if (dtype == HC_DTYPE_BF16)
            bn_bwd_apply_out(static_cast<const bf16*>(d_relu), xhat, n, c, s1, s2, inv_std, d_conv, out_dtype, n_total, s);
        else
            bn_bwd_apply_out(static_cast<const float*>(d_relu), xhat, n, c, s1, s2, inv_std, d_conv, out_dtype, n_total,
                             s);
        launched("batch-norm + relu backward");
    });
}

hc_status hc_native_dense_pool(const int32_t* cmap, int32_t b, const void* x_bf16, int32_t c, float* head,
                               int32_t* src, hc_stream stream) {
    return hc_native_dense_pool_dt(cmap, b, x_bf16, HC_DTYPE_BF16, c, head, src, stream);
}

hc_status hc_native_dense_pool_dt(const int32_t* cmap, int32_t b, const void* x, hc_dtype dtype, int32_t c,
                                  float* head, int32_t* src, hc_stream stream) {
    return guard([&] {
        check_out_dtype(dtype);
        if (b <= 0 || c <= 0) return;
        const int n = b * 8 * c;
        cudaStream_t s = as_stream(stream);
        if (dtype == HC_DTYPE_F32)
            k_dense_pool<float><<<grid_for(n, kT), kT, 0, s>>>(cmap, b, static_cast<const float*>(x), c, head, src);
        else
            k_dense_pool<bf16><<<grid_for(n, kT), kT, 0, s>>>(cmap, b, static_cast<const bf16*>(x), c, head, src);
        launched("dense pool");
    });
}

hc_status hc_native_dense_pool_backward(const float* d_head, const int32_t* src, int32_t b, int32_t c,
                                        int64_t n_fine, float* dx, hc_stream stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        if (n_fine > 0) cuda_check(cudaMemsetAsync(dx, 0, sizeof(float) * n_fine * c, s), "memset");
        if (b <= 0 || c <= 0) return;
        const int n = c * 8 * b;
        k_dense_pool_bwd<<<grid_for(n, kT), kT, 0, s>>>(d_head, src, b, c, dx);
        launched("dense pool backward");
    });
}

hc_status hc_native_dropout_apply(const float* u, const float* x, int64_t n, float keep, float* mask, float* out,
                                  hc_stream stream) {
    return guard([&] {
        if (n < 0 || !(keep > 0.0f && keep <= 1.0f)) throw std::invalid_argument("native dropout: bad arguments");
        if (n == 0) return;
        k_dropout_apply<<<grid_for(n, kT), kT, 0, as_stream(stream)>>>(u, x, n, keep, mask, out);
        launched("dropout");
    });
}

hc_status hc_native_softmax_xent(const float* scores, int32_t classes, int32_t b, const int64_t* labels,
                                 int64_t denom, double* loss, float* dscores, hc_stream stream) {
    return guard([&] {
        if (classes <= 0 || b <= 0 || denom <= 0 || !scores || !labels || !loss || !dscores)
            throw std::invalid_argument("native softmax cross-entropy: bad arguments");
        k_softmax_xent<<<1, 1024, 0, as_stream(stream)>>>(scores, classes, b, reinterpret_cast<const long long*>(labels),
                                                          1.0 / (double)denom, loss, dscores);
        launched("softmax cross-entropy");
    });
}

hc_status hc_native_sgd_update_multi(float* const* w, float* const* v, const float* const* g, const int64_t* n,
                                     int32_t count, float lr, float momentum, float weight_decay, hc_stream stream) {
    return guard([&] {
        if (count < 0 || count > kSgdMax) throw std::invalid_argument("native sgd: 0..32 tensors per call");
        SgdList L{};
        L.count = count;
        int blocks = 0;
        for (int k = 0; k < count; ++k) {
            if (n[k] < 0) throw std::invalid_argument("native sgd: negative tensor size");
            L.w[k] = w[k];
            L.v[k] = v[k];
            L.g[k] = g[k];
            L.n[k] = n[k];
            L.first[k] = blocks;
            blocks += (int)((n[k] + kT - 1) / kT);
        }
        L.first[count] = blocks;
        if (blocks == 0) return;
        k_sgd_multi<<<blocks, kT, 0, as_stream(stream)>>>(L, lr, momentum, weight_decay);
        launched("sgd update (multi-tensor)");
    });
}

hc_status hc_native_sgd_update(float* w, float* v, const float* g, int64_t n, float lr, float momentum,
                               float weight_decay, hc_stream stream) {
    return guard([&] {
        if (n <= 0) return;
        k_sgd<<<grid_for(n, kT), kT, 0, as_stream(stream)>>>(w, v, g, n, lr, momentum, weight_decay);
        launched("sgd update");
    });
}

}  // extern "C"
