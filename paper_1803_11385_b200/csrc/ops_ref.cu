// ops_ref.cu — the hot-path operators in the reference's layouts (channel-major
// feature matrices, (C*F^3) x N column matrices), bit-exact with
// src/cnn_ops.cpp. Work is enumerated by DATA COLUMN (one thread per output
// column for gathers, one per input column for the pull-based adjoints), so
// consecutive threads are z,y,x-raster neighbours: their probes and gathers hit
// the same L2 lines and their column-matrix stores coalesce.
//
// Arithmetic: order-defined reductions keep the reference order and use
// __fadd_rn/__fmul_rn so nvcc cannot contract them into FMAs.
#include <cuda_runtime.h>

#include <cmath>
#include <type_traits>
#include <string>

#include "dev_psh.cuh"
#include "hc_internal.h"
#include "hc_launch.cuh"
#include "tc_common.cuh"

namespace hcb {

namespace {

constexpr int kThreads = 256;

// tuning knobs read once from the environment (A/B experiments; defaults are the tuned values)
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// cnn_ops.cpp:20-33 check_pair (same messages, same order)
void check_pair(const hc_psh* in, const hc_psh* out, const hc_conv_spec& sp) {
    if (!in || !out) throw std::invalid_argument("null super-PSH handle");
    if (in->d.dim != out->d.dim) throw std::invalid_argument("structure dim mismatch");
    if (in->d.batch != out->d.batch) throw std::invalid_argument("batch size mismatch");
    if (sp.kernel < 1 || sp.stride < 1 || sp.pad < 0) throw std::invalid_argument("bad conv spec");
    if (sp.stride == 1) {
        if (sp.kernel % 2 == 0) throw std::invalid_argument("stride-1 fields need an odd kernel size");
        if (in->d.resolution != out->d.resolution) throw std::invalid_argument("stride-1 ops keep the level fixed");
    } else if (in->d.resolution != out->d.resolution * sp.stride) {
        throw std::invalid_argument("input resolution must be output resolution * stride");
    }
}

long long field_volume(const hc_conv_spec& sp, int dim) {
    long long v = 1;
    for (int a = 0; a < dim; ++a) v *= sp.kernel;
    return v;
}

// ============================================================== K0 field map
// Row-major K0 ([N_out][F^dim]): batched probes (see k_field_map_tiled), results staged in
// shared memory so the block's 128 * F^dim entries (one contiguous span of the map) leave
// in coalesced stores instead of 27 strided 4-byte stores per thread.
template <int F>
__global__ void __launch_bounds__(128, 4) k_field_map(DevPsh in, DevPsh out, int S, int pad, int* map) {
    constexpr int T = F * F * F;
    __shared__ int st[128 * T];
    const long long col0 = (long long)blockIdx.x * 128;
    const long long col = col0 + threadIdx.x;
    const int fd = in.dim == 3 ? T : F * F;
    if (col < out.N) {
        const int4 c = out.cols[col];
        const ModelParam mp = in.models[c.w - 1];
        int nb[T];
        probe_field_batched<F>(in, mp, origin_axis(c.x, F, S, pad), origin_axis(c.y, F, S, pad),
                               origin_axis(c.z, F, S, pad), nb);
#pragma unroll
        for (int t = 0; t < T; ++t)
            if (t < fd) st[threadIdx.x * fd + t] = nb[t];
    }
    __syncthreads();
    const long long cols = min(128LL, out.N - col0);
    int* dst = map + col0 * fd;
    for (int i = threadIdx.x; i < cols * fd; i += 128) dst[i] = st[i];
}

// Tap-major K0 ([F^3][N_out]): lanes of a warp write consecutive columns of each
// tap row, so every store instruction is fully coalesced (the native conv layout).
template <int F>
__global__ void k_field_map_t(DevPsh in, DevPsh out, int S, int pad, int* map) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int fd = in.dim == 3 ? F * F * F : F * F;
    int nb[F * F * F];
    probe_field_batched<F>(in, mp, origin_axis(c.x, F, S, pad), origin_axis(c.y, F, S, pad),
                           origin_axis(c.z, F, S, pad), nb);
    const long long N = out.N;
#pragma unroll
    for (int t = 0; t < F * F * F; ++t)
        if (t < fd) map[t * N + col] = nb[t];
}

// Tile-major K0 ([ceil(N/128)][F^3][128]): one 128-column tile's whole map is a
// contiguous block (fetched by one bulk copy in the native conv); padded columns
// beyond N are -1.
template <int F>
#ifndef HCB_K0_MINB
#define HCB_K0_MINB 2
#endif
__global__ void __launch_bounds__(256, HCB_K0_MINB) k_field_map_tiled(DevPsh in, DevPsh out, int S, int pad, int* map) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long padded = (out.N + 127) / 128 * 128;
    if (col >= padded) return;
    const int fd = in.dim == 3 ? F * F * F : F * F;
    int nb[F * F * F];
    if (col < out.N) {
        const int4 c = out.cols[col];
        const ModelParam mp = in.models[c.w - 1];
        probe_field_batched<F>(in, mp, origin_axis(c.x, F, S, pad), origin_axis(c.y, F, S, pad),
                       origin_axis(c.z, F, S, pad), nb);
    } else {
#pragma unroll
        for (int t = 0; t < F * F * F; ++t) nb[t] = -1;
    }
    int* dst = map + (col >> 7) * fd * 128 + (col & 127);
#pragma unroll
    for (int t = 0; t < F * F * F; ++t)
        if (t < fd) dst[t * 128] = nb[t];
}

__global__ void k_field_map_any_tiled(DevPsh in, DevPsh out, int F, int S, int pad, int fd, int* map) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long padded = (out.N + 127) / 128 * 128;
    if (col >= padded) return;
    int* dst = map + (col >> 7) * fd * 128 + (col & 127);
    if (col >= out.N) {
        for (int t = 0; t < fd; ++t) dst[t * 128] = -1;
        return;
    }
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int bx = origin_axis(c.x, F, S, pad), by = origin_axis(c.y, F, S, pad), bz = origin_axis(c.z, F, S, pad);
    for (int t = 0; t < fd; ++t) dst[t * 128] = probe_tap(in, mp, bx, by, bz, F, t);
}

__global__ void k_field_map_any_t(DevPsh in, DevPsh out, int F, int S, int pad, int fd, int* map) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int bx = origin_axis(c.x, F, S, pad), by = origin_axis(c.y, F, S, pad), bz = origin_axis(c.z, F, S, pad);
    for (int t = 0; t < fd; ++t) map[t * out.N + col] = probe_tap(in, mp, bx, by, bz, F, t);
}

__global__ void k_field_map_any(DevPsh in, DevPsh out, int F, int S, int pad, int fd, int* map) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int bx = origin_axis(c.x, F, S, pad), by = origin_axis(c.y, F, S, pad), bz = origin_axis(c.z, F, S, pad);
    for (int t = 0; t < fd; ++t) map[col * fd + t] = probe_tap(in, mp, bx, by, bz, F, t);
}

// ============================================================== hash2col
// cnn_ops.cpp:123-158: cols[(c*fd + row), col] = data[c, hit] or 0.
// Memory-bound: occupancy matters more than per-thread ILP, so registers are capped
// (MINB resident 256-thread blocks per SM).
template <int F, int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_hash2col(DevPsh in, DevPsh out, int S, int pad, const float* __restrict__ data, int C,
               float* __restrict__ cols) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int fd = in.dim == 3 ? F * F * F : F * F;
    int nb[F * F * F];
    probe_field<F>(in, mp, origin_axis(c.x, F, S, pad), origin_axis(c.y, F, S, pad),
                   origin_axis(c.z, F, S, pad), nb);
    const long long Nin = in.N, Nout = out.N;
    for (int ch = 0; ch < C; ++ch) {
        const float* src = data + ch * Nin;
        float* dst = cols + (long long)ch * fd * Nout + col;
#pragma unroll
        for (int t = 0; t < F * F * F; ++t) {
            if (t < fd) {
                const float v = nb[t] >= 0 ? __ldg(src + nb[t]) : 0.0f;
                __stcs(dst + (long long)t * Nout, v);
            }
        }
    }
}

template <typename T>
__global__ void k_hash2col_any(DevPsh in, DevPsh out, int F, int S, int pad, int fd, const T* __restrict__ data,
                               int C, T* __restrict__ cols) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int bx = origin_axis(c.x, F, S, pad), by = origin_axis(c.y, F, S, pad), bz = origin_axis(c.z, F, S, pad);
    const long long Nin = in.N, Nout = out.N;
    for (int t = 0; t < fd; ++t) {
        const int g = probe_tap(in, mp, bx, by, bz, F, t);
        for (int ch = 0; ch < C; ++ch)
            cols[((long long)ch * fd + t) * Nout + col] = g >= 0 ? __ldg(data + ch * Nin + g) : T(0);
    }
}

// ============================================================== covering probes
// Covering outputs of input voxel p_i in ascending (z,y,x) order with the field
// row of p_i inside each (cnn_ops.cpp:70-92, 184-196). KA = max outputs per axis.
template <int KA>
__device__ __forceinline__ int cover_hits(const DevPsh& out, const ModelParam& mp, int px, int py, int pz, int F,
                                          int S, int pad, int* hcol, int* hrow) {
    const int dim = out.dim;
    int lox, hix, loy, hiy, loz = 0, hiz = 0;
    cover_axis(px, F, S, pad, out.resolution, lox, hix);
    cover_axis(py, F, S, pad, out.resolution, loy, hiy);
    if (dim == 3) cover_axis(pz, F, S, pad, out.resolution, loz, hiz);
    int n = 0;
    for (int z = loz; z <= hiz; ++z)
        for (int y = loy; y <= hiy; ++y)
            for (int x = lox; x <= hix; ++x) {
                const int g = probe(out, mp, x, y, z);
                if (g < 0) continue;
                const int rx = px - origin_axis(x, F, S, pad), ry = py - origin_axis(y, F, S, pad);
                const int rz = dim == 3 ? pz - origin_axis(z, F, S, pad) : 0;
                hcol[n] = g;
                hrow[n] = (rz * F + ry) * F + rx;
                ++n;
            }
    return n;
}

// Stride-1 covering set via the residue-sharing field probe: outputs p_i + d,
// row = fd - 1 - tap (the field of p_o = p_i + d holds p_i at offset -d).
template <int F>
__device__ __forceinline__ int cover_hits_s1(const DevPsh& out, const ModelParam& mp, int px, int py, int pz,
                                             int* hcol, int* hrow) {
    const int h = (F - 1) / 2;
    const int fd = out.dim == 3 ? F * F * F : F * F;
    int nb[F * F * F];
    probe_field<F>(out, mp, px - h, py - h, pz - h, nb);
    int n = 0;
#pragma unroll
    for (int t = 0; t < F * F * F; ++t) {
        if (t < fd && nb[t] >= 0) {
            hcol[n] = nb[t];
            hrow[n] = fd - 1 - t;
            ++n;
        }
    }
    return n;
}

// ============================================================== col2hash
// cnn_ops.cpp:160-204 (Alg. 2): pull per input column; per channel the sum runs
// over covering outputs in ascending order (deterministic, bit-exact).
// Stride 1: the covering outputs are the field taps around p_i in the OUTPUT
// structure, visited in ascending tap order (= ascending p_o) WITHOUT compaction, so
// at every step all lanes of a warp read the same column-matrix row (fd-1-t) at
// neighbouring columns: coalesced gathers instead of per-lane scattered rows.
// Taps-outer variant: the 27 probed columns are parked in shared memory ([tap][thread],
// conflict-free), then for each tap every thread issues CB independent channel loads
// into CB accumulators. Per channel the taps are still added in ascending order, so the
// result is bit-identical to cnn_ops.cpp:184-196.
template <int F, int CB>
__global__ void __launch_bounds__(256, 4)
    k_col2hash_s1_tb(DevPsh in, DevPsh out, const float* __restrict__ g, int C, float* __restrict__ res) {
    constexpr int T3 = F * F * F;
    __shared__ int nbs[T3][256];
    const long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const bool live = gi < in.N;
    const int fd = out.dim == 3 ? T3 : F * F;
    if (live) {
        const int4 c = in.cols[gi];
        const ModelParam mp = out.models[c.w - 1];
        constexpr int h = (F - 1) / 2;
        int nb[T3];
        probe_field<F>(out, mp, c.x - h, c.y - h, c.z - h, nb);
#pragma unroll
        for (int t = 0; t < T3; ++t) nbs[t][threadIdx.x] = t < fd ? nb[t] : -1;
    }
    if (!live) return;  // no block-wide barrier below: each thread reads only its own column
    const int Nout = (int)out.N;  // fd * N_out < 2^31 (checked at launch): 32-bit row offsets
    const long long Nin = in.N;
    const long long plane = (long long)fd * Nout;
    for (int cb = 0; cb < C; cb += CB) {
        // one 64-bit base per channel (clamped past C: loads stay in bounds, results unused);
        // per tap a 32-bit offset shared by all CB loads -> ~3 instructions per gathered float
        const float* bp[CB];
#pragma unroll
        for (int u = 0; u < CB; ++u) bp[u] = g + (long long)min(cb + u, C - 1) * plane;
        float acc[CB];
#pragma unroll
        for (int u = 0; u < CB; ++u) acc[u] = 0.0f;
        for (int t = 0; t < fd; ++t) {
            const int col = nbs[t][threadIdx.x];
            if (col < 0) continue;
            const unsigned off = (unsigned)(fd - 1 - t) * (unsigned)Nout + (unsigned)col;
#pragma unroll
            for (int u = 0; u < CB; ++u) acc[u] = __fadd_rn(acc[u], __ldg(bp[u] + off));
        }
#pragma unroll
        for (int u = 0; u < CB; ++u)
            if (cb + u < C) res[(long long)(cb + u) * Nin + gi] = acc[u];
    }
}

// CU channels per pass: CU independent accumulator chains (each still adds its taps in
// ascending order -> bit-exact); registers capped for MINB resident blocks per SM.
template <int F, int CU, int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_col2hash_s1(DevPsh in, DevPsh out, const float* __restrict__ g, int C, float* __restrict__ res) {
    const long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (gi >= in.N) return;
    const int4 c = in.cols[gi];
    const ModelParam mp = out.models[c.w - 1];
    constexpr int h = (F - 1) / 2;
    const int fd = out.dim == 3 ? F * F * F : F * F;
    int nb[F * F * F];
    probe_field<F>(out, mp, c.x - h, c.y - h, c.z - h, nb);
    const long long Nout = out.N, Nin = in.N;
    const long long plane = (long long)fd * Nout;  // one channel's block of the column matrix
    int ch = 0;
    for (; ch + CU <= C; ch += CU) {
        float a[CU];
#pragma unroll
        for (int u = 0; u < CU; ++u) a[u] = 0.0f;
        const float* b0 = g + (long long)ch * plane;
#pragma unroll
        for (int t = 0; t < F * F * F; ++t) {
            if (t < fd && nb[t] >= 0) {
                const float* p = b0 + (long long)(fd - 1 - t) * Nout + nb[t];
#pragma unroll
                for (int u = 0; u < CU; ++u) a[u] = __fadd_rn(a[u], __ldg(p + u * plane));
            }
        }
#pragma unroll
        for (int u = 0; u < CU; ++u) res[(ch + u) * Nin + gi] = a[u];
    }
    for (; ch < C; ++ch) {
        float acc = 0.0f;
        const float* base = g + (long long)ch * plane;
#pragma unroll
        for (int t = 0; t < F * F * F; ++t)
            if (t < fd && nb[t] >= 0) acc = __fadd_rn(acc, __ldg(base + (long long)(fd - 1 - t) * Nout + nb[t]));
        res[ch * Nin + gi] = acc;
    }
}

template <int KMAX, bool STRIDE1, int F>
__global__ void k_col2hash(DevPsh in, DevPsh out, int Fr, int S, int pad, int fd, const float* __restrict__ g,
                           int C, float* __restrict__ res) {
    const long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (gi >= in.N) return;
    const int4 c = in.cols[gi];
    const ModelParam mp = out.models[c.w - 1];
    int hcol[KMAX], hrow[KMAX];
    int n;
    if constexpr (STRIDE1) n = cover_hits_s1<F>(out, mp, c.x, c.y, c.z, hcol, hrow);
    else n = cover_hits<1>(out, mp, c.x, c.y, c.z, Fr, S, pad, hcol, hrow);
    const long long Nout = out.N, Nin = in.N;
    for (int ch = 0; ch < C; ++ch) {
        float acc = 0.0f;
        const float* base = g + (long long)ch * fd * Nout;
#pragma unroll
        for (int h = 0; h < KMAX; ++h)
            if (h < n) acc = __fadd_rn(acc, __ldg(base + (long long)hrow[h] * Nout + hcol[h]));
        res[ch * Nin + gi] = acc;
    }
}

// any F / stride: recompute covering probes per channel (no register arrays)
template <typename T>
__global__ void k_col2hash_any(DevPsh in, DevPsh out, int F, int S, int pad, int fd, const T* __restrict__ g,
                               int C, T* __restrict__ res) {
    const long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (gi >= in.N) return;
    const int4 c = in.cols[gi];
    const ModelParam mp = out.models[c.w - 1];
    const int dim = out.dim;
    int lox, hix, loy, hiy, loz = 0, hiz = 0;
    cover_axis(c.x, F, S, pad, out.resolution, lox, hix);
    cover_axis(c.y, F, S, pad, out.resolution, loy, hiy);
    if (dim == 3) cover_axis(c.z, F, S, pad, out.resolution, loz, hiz);
    const long long Nout = out.N, Nin = in.N;
    for (int ch = 0; ch < C; ++ch) {
        T acc = T(0);
        for (int z = loz; z <= hiz; ++z)
            for (int y = loy; y <= hiy; ++y)
                for (int x = lox; x <= hix; ++x) {
                    const int col = probe(out, mp, x, y, z);
                    if (col < 0) continue;
                    const int rx = c.x - origin_axis(x, F, S, pad), ry = c.y - origin_axis(y, F, S, pad);
                    const int rz = dim == 3 ? c.z - origin_axis(z, F, S, pad) : 0;
                    const int row = (rz * F + ry) * F + rx;
                    acc = add_rn(acc, g[((long long)ch * fd + row) * Nout + col]);
                }
        res[ch * Nin + gi] = acc;
    }
}

// ============================================================== pooling
// cnn_ops.cpp:234-284 max_pool: first present tap seeds, strict '>' (ties keep
// the smallest field row); empty field -> 0 / -1.
// Channels are processed CB at a time with all (tap, channel) loads issued before any
// compare, so each thread keeps CB*F^3 independent gathers in flight (a per-channel loop
// is one dependent latency chain per channel). Per channel the taps are still visited in
// row order with the same seed/tie rule -> bit-identical results.
#ifndef HCB_POOL_MINB
#define HCB_POOL_MINB 1
#endif
template <int F, int CB>
__global__ void __launch_bounds__(256, HCB_POOL_MINB) k_max_pool(DevPsh in, DevPsh out, int S, int pad,
                                                  const float* __restrict__ data, int C, float* __restrict__ res,
                                                  int* __restrict__ sw) {
    constexpr int T = F * F * F;
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int fd = in.dim == 3 ? T : F * F;
    int nb[T];
    probe_field<F>(in, mp, origin_axis(c.x, F, S, pad), origin_axis(c.y, F, S, pad),
                   origin_axis(c.z, F, S, pad), nb);
#pragma unroll
    for (int t = 0; t < T; ++t)
        if (t >= fd) nb[t] = -1;
    const long long Nin = in.N, Nout = out.N;
    int kt[T];  // gather offsets (0 for absent taps: the load is harmless, the value unused)
#pragma unroll
    for (int t = 0; t < T; ++t) kt[t] = max(nb[t], 0);
    const float* src = data;
    float* rp = res + col;
    int* sp = sw + col;
    for (int ch0 = 0; ch0 < C; ch0 += CB) {
        float v[CB][T];
#pragma unroll
        for (int u = 0; u < CB; ++u) {
            const float* su = src + (ch0 + u < C ? u * Nin : 0);
#pragma unroll
            for (int t = 0; t < T; ++t) v[u][t] = __ldg(su + kt[t]);
        }
#pragma unroll
        for (int u = 0; u < CB; ++u) {
            if (ch0 + u >= C) break;
            float best = 0.0f;
            int arg = -1;
#pragma unroll
            for (int t = 0; t < T; ++t) {
                if (nb[t] >= 0 && (arg < 0 || v[u][t] > best)) {
                    best = v[u][t];
                    arg = t;
                }
            }
            rp[u * Nout] = arg < 0 ? 0.0f : best;
            sp[u * Nout] = arg;
        }
        src += CB * Nin;
        rp += CB * Nout;
        sp += CB * Nout;
    }
}

template <typename T>
__global__ void k_max_pool_any(DevPsh in, DevPsh out, int F, int S, int pad, int fd, const T* __restrict__ data,
                               int C, T* __restrict__ res, int* __restrict__ sw) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int bx = origin_axis(c.x, F, S, pad), by = origin_axis(c.y, F, S, pad), bz = origin_axis(c.z, F, S, pad);
    const long long Nin = in.N, Nout = out.N;
    for (int ch = 0; ch < C; ++ch) {
        T best = T(0);
        int arg = -1;
        for (int t = 0; t < fd; ++t) {
            const int g = probe_tap(in, mp, bx, by, bz, F, t);
            if (g < 0) continue;
            const T v = data[ch * Nin + g];
            if (arg < 0 || v > best) {
                best = v;
                arg = t;
            }
        }
        res[ch * Nout + col] = arg < 0 ? T(0) : best;
        sw[ch * Nout + col] = arg;
    }
}

// cnn_ops.cpp:286-322 avg_pool: (sum over present taps, row order) * inv_fd; CB channels
// per pass with independent loads (see k_max_pool).
template <int F, int CB>
__global__ void __launch_bounds__(256, HCB_POOL_MINB) k_avg_pool(DevPsh in, DevPsh out, int S, int pad,
                                                  const float* __restrict__ data, int C, float inv,
                                                  float* __restrict__ res) {
    constexpr int T = F * F * F;
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int fd = in.dim == 3 ? T : F * F;
    int nb[T];
    probe_field<F>(in, mp, origin_axis(c.x, F, S, pad), origin_axis(c.y, F, S, pad),
                   origin_axis(c.z, F, S, pad), nb);
#pragma unroll
    for (int t = 0; t < T; ++t)
        if (t >= fd) nb[t] = -1;
    const long long Nin = in.N, Nout = out.N;
    int kt[T];
#pragma unroll
    for (int t = 0; t < T; ++t) kt[t] = max(nb[t], 0);
    const float* src = data;
    float* rp = res + col;
    for (int ch0 = 0; ch0 < C; ch0 += CB) {
        float v[CB][T];
#pragma unroll
        for (int u = 0; u < CB; ++u) {
            const float* su = src + (ch0 + u < C ? u * Nin : 0);
#pragma unroll
            for (int t = 0; t < T; ++t) v[u][t] = __ldg(su + kt[t]);
        }
#pragma unroll
        for (int u = 0; u < CB; ++u) {
            if (ch0 + u >= C) break;
            float acc = 0.0f;
#pragma unroll
            for (int t = 0; t < T; ++t)
                if (nb[t] >= 0) acc = __fadd_rn(acc, v[u][t]);
            rp[u * Nout] = __fmul_rn(acc, inv);
        }
        src += CB * Nin;
        rp += CB * Nout;
    }
}

// ------------------------------------------------- staged 2^3 pooling (F = 2, dim 3)
// The children of 256 consecutive coarse voxels lie in a few contiguous spans of fine
// columns, one per (model, coarse z, child dz) — columns are z,y,x-sorted — covering
// ~2048 columns plus partial rows at the span ends. A block finds those spans once
// (block scan of (model, z) changes, warp min/max reductions), then streams PL channel
// planes of every span per stage into shared memory with 1-D bulk copies (one mbarrier
// per stage, NS stages in flight) and reduces the children from shared memory: DRAM
// sees contiguous multi-KB reads instead of scattered 4-byte gathers, and a warp waits
// once per PL planes. Per channel the taps are visited in row order with
// the first-hit seed / strict '>' rule (max) or the row-order __fadd_rn sum (avg), so the
// results are bit-identical to k_max_pool / k_avg_pool. A block whose spans do not fit
// (more than NKEY/2 (model, z) pairs, > CAP columns, or a copy that would run past the
// last plane) runs the direct per-thread gathers instead. A ninth warp only issues the
// copies: each consumer warp releases a stage on its own "empty" mbarrier arrival, so warps
// never wait for each other (a block barrier per stage: 0.170 ms).
constexpr int kPoolCap = 2304;  // staged columns per plane (2048 children + span slack)
constexpr int kPoolKeys = 16;   // (model, z) pair x child dz spans per block

template <bool AVG>
__device__ __forceinline__ void pool_reduce(const float (&v)[8], const int (&nb)[8], float inv, float& out, int& arg) {
    if constexpr (AVG) {
        float acc = 0.0f;
#pragma unroll
        for (int t = 0; t < 8; ++t)
            if (nb[t] >= 0) acc = __fadd_rn(acc, v[t]);
        out = __fmul_rn(acc, inv);
        arg = 0;
    } else {
        float best = 0.0f;
        arg = -1;
#pragma unroll
        for (int t = 0; t < 8; ++t)
            if (nb[t] >= 0 && (arg < 0 || v[t] > best)) {
                best = v[t];
                arg = t;
            }
        out = arg < 0 ? 0.0f : best;
    }
}

template <int PL, int NS, bool AVG, int MINB = 1, int BO = 256>
__global__ void __launch_bounds__(BO + 32, MINB) k_pool_staged(DevPsh in, DevPsh out, int S, int pad,
                                                        const float* __restrict__ data, int C, float inv,
                                                        float* __restrict__ res, int* __restrict__ sw) {
    constexpr int NKEY = kPoolKeys, CAP = kPoolCap * BO / 256, NW = BO / 32;  // NW consumer warps
    extern __shared__ __align__(128) float stage[];  // [NS][PL][CAP]
    __shared__ int rmin[NKEY], rmax[NKEY], roff[NKEY], wtot[NW + 1];
    __shared__ int s_over;
    __shared__ __align__(8) unsigned long long full[NS], empty[NS];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long col = blockIdx.x * (long long)BO + tid;
    const bool live = tid < BO && col < out.N;
    const long long Nin = in.N, Nout = out.N;
    if (tid < NKEY) {
        rmin[tid] = INT_MAX;
        rmax[tid] = -1;
    }
    if (tid < NS * PL) *reinterpret_cast<float4*>(stage + tid * CAP + CAP - 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid == 0) {
        s_over = 0;
        for (int s = 0; s < NS; ++s) {
            tc::mbar_init(tc::smem_u32(&full[s]), 1);
            tc::mbar_init(tc::smem_u32(&empty[s]), NW);
        }
        tc::mbar_init_fence();
    }
    int nb[8];
    int4 c = make_int4(0, 0, 0, 0);
    if (live) {
        c = out.cols[col];
        const ModelParam mp = in.models[c.w - 1];
        probe_field_batched<2>(in, mp, origin_axis(c.x, 2, S, pad), origin_axis(c.y, 2, S, pad),
                               origin_axis(c.z, 2, S, pad), nb);
    } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) nb[t] = -1;
    }
    // span key: number of (model, z) changes before this voxel in the block
    int pw = __shfl_up_sync(0xffffffffu, c.w, 1), pz = __shfl_up_sync(0xffffffffu, c.z, 1);
    if (lane == 0 && tid > 0 && live) {
        const int4 p = out.cols[col - 1];
        pw = p.w;
        pz = p.z;
    }
    const bool flag = live && tid > 0 && (pw != c.w || pz != c.z);
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    if (lane == 31) wtot[wid] = __popc(bal);
    int lmin0 = INT_MAX, lmax0 = -1, lmin1 = INT_MAX, lmax1 = -1;
#pragma unroll
    for (int t = 0; t < 4; ++t)
        if (nb[t] >= 0) {
            lmin0 = min(lmin0, nb[t]);
            lmax0 = max(lmax0, nb[t]);
        }
#pragma unroll
    for (int t = 4; t < 8; ++t)
        if (nb[t] >= 0) {
            lmin1 = min(lmin1, nb[t]);
            lmax1 = max(lmax1, nb[t]);
        }
    __syncthreads();
    int k = __popc(bal & (0xffffffffu >> (31 - lane)));
    for (int w = 0; w < wid; ++w) k += wtot[w];
    {
        const int kmin = __reduce_min_sync(0xffffffffu, k), kmax = __reduce_max_sync(0xffffffffu, k);
        if (2 * kmax + 1 >= NKEY) {
            if (lane == 0) s_over = 1;
        } else {
            for (int kk = kmin; kk <= kmax; ++kk) {
                const bool me = k == kk;
                const int a0 = __reduce_min_sync(0xffffffffu, me ? lmin0 : INT_MAX);
                const int b0 = __reduce_max_sync(0xffffffffu, me ? lmax0 : -1);
                const int a1 = __reduce_min_sync(0xffffffffu, me ? lmin1 : INT_MAX);
                const int b1 = __reduce_max_sync(0xffffffffu, me ? lmax1 : -1);
                if (lane == 0) {
                    atomicMin(&rmin[2 * kk], a0);
                    atomicMax(&rmax[2 * kk], b0);
                    atomicMin(&rmin[2 * kk + 1], a1);
                    atomicMax(&rmax[2 * kk + 1], b1);
                }
            }
        }
    }
    __syncthreads();
    if (tid == 0 && !s_over) {
        int off = 0;
        const long long total = (long long)C * Nin;
        for (int j = 0; j < NKEY; ++j) {
            roff[j] = off;
            if (rmax[j] < 0) continue;
            const int len = rmax[j] - rmin[j] + 1;
            off += (len + 6) & ~3;  // room for a 0..3 column alignment shift, 16-byte granules
            const long long g = (long long)(C - 1) * Nin + rmin[j], a = g & ~3LL;
            if (a + ((g + len - a + 3) & ~3LL) > total) s_over = 1;  // last plane's copy past the end
        }
        if (off > CAP - 4) s_over = 1;  // the last 4 columns of every plane slot stay zero
    }
    __syncthreads();
    if (s_over) {  // direct gathers (same arithmetic)
        if (!live) return;
        int kt[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) kt[t] = max(nb[t], 0);
        for (int ch = 0; ch < C; ++ch) {
            const float* src = data + ch * Nin;
            float v[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) v[t] = __ldg(src + kt[t]);
            float o;
            int arg;
            pool_reduce<AVG>(v, nb, inv, o, arg);
            res[ch * Nout + col] = o;
            if constexpr (!AVG) sw[ch * Nout + col] = arg;
        }
        return;
    }
    // per-tap shared offsets: roff + (child - span start) + the plane's alignment shift.
    // Absent taps read a present one (max: the first present tap, whose value seeds the
    // running max, so a copy never passes the strict '>') or the zero columns at the end of
    // the slot (avg: adding +0.0 to a row-order sum that starts at +0.0 is exact), so the
    // reduction needs no per-tap presence test.
    int tf = -1;
#pragma unroll
    for (int t = 7; t >= 0; --t)
        if (nb[t] >= 0) tf = t;
    int pb[8], rm3[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int j = 2 * k + (t >> 2);
        pb[t] = nb[t] >= 0 ? roff[j] + nb[t] - rmin[j] : CAP - 4;
        rm3[t] = nb[t] >= 0 ? rmin[j] & 3 : 0;
    }
    if constexpr (!AVG) {
        if (tf >= 0) {
            int pf = 0, rf = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (t == tf) {
                    pf = pb[t];
                    rf = rm3[t];
                }
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (nb[t] < 0) {
                    pb[t] = pf;
                    rm3[t] = rf;
                }
        }
    }
    const int nin3 = (int)(Nin & 3);
    const int nsteps = (C + PL - 1) / PL;
    const uint32_t stage0 = tc::smem_u32(stage);
    auto issue = [&](int j) {  // producer warp: the PL planes of step j into slot j % NS
        const int slot = j % NS;
        const uint32_t bar = tc::smem_u32(&full[slot]);
        uint32_t bytes = 0;
        for (int i = lane; i < PL * NKEY; i += 32) {
            const int p = i / NKEY, key = i % NKEY, ch = j * PL + p;
            if (ch >= C || rmax[key] < 0) continue;
            const long long g = (long long)ch * Nin + rmin[key], a = g & ~3LL;
            bytes += (uint32_t)(((g + rmax[key] - rmin[key] + 1 - a + 3) & ~3LL) * 4);
        }
        bytes = __reduce_add_sync(0xffffffffu, bytes);
        if (lane == 0) tc::mbar_arrive_expect_tx(bar, bytes);
        __syncwarp();
        for (int i = lane; i < PL * NKEY; i += 32) {
            const int p = i / NKEY, key = i % NKEY, ch = j * PL + p;
            if (ch >= C || rmax[key] < 0) continue;
            const long long g = (long long)ch * Nin + rmin[key], a = g & ~3LL;
            const uint32_t n = (uint32_t)(((g + rmax[key] - rmin[key] + 1 - a + 3) & ~3LL) * 4);
            tc::bulk_g2s(stage0 + (uint32_t)(((slot * PL + p) * CAP + roff[key]) * 4), data + a, n, bar);
        }
    };
    if (wid == NW) {  // producer warp
        for (int j = 0; j < nsteps; ++j) {
            if (j >= NS) tc::mbar_wait(tc::smem_u32(&empty[j % NS]), ((j / NS) - 1) & 1);
            issue(j);
        }
        return;
    }
    // consumers; AL: every plane starts 16-byte aligned (N % 4 == 0), so the alignment
    // shift is the span's own and folds into the tap offsets
    auto consume = [&](auto aligned) {
        constexpr bool AL = decltype(aligned)::value;
        int pa[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) pa[t] = pb[t] + rm3[t];
        float* rp = res + col;
        int* sp = AVG ? nullptr : sw + col;  // avg pooling has no switches (sw == nullptr)
        for (int j = 0; j < nsteps; ++j) {
            const int slot = j % NS;
            tc::mbar_wait(tc::smem_u32(&full[slot]), (j / NS) & 1);
            if (live) {
#pragma unroll
                for (int p = 0; p < PL; ++p) {
                    const int ch = j * PL + p;
                    if (ch >= C) break;
                    const float* pl = stage + (slot * PL + p) * CAP;
                    const int cs = ch * nin3;
                    float v[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) v[t] = pl[AL ? pa[t] : pb[t] + ((cs + rm3[t]) & 3)];
                    float o;
                    int arg = 0;
                    if constexpr (AVG) {
                        float acc = 0.0f;
#pragma unroll
                        for (int t = 0; t < 8; ++t) acc = __fadd_rn(acc, v[t]);
                        o = __fmul_rn(acc, inv);
                    } else {
                        float best = v[0];
                        arg = tf;
#pragma unroll
                        for (int t = 1; t < 8; ++t)
                            if (v[t] > best) {
                                best = v[t];
                                arg = t;
                            }
                        o = tf < 0 ? 0.0f : best;
                    }
                    *rp = o;
                    rp += Nout;
                    if constexpr (!AVG) {
                        *sp = arg;
                        sp += Nout;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&empty[slot]));
        }
    };
    if (nin3 == 0) consume(std::true_type{});
    else consume(std::false_type{});
}

template <typename T>
__global__ void k_avg_pool_any(DevPsh in, DevPsh out, int F, int S, int pad, int fd, const T* __restrict__ data,
                               int C, T inv, T* __restrict__ res) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= out.N) return;
    const int4 c = out.cols[col];
    const ModelParam mp = in.models[c.w - 1];
    const int bx = origin_axis(c.x, F, S, pad), by = origin_axis(c.y, F, S, pad), bz = origin_axis(c.z, F, S, pad);
    const long long Nin = in.N, Nout = out.N;
    for (int ch = 0; ch < C; ++ch) {
        T acc = T(0);
        for (int t = 0; t < fd; ++t) {
            const int g = probe_tap(in, mp, bx, by, bz, F, t);
            if (g >= 0) acc = add_rn(acc, data[ch * Nin + g]);
        }
        res[ch * Nout + col] = mul_rn(acc, inv);
    }
}

// ============================================================== unpooling
// cnn_ops.cpp:336-372 max_unpool: out[c,g] = 0 (+) coarse[c,col] for covering
// outputs whose switch equals g's field row, ascending output order.
// CB channels per pass: the switch and value loads of all CB channels are issued before
// any compare (the per-channel form serialised a switch load -> value load chain per channel).
// Range scan of the switches (cnn_ops.cpp:326-332): 4 x 16-byte loads per thread per pass (one
// 4-byte load per thread kept too few bytes in flight: 72 us for 110 MB, 1.5 TB/s); thread tid
// of nth scanning threads; an out-of-range switch raises the mapped host flag.
__device__ __forceinline__ void check_switches_body(const int* sw, long long n, int fd, int* bad, long long tid,
                                                    long long nth) {
    const unsigned lim = (unsigned)fd + 1u;  // s in [-1, fd)  <=>  (unsigned)(s + 1) < fd + 1
    bool ok = true;
    const long long head = (long long)(((16 - (reinterpret_cast<uintptr_t>(sw) & 15)) & 15) / 4);
    const long long h = head < n ? head : n;
    if (tid < h) ok = (unsigned)sw[tid] + 1u < lim;
    const int4* v = reinterpret_cast<const int4*>(sw + h);
    const long long nv = (n - h) / 4;
    for (long long i = tid; i < nv; i += 4 * nth) {
        int4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = i + u * nth < nv ? __ldcs(v + i + u * nth) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            ok &= ((unsigned)q[u].x + 1u < lim) & ((unsigned)q[u].y + 1u < lim) & ((unsigned)q[u].z + 1u < lim) &
                  ((unsigned)q[u].w + 1u < lim);
    }
    const long long t0 = h + nv * 4;
    if (t0 + tid < n) ok &= (unsigned)sw[t0 + tid] + 1u < lim;
    if (!ok) *reinterpret_cast<volatile int*>(bad) = 1;  // mapped host word
}

template <int KMAX, bool AVG, int CB>
__device__ __forceinline__ void unpool_body(const DevPsh& fine, const DevPsh& coarse, int F, int S, int pad,
                                            const float* __restrict__ cd, const int* __restrict__ sw, int C,
                                            float inv, float* __restrict__ res) {
    const long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (gi >= fine.N) return;
    const int4 c = fine.cols[gi];
    const ModelParam mp = coarse.models[c.w - 1];
    int hcol[KMAX], hrow[KMAX];
    const int n = cover_hits<1>(coarse, mp, c.x, c.y, c.z, F, S, pad, hcol, hrow);
    const long long Nc = coarse.N, Nf = fine.N;
    const float* cp = cd;
    const int* wp = sw;
    float* rp = res + gi;
    for (int ch0 = 0; ch0 < C; ch0 += CB) {
        float acc[CB];
#pragma unroll
        for (int u = 0; u < CB; ++u) acc[u] = 0.0f;
#pragma unroll
        for (int h = 0; h < KMAX; ++h) {
            if (h < n) {
                float v[CB];
                int w[CB];
#pragma unroll
                for (int u = 0; u < CB; ++u) {
                    const long long k = (ch0 + u < C ? u * Nc : 0) + hcol[h];
                    v[u] = __ldg(cp + k);
                    if constexpr (!AVG) w[u] = __ldg(wp + k);
                }
#pragma unroll
                for (int u = 0; u < CB; ++u) {
                    if constexpr (AVG) acc[u] = __fadd_rn(acc[u], __fmul_rn(v[u], inv));
                    else if (w[u] == hrow[h]) acc[u] = __fadd_rn(acc[u], v[u]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < CB; ++u)
            if (ch0 + u < C) rp[u * Nf] = acc[u];
        cp += CB * Nc;
        wp += CB * Nc;
        rp += CB * Nf;
    }
}

template <int KMAX, bool AVG, int CB>
__global__ void __launch_bounds__(256, HCB_POOL_MINB) k_unpool(DevPsh fine, DevPsh coarse, int F, int S, int pad,
                                                const float* __restrict__ cd, const int* __restrict__ sw, int C,
                                                float inv, float* __restrict__ res) {
    unpool_body<KMAX, AVG, CB>(fine, coarse, F, S, pad, cd, sw, C, inv, res);
}

// max_unpool (one covering output per fine voxel) and its switch-range check in one launch:
// blocks [0, ub) unpool, the others scan the switches, so the scan's 4 bytes per coarse entry
// stream beside the unpool's traffic instead of in a launch of their own.
__global__ void __launch_bounds__(256, HCB_POOL_MINB) k_unpool1_checked(DevPsh fine, DevPsh coarse, int F, int S,
                                                                        int pad, const float* __restrict__ cd,
                                                                        const int* __restrict__ sw, int C,
                                                                        float* __restrict__ res, long long nsw,
                                                                        int fd, int* bad, unsigned ub) {
    if (blockIdx.x >= ub) {
        check_switches_body(sw, nsw, fd, bad, (blockIdx.x - ub) * (long long)blockDim.x + threadIdx.x,
                            (long long)(gridDim.x - ub) * blockDim.x);
        return;
    }
    unpool_body<1, false, 16>(fine, coarse, F, S, pad, cd, sw, C, 0.0f, res);
}

template <bool AVG, typename T>
__global__ void k_unpool_any(DevPsh fine, DevPsh coarse, int F, int S, int pad, const T* __restrict__ cd,
                             const int* __restrict__ sw, int C, T inv, T* __restrict__ res) {
    const long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (gi >= fine.N) return;
    const int4 c = fine.cols[gi];
    const ModelParam mp = coarse.models[c.w - 1];
    const int dim = fine.dim;
    int lox, hix, loy, hiy, loz = 0, hiz = 0;
    cover_axis(c.x, F, S, pad, coarse.resolution, lox, hix);
    cover_axis(c.y, F, S, pad, coarse.resolution, loy, hiy);
    if (dim == 3) cover_axis(c.z, F, S, pad, coarse.resolution, loz, hiz);
    const long long Nc = coarse.N, Nf = fine.N;
    for (int ch = 0; ch < C; ++ch) {
        T acc = T(0);
        for (int z = loz; z <= hiz; ++z)
            for (int y = loy; y <= hiy; ++y)
                for (int x = lox; x <= hix; ++x) {
                    const int col = probe(coarse, mp, x, y, z);
                    if (col < 0) continue;
                    const long long k = ch * Nc + col;
                    if constexpr (AVG) {
                        acc = add_rn(acc, mul_rn(cd[k], inv));
                    } else {
                        const int rx = c.x - origin_axis(x, F, S, pad), ry = c.y - origin_axis(y, F, S, pad);
                        const int rz = dim == 3 ? c.z - origin_axis(z, F, S, pad) : 0;
                        if (sw[k] == (rz * F + ry) * F + rx) acc = add_rn(acc, cd[k]);
                    }
                }
        res[ch * Nf + gi] = acc;
    }
}

// Range scan of the switches (check_switches_body above): a standalone launch for the unpool
// variants that do not fold it in.
__global__ void k_check_switches(const int* sw, long long n, int fd, int* bad) {
    check_switches_body(sw, n, fd, bad, blockIdx.x * (long long)blockDim.x + threadIdx.x,
                        (long long)gridDim.x * blockDim.x);
}

// ============================================================== dispatch helpers
// cover count per axis: stride 1 -> F, else ceil(F/S)
int cover_per_axis(const hc_conv_spec& sp) {
    return sp.stride == 1 ? sp.kernel : (sp.kernel + sp.stride - 1) / sp.stride;
}

}  // namespace

// ------------------------------------------------------------------ launchers
void launch_field_map(const hc_psh* in, const hc_psh* out, const hc_conv_spec& sp, int* map, cudaStream_t s,
                      int layout = 0 /* 0 row-major, 1 tap-major, 2 tile-major */) {
    const long long n = out->d.N;
    if (n == 0) return;
    const unsigned g = grid_for(n, kThreads);
    const bool tap_major = layout == 1;
    if (layout == 2) {
        const unsigned gp = grid_for((n + 127) / 128 * 128, kThreads);
        if (sp.kernel == 3) k_field_map_tiled<3><<<gp, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, map);
        else if (sp.kernel == 2) k_field_map_tiled<2><<<gp, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, map);
        else k_field_map_any_tiled<<<gp, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad,
                                                         (int)field_volume(sp, in->d.dim), map);
    } else if (tap_major) {
        if (sp.kernel == 3) k_field_map_t<3><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, map);
        else if (sp.kernel == 2) k_field_map_t<2><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, map);
        else k_field_map_any_t<<<g, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad,
                                                     (int)field_volume(sp, in->d.dim), map);
    } else if (sp.kernel == 3) {
        k_field_map<3><<<grid_for(n, 128), 128, 0, s>>>(in->d, out->d, sp.stride, sp.pad, map);
    } else if (sp.kernel == 2) {
        k_field_map<2><<<grid_for(n, 128), 128, 0, s>>>(in->d, out->d, sp.stride, sp.pad, map);
    }
    else k_field_map_any<<<g, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad,
                                              (int)field_volume(sp, in->d.dim), map);
    launched("field_map");
}

void launch_hash2col(const hc_psh* in, const float* data, const hc_psh* out, const hc_conv_spec& sp, float* cols,
                     cudaStream_t s) {
    const long long n = out->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    const unsigned g = grid_for(n, kThreads);
    if (sp.kernel == 3)
    {
        static const int minb = env_int("HCB_H2C_MINB", 4);
        if (minb >= 4) k_hash2col<3, 4><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, cols);
        else if (minb >= 2) k_hash2col<3, 2><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, cols);
        else k_hash2col<3, 1><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, cols);
    }
    else if (sp.kernel == 2)
        k_hash2col<2, 4><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, cols);
    else
        k_hash2col_any<float><<<g, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad,
                                            (int)field_volume(sp, in->d.dim), data, sp.in_channels, cols);
    launched("hash2col");
}

void launch_col2hash(const float* gcols, const hc_psh* in, const hc_psh* out, const hc_conv_spec& sp, float* res,
                     cudaStream_t s) {
    const long long n = in->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    const unsigned g = grid_for(n, kThreads);
    const int fd = (int)field_volume(sp, in->d.dim);
    const int C = sp.in_channels;
    if (sp.stride == 1 && sp.kernel == 3 && (long long)fd * out->d.N < (1LL << 31))
    {
        static const int cu = env_int("HCB_C2H_CU", 16);
        if (cu == 16) k_col2hash_s1_tb<3, 16><<<g, kThreads, 0, s>>>(in->d, out->d, gcols, C, res);
        else if (cu == 8) k_col2hash_s1_tb<3, 8><<<g, kThreads, 0, s>>>(in->d, out->d, gcols, C, res);
        else if (cu >= 4) k_col2hash_s1<3, 4, 3><<<g, kThreads, 0, s>>>(in->d, out->d, gcols, C, res);
        else if (cu >= 2) k_col2hash_s1<3, 2, 3><<<g, kThreads, 0, s>>>(in->d, out->d, gcols, C, res);
        else k_col2hash_s1<3, 1, 4><<<g, kThreads, 0, s>>>(in->d, out->d, gcols, C, res);
    }
    else if (sp.stride == 1 && sp.kernel == 1)
        k_col2hash<1, true, 1><<<g, kThreads, 0, s>>>(in->d, out->d, 1, 1, 0, fd, gcols, C, res);
    else if (sp.stride > 1 && cover_per_axis(sp) == 1)
        k_col2hash<1, false, 1><<<g, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad, fd, gcols, C, res);
    else if (sp.stride > 1 && cover_per_axis(sp) == 2)
        k_col2hash<8, false, 1><<<g, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad, fd, gcols, C, res);
    else
        k_col2hash_any<float><<<g, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad, fd, gcols, C, res);
    launched("col2hash");
}

// staged 2^3 pooling (k_pool_staged) when the layout allows it; HCB_POOL_STAGED picks the
// (planes per stage, stages) shape for A/B runs, 0 = direct kernels
template <bool AVG>
bool launch_pool_staged(const hc_psh* in, const float* data, const hc_psh* out, const hc_conv_spec& sp, float inv,
                        float* res, int* sw, cudaStream_t s) {
    static const int mode = env_int("HCB_POOL_STAGED", 1);
    if (mode <= 0 || sp.kernel != 2 || in->d.dim != 3 || (reinterpret_cast<uintptr_t>(data) & 15) != 0) return false;
    const long long n = out->d.N;
    auto go = [&](auto kern, int pl, int ns, int bo = 256) {
        const int smem = pl * ns * (kPoolCap * bo / 256) * 4;
        const unsigned g = (unsigned)((n + bo - 1) / bo);
        smem_optin(kern, smem);  // once per (kernel, device)
        kern<<<g, bo + 32, smem, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, inv, res, sw);
    };
    // A/B at 256^3 x 8 (C 16 / 64 / 128, max_pool ms): (2 planes, 2 stages, 4 blocks/SM) 0.064 / 0.155 /
    // 0.278; (2, 3, 4) 0.083 / 0.157 / 0.264; (2, 3, 3) 0.070 / 0.152 / 0.269; (4, 2, 3) - / 0.164 / -
    // (before the presence-free reduction and batched probes); 128-voxel blocks: C 16 / 32 / 64 / 128
    // 0.058 / 0.086 / 0.143 / 0.258 vs 256-voxel blocks 0.058 / 0.087 / 0.147 / 0.260
    switch (mode) {
        case 2: go(k_pool_staged<2, 3, AVG, 4>, 2, 3); break;
        case 3: go(k_pool_staged<2, 3, AVG>, 2, 3); break;
        case 4: go(k_pool_staged<4, 2, AVG>, 4, 2); break;
        case 5: go(k_pool_staged<2, 2, AVG, 8, 128>, 2, 2, 128); break;
        case 6: go(k_pool_staged<2, 3, AVG, 6, 128>, 2, 3, 128); break;
        default:  // C >= 64: 128 coarse voxels per block, 6 blocks/SM (C 64 max 0.147 -> 0.143 ms)
            if (sp.in_channels >= 64) go(k_pool_staged<2, 3, AVG, 6, 128>, 2, 3, 128);
            else go(k_pool_staged<2, 2, AVG, 4>, 2, 2);
            break;
    }
    return true;
}

void launch_max_pool(const hc_psh* in, const float* data, const hc_psh* out, const hc_conv_spec& sp, float* res,
                     int* sw, cudaStream_t s) {
    const long long n = out->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    const unsigned g = grid_for(n, kThreads);
    // CB = 4 channels per pass (A/B at 256^3 x 8, C=64: CB 2 / 4 / 8 = 0.195 / 0.188 / 0.574 ms)
    if (launch_pool_staged<false>(in, data, out, sp, 0.0f, res, sw, s)) {
    } else if (sp.kernel == 2)
        k_max_pool<2, 4><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, res, sw);
    else if (sp.kernel == 3)
        k_max_pool<3, 1><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, res, sw);
    else
        k_max_pool_any<float><<<g, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad,
                                            (int)field_volume(sp, in->d.dim), data, sp.in_channels, res, sw);
    launched("max_pool");
}

void launch_avg_pool(const hc_psh* in, const float* data, const hc_psh* out, const hc_conv_spec& sp, float* res,
                     cudaStream_t s) {
    const long long n = out->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    const unsigned g = grid_for(n, kThreads);
    const long long fd = field_volume(sp, in->d.dim);
    const float inv = 1.0f / static_cast<float>(fd);  // cnn_ops.cpp:295
    if (launch_pool_staged<true>(in, data, out, sp, inv, res, nullptr, s)) {
    } else if (sp.kernel == 2)
        k_avg_pool<2, 4><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, inv, res);
    else if (sp.kernel == 3)
        k_avg_pool<3, 1><<<g, kThreads, 0, s>>>(in->d, out->d, sp.stride, sp.pad, data, sp.in_channels, inv, res);
    else
        k_avg_pool_any<float><<<g, kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad, (int)fd, data,
                                            sp.in_channels, inv, res);
    launched("avg_pool");
}

unsigned check_grid(long long nsw) {
    return (unsigned)std::min<long long>((nsw + 16 * kThreads - 1) / (16 * kThreads), 148 * 8);
}

// chk_flag: max_unpool's switch-range check (nsw switches, fd field rows) — folded into the
// F == S unpool launch, else launched first on its own
void launch_unpool(bool avg, const float* cd, const int* sw, const hc_psh* fine, const hc_psh* coarse,
                   const hc_conv_spec& sp, float* res, cudaStream_t s, int* chk_flag = nullptr, long long nsw = 0,
                   int fd = 0) {
    const long long n = fine->d.N;
    const int ka1 = cover_per_axis(sp);
    const bool fold = chk_flag && nsw > 0 && !avg && (fine->d.dim == 3 ? ka1 * ka1 * ka1 : ka1 * ka1) <= 1 &&
                      n > 0 && sp.in_channels > 0;
    if (chk_flag && nsw > 0 && !fold) {
        k_check_switches<<<check_grid(nsw), kThreads, 0, s>>>(sw, nsw, fd, chk_flag);
        launched("switch check");
    }
    if (n == 0 || sp.in_channels == 0) return;
    if (fold) {
        const unsigned ub = grid_for(n, kThreads);
        k_unpool1_checked<<<ub + check_grid(nsw), kThreads, 0, s>>>(fine->d, coarse->d, sp.kernel, sp.stride, sp.pad,
                                                                     cd, sw, sp.in_channels, res, nsw, fd, chk_flag,
                                                                     ub);
        launched("unpool + switch check");
        return;
    }
    const unsigned g = grid_for(n, kThreads);
    const float inv = 1.0f / static_cast<float>(field_volume(sp, fine->d.dim));  // cnn_ops.cpp:381
    const int ka = cover_per_axis(sp);
    const int kmax = fine->d.dim == 3 ? ka * ka * ka : ka * ka;
    const int C = sp.in_channels;
#define HC_UNPOOL(K)                                                                                             \
    (avg ? k_unpool<K, true, (K <= 1 ? 8 : 4)><<<g, kThreads, 0, s>>>(fine->d, coarse->d, sp.kernel, sp.stride, \
                                                                        sp.pad, cd, sw, C, inv, res)             \
         : k_unpool<K, false, (K <= 1 ? 8 : 4)><<<g, kThreads, 0, s>>>(fine->d, coarse->d, sp.kernel, sp.stride, \
                                                                         sp.pad, cd, sw, C, inv, res))
    // max_unpool with one covering output (F == S pooling): 16 channels per pass (A/B at 256^3 x 8,
    // C=64: CB 4 / 8 / 16 = 0.308 / 0.252 / 0.240 ms)
    if (kmax <= 1 && !avg)
        k_unpool<1, false, 16><<<g, kThreads, 0, s>>>(fine->d, coarse->d, sp.kernel, sp.stride, sp.pad, cd, sw, C,
                                                       inv, res);
    else if (kmax <= 1) HC_UNPOOL(1);
    else if (kmax <= 8) HC_UNPOOL(8);
    else if (kmax <= 27) HC_UNPOOL(27);
    else if (avg)
        k_unpool_any<true, float><<<g, kThreads, 0, s>>>(fine->d, coarse->d, sp.kernel, sp.stride, sp.pad, cd, sw, C, inv, res);
    else
        k_unpool_any<false, float><<<g, kThreads, 0, s>>>(fine->d, coarse->d, sp.kernel, sp.stride, sp.pad, cd, sw, C, inv, res);
#undef HC_UNPOOL
    launched("unpool");
}

// ------------------------------------------------------------------ contraction dispatch
void fast_gemm_nn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, cudaStream_t s);
void fast_gemm_tn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, cudaStream_t s);
void fast_gemm_nt(const float* a, const float* b, float* c, long long ra, long long k, long long rb, cudaStream_t s);
bool tc_gemm_nn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, bool three,
                cudaStream_t s);
bool tc_gemm_tn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, bool three,
                cudaStream_t s);
bool tc_gemm_nt(const float* a, const float* b, float* c, long long ra, long long k, long long rb, bool three,
                cudaStream_t s);

// HC_MATH_FAST: 3xTF32 tcgen05 (gemm_tc.cu) where the shapes are TMA-eligible, else FFMA
// tiles (gemm_fast.cu); HC_MATH_TF32: single-pass tf32 (same eligibility, FFMA otherwise).
void gemm_nn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, cudaStream_t s) {
    const hc_math m = current_math();
    if (m == HC_MATH_EXACT) return gemm_nn_exact(a, b, c, ra, k, cb, s);
    if (!tc_gemm_nn(a, b, c, ra, k, cb, m == HC_MATH_FAST, s)) fast_gemm_nn(a, b, c, ra, k, cb, s);
}
void gemm_tn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, cudaStream_t s) {
    const hc_math m = current_math();
    if (m == HC_MATH_EXACT) return gemm_tn_exact(a, b, c, ra, k, cb, s);
    if (!tc_gemm_tn(a, b, c, ra, k, cb, m == HC_MATH_FAST, s)) fast_gemm_tn(a, b, c, ra, k, cb, s);
}
void gemm_nt(const float* a, const float* b, float* c, long long ra, long long k, long long rb, cudaStream_t s) {
    const hc_math m = current_math();
    if (m == HC_MATH_EXACT) return gemm_nt_exact(a, b, c, ra, k, rb, s);
    if (!tc_gemm_nt(a, b, c, ra, k, rb, m == HC_MATH_FAST, s)) fast_gemm_nt(a, b, c, ra, k, rb, s);
}

// ------------------------------------------------------------------ fp64 (the reference's double
// instantiation, cnn_ops.cpp:652-653): the generic kernels, same order and rounding rules.
void launch_hash2col(const hc_psh* in, const double* data, const hc_psh* out, const hc_conv_spec& sp, double* cols,
                     cudaStream_t s) {
    const long long n = out->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    k_hash2col_any<double><<<grid_for(n, kThreads), kThreads, 0, s>>>(
        in->d, out->d, sp.kernel, sp.stride, sp.pad, (int)field_volume(sp, in->d.dim), data, sp.in_channels, cols);
    launched("hash2col (f64)");
}
void launch_col2hash(const double* gcols, const hc_psh* in, const hc_psh* out, const hc_conv_spec& sp, double* res,
                     cudaStream_t s) {
    const long long n = in->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    k_col2hash_any<double><<<grid_for(n, kThreads), kThreads, 0, s>>>(
        in->d, out->d, sp.kernel, sp.stride, sp.pad, (int)field_volume(sp, in->d.dim), gcols, sp.in_channels, res);
    launched("col2hash (f64)");
}
void launch_max_pool(const hc_psh* in, const double* data, const hc_psh* out, const hc_conv_spec& sp, double* res,
                     int* sw, cudaStream_t s) {
    const long long n = out->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    k_max_pool_any<double><<<grid_for(n, kThreads), kThreads, 0, s>>>(
        in->d, out->d, sp.kernel, sp.stride, sp.pad, (int)field_volume(sp, in->d.dim), data, sp.in_channels, res, sw);
    launched("max_pool (f64)");
}
void launch_avg_pool(const hc_psh* in, const double* data, const hc_psh* out, const hc_conv_spec& sp, double* res,
                     cudaStream_t s) {
    const long long n = out->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    const long long fd = field_volume(sp, in->d.dim);
    const double inv = 1.0 / static_cast<double>(fd);  // cnn_ops.cpp:295
    k_avg_pool_any<double><<<grid_for(n, kThreads), kThreads, 0, s>>>(in->d, out->d, sp.kernel, sp.stride, sp.pad,
                                                                      (int)fd, data, sp.in_channels, inv, res);
    launched("avg_pool (f64)");
}
void launch_unpool(bool avg, const double* cd, const int* sw, const hc_psh* fine, const hc_psh* coarse,
                   const hc_conv_spec& sp, double* res, cudaStream_t s) {
    const long long n = fine->d.N;
    if (n == 0 || sp.in_channels == 0) return;
    const unsigned g = grid_for(n, kThreads);
    const double inv = 1.0 / static_cast<double>(field_volume(sp, fine->d.dim));  // cnn_ops.cpp:381
    if (avg)
        k_unpool_any<true, double><<<g, kThreads, 0, s>>>(fine->d, coarse->d, sp.kernel, sp.stride, sp.pad, cd, sw,
                                                          sp.in_channels, inv, res);
    else
        k_unpool_any<false, double><<<g, kThreads, 0, s>>>(fine->d, coarse->d, sp.kernel, sp.stride, sp.pad, cd, sw,
                                                           sp.in_channels, inv, res);
    launched("unpool (f64)");
}
// fp64 contraction: always the order-exact kernels (the math mode selects fp32 paths only)
void gemm_nn(const double* a, const double* b, double* c, long long ra, long long k, long long cb, cudaStream_t s) {
    gemm_nn_exact(a, b, c, ra, k, cb, s);
}
void gemm_tn(const double* a, const double* b, double* c, long long ra, long long k, long long cb, cudaStream_t s) {
    gemm_tn_exact(a, b, c, ra, k, cb, s);
}
void gemm_nt(const double* a, const double* b, double* c, long long ra, long long k, long long rb, cudaStream_t s) {
    gemm_nt_exact(a, b, c, ra, k, rb, s);
}

}  // namespace hcb

using namespace hcb;

// ====================================================================== C ABI
namespace hcb {

template <typename T>
hc_status hash2col_impl(const hc_psh* in, const T* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, T* cols, hc_stream stream) {
    return guard([&] {
        check_pair(in, out, spec);
        if (data_rows != spec.in_channels || data_cols != in->d.N)
            throw std::invalid_argument("hash2col: input data shape mismatch");
        launch_hash2col(in, data, out, spec, cols, as_stream(stream));
    });
}

template <typename T>
hc_status col2hash_impl(const T* col_grads, int64_t rows, int64_t cols, const hc_psh* in, const hc_psh* out,
                          hc_conv_spec spec, T* result, hc_stream stream) {
    return guard([&] {
        check_pair(in, out, spec);
        const long long fd = field_volume(spec, in->d.dim);
        if (rows != spec.in_channels * fd || cols != out->d.N)
            throw std::invalid_argument("col2hash: column gradient shape mismatch");
        launch_col2hash(col_grads, in, out, spec, result, as_stream(stream));
    });
}

template <typename T>
hc_status conv_forward_impl(const hc_psh* in, const T* data, int64_t data_rows, int64_t data_cols,
                              const hc_psh* out, const T* w, int64_t w_rows, int64_t w_cols, hc_conv_spec spec,
                              T* result, hc_stream stream) {
    return guard([&] {
        if (!in || !out) throw std::invalid_argument("null super-PSH handle");
        const long long fd = field_volume(spec, in->d.dim);
        if (w_rows != spec.out_channels || w_cols != spec.in_channels * fd)
            throw std::invalid_argument("conv_forward: weight shape mismatch");
        check_pair(in, out, spec);
        if (data_rows != spec.in_channels || data_cols != in->d.N)
            throw std::invalid_argument("hash2col: input data shape mismatch");
        cudaStream_t s = as_stream(stream);
        const long long K = spec.in_channels * fd, N = out->d.N;
        if constexpr (std::is_same_v<T, float>) {
            if (current_math() == HC_MATH_FAST && N > 0 && fused_x2_eligible(in, out, spec, (int)fd)) {
                fused_conv_forward_f32(in, data, w, spec, (int)fd, N, result, s);  // no column matrix
                fused_route_count(1);
                return;
            }
        }
        Scratch cols(sizeof(T) * K * N, s);
        launch_hash2col(in, data, out, spec, cols.as<T>(), s);
        gemm_nn(w, cols.as<T>(), result, spec.out_channels, K, N, s);
    });
}

template <typename T>
hc_status conv_backward_impl(const T* output_grad, int64_t g_rows, int64_t g_cols, const T* w,
                               int64_t w_rows, int64_t w_cols, const T* cached_cols, int64_t c_rows,
                               int64_t c_cols, const hc_psh* in, const hc_psh* out, hc_conv_spec spec, T* dw,
                               T* dx, hc_stream stream) {
    return guard([&] {
        if (!in || !out) throw std::invalid_argument("null super-PSH handle");
        const long long fd = field_volume(spec, in->d.dim);
        if (g_rows != spec.out_channels || g_cols != out->d.N)
            throw std::invalid_argument("conv_backward: output gradient shape mismatch");
        if (c_rows != spec.in_channels * fd || c_cols != out->d.N)
            throw std::invalid_argument("conv_backward: cached column shape mismatch");
        // gemm.cpp:80-93 shape checks of the two products, then col2hash's
        if (w_rows != g_rows) throw std::invalid_argument("matmul_trans_a: shape mismatch");
        check_pair(in, out, spec);
        if (w_cols != spec.in_channels * fd) throw std::invalid_argument("col2hash: column gradient shape mismatch");
        cudaStream_t s = as_stream(stream);
        if constexpr (std::is_same_v<T, float>) {
            if (current_math() == HC_MATH_FAST && g_cols > 0 && fused_x2_eligible(in, out, spec, (int)fd)) {
                fused_conv_backward_f32(output_grad, w, cached_cols, in, spec, (int)fd, g_cols, dw, dx, s);
                fused_route_count(1);
                return;
            }
        }
        gemm_nt(output_grad, cached_cols, dw, g_rows, g_cols, c_rows, s);  // dW = dDo * cols^T
        Scratch dcols(sizeof(T) * w_cols * g_cols, s);
        gemm_tn(w, output_grad, dcols.as<T>(), w_rows, w_cols, g_cols, s);  // W^T * dDo
        launch_col2hash(dcols.as<T>(), in, out, spec, dx, s);
    });
}

template <typename T>
hc_status max_pool_impl(const hc_psh* in, const T* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, T* result, int32_t* switches, hc_stream stream) {
    return guard([&] {
        check_pair(in, out, spec);
        if (spec.stride < 2) throw std::invalid_argument("pooling requires stride >= 2");
        if (data_rows != spec.in_channels || data_cols != in->d.N)
            throw std::invalid_argument("max_pool: input data shape mismatch");
        launch_max_pool(in, data, out, spec, result, switches, as_stream(stream));
    });
}

template <typename T>
hc_status avg_pool_impl(const hc_psh* in, const T* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, T* result, hc_stream stream) {
    return guard([&] {
        check_pair(in, out, spec);
        if (spec.stride < 2) throw std::invalid_argument("pooling requires stride >= 2");
        if (data_rows != spec.in_channels || data_cols != in->d.N)
            throw std::invalid_argument("avg_pool: input data shape mismatch");
        launch_avg_pool(in, data, out, spec, result, as_stream(stream));
    });
}

template <typename T>
hc_status max_unpool_impl(const T* coarse_data, int64_t c_rows, int64_t c_cols, const int32_t* switches,
                            int64_t s_rows, int64_t s_cols, const hc_psh* fine, const hc_psh* coarse,
                            hc_conv_spec spec, T* result, hc_stream stream) {
    return guard([&] {
        check_pair(fine, coarse, spec);
        const long long fd = field_volume(spec, fine->d.dim);
        if (c_rows != spec.in_channels || c_cols != coarse->d.N)
            throw std::invalid_argument("max_unpool: coarse data shape mismatch");
        // cnn_ops.cpp:326-332 check_switches, stream-ordered and without a host round trip: the
        // scan raises a sticky flag in mapped host memory that hc_deferred_status() reports
        // (with the reference's message) once the caller has synchronised; an out-of-range
        // switch matches no field row, so the unpool itself stays in bounds.
        if (s_rows != spec.in_channels || s_cols != coarse->d.N)
            throw std::invalid_argument("unpool: switch shape mismatch");
        cudaStream_t s = as_stream(stream);
        const long long n = s_rows * s_cols;
        if constexpr (std::is_same_v<T, float>) {
            launch_unpool(false, coarse_data, switches, fine, coarse, spec, result, s, deferred_flag_device(), n,
                          (int)fd);
        } else {
            if (n > 0) {
                k_check_switches<<<check_grid(n), kThreads, 0, s>>>(switches, n, (int)fd, deferred_flag_device());
                launched("switch check");
            }
            launch_unpool(false, coarse_data, switches, fine, coarse, spec, result, s);
        }
    });
}

template <typename T>
hc_status avg_unpool_impl(const T* coarse_data, int64_t c_rows, int64_t c_cols, const hc_psh* fine,
                            const hc_psh* coarse, hc_conv_spec spec, T* result, hc_stream stream) {
    return guard([&] {
        check_pair(fine, coarse, spec);
        if (c_rows != spec.in_channels || c_cols != coarse->d.N)
            throw std::invalid_argument("avg_unpool: coarse data shape mismatch");
        launch_unpool(true, coarse_data, nullptr, fine, coarse, spec, result, as_stream(stream));
    });
}

template <typename T>
hc_status deconv_forward_impl(const hc_psh* coarse, const T* coarse_data, int64_t d_rows, int64_t d_cols,
                                const hc_psh* fine, const T* w, int64_t w_rows, int64_t w_cols,
                                hc_conv_spec spec, T* result, hc_stream stream) {
    return guard([&] {
        if (!coarse || !fine) throw std::invalid_argument("null super-PSH handle");
        const long long fd = field_volume(spec, fine->d.dim);
        if (w_rows != spec.out_channels || w_cols != spec.in_channels * fd)
            throw std::invalid_argument("deconv_forward: weight shape mismatch");
        if (d_rows != spec.out_channels || d_cols != coarse->d.N)
            throw std::invalid_argument("deconv_forward: coarse data shape mismatch");
        check_pair(fine, coarse, spec);
        cudaStream_t s = as_stream(stream);
        Scratch cols(sizeof(T) * w_cols * d_cols, s);
        gemm_tn(w, coarse_data, cols.as<T>(), w_rows, w_cols, d_cols, s);  // W^T * D_i
        launch_col2hash(cols.as<T>(), fine, coarse, spec, result, s);
    });
}

template <typename T>
hc_status deconv_backward_impl(const T* fine_grad, int64_t g_rows, int64_t g_cols, const T* w,
                                 int64_t w_rows, int64_t w_cols, const T* cached_coarse, int64_t c_rows,
                                 int64_t c_cols, const hc_psh* coarse, const hc_psh* fine, hc_conv_spec spec,
                                 T* dw, T* dx, hc_stream stream) {
    return guard([&] {
        if (!coarse || !fine) throw std::invalid_argument("null super-PSH handle");
        if (g_rows != spec.in_channels || g_cols != fine->d.N)
            throw std::invalid_argument("deconv_backward: fine gradient shape mismatch");
        check_pair(fine, coarse, spec);
        const long long fd = field_volume(spec, fine->d.dim);
        const long long K = spec.in_channels * fd, N = coarse->d.N;
        if (c_cols != N) throw std::invalid_argument("matmul_trans_b: shape mismatch");
        if (w_cols != K) throw std::invalid_argument("matmul: shape mismatch");
        cudaStream_t s = as_stream(stream);
        Scratch dcols(sizeof(T) * K * N, s);
        launch_hash2col(fine, fine_grad, coarse, spec, dcols.as<T>(), s);  // adjoint of col2hash
        gemm_nt(cached_coarse, dcols.as<T>(), dw, c_rows, N, K, s);        // dW = D_i * dcols^T
        gemm_nn(w, dcols.as<T>(), dx, w_rows, K, N, s);                    // dD_i = W * dcols
    });
}

template <typename T>
hc_status matmul_impl(const T* a, const T* b, T* c, int64_t ra, int64_t k, int64_t cb, hc_stream stream) {
    return guard([&] { gemm_nn(a, b, c, ra, k, cb, as_stream(stream)); });
}

template <typename T>
hc_status matmul_trans_a_impl(const T* a, const T* b, T* c, int64_t ra, int64_t k, int64_t cb,
                                hc_stream stream) {
    return guard([&] { gemm_tn(a, b, c, ra, k, cb, as_stream(stream)); });
}

template <typename T>
hc_status matmul_trans_b_impl(const T* a, const T* b, T* c, int64_t ra, int64_t k, int64_t rb,
                                hc_stream stream) {
    return guard([&] { gemm_nt(a, b, c, ra, k, rb, as_stream(stream)); });
}

}  // namespace hcb

extern "C" {

hc_status hc_field_map(const hc_psh* in, const hc_psh* out, hc_conv_spec spec, int32_t* map, hc_stream stream) {
    return guard([&] {
        check_pair(in, out, spec);
        launch_field_map(in, out, spec, map, as_stream(stream));
    });
}

hc_status hc_field_map_tap_major(const hc_psh* in, const hc_psh* out, hc_conv_spec spec, int32_t* map,
                                 hc_stream stream) {
    return guard([&] {
        check_pair(in, out, spec);
        launch_field_map(in, out, spec, map, as_stream(stream), 1);
    });
}

hc_status hc_field_map_tiled(const hc_psh* in, const hc_psh* out, hc_conv_spec spec, int32_t* map,
                             hc_stream stream) {
    return guard([&] {
        check_pair(in, out, spec);
        launch_field_map(in, out, spec, map, as_stream(stream), 2);
    });
}

hc_status hc_hash2col_f32(const hc_psh* in, const float* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, float* cols, hc_stream stream) {
    return hash2col_impl<float>(in, data, data_rows, data_cols, out, spec, cols, stream);
}
hc_status hc_hash2col_f64(const hc_psh* in, const double* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, double* cols, hc_stream stream) {
    return hash2col_impl<double>(in, data, data_rows, data_cols, out, spec, cols, stream);
}

hc_status hc_col2hash_f32(const float* col_grads, int64_t rows, int64_t cols, const hc_psh* in, const hc_psh* out,
                          hc_conv_spec spec, float* result, hc_stream stream) {
    return col2hash_impl<float>(col_grads, rows, cols, in, out, spec, result, stream);
}
hc_status hc_col2hash_f64(const double* col_grads, int64_t rows, int64_t cols, const hc_psh* in, const hc_psh* out,
                          hc_conv_spec spec, double* result, hc_stream stream) {
    return col2hash_impl<double>(col_grads, rows, cols, in, out, spec, result, stream);
}

hc_status hc_conv_forward_f32(const hc_psh* in, const float* data, int64_t data_rows, int64_t data_cols,
                              const hc_psh* out, const float* w, int64_t w_rows, int64_t w_cols, hc_conv_spec spec,
                              float* result, hc_stream stream) {
    return conv_forward_impl<float>(in, data, data_rows, data_cols, out, w, w_rows, w_cols, spec, result, stream);
}
hc_status hc_conv_forward_f64(const hc_psh* in, const double* data, int64_t data_rows, int64_t data_cols,
                              const hc_psh* out, const double* w, int64_t w_rows, int64_t w_cols, hc_conv_spec spec,
                              double* result, hc_stream stream) {
    return conv_forward_impl<double>(in, data, data_rows, data_cols, out, w, w_rows, w_cols, spec, result, stream);
}

hc_status hc_conv_backward_f32(const float* output_grad, int64_t g_rows, int64_t g_cols, const float* w,
                               int64_t w_rows, int64_t w_cols, const float* cached_cols, int64_t c_rows,
                               int64_t c_cols, const hc_psh* in, const hc_psh* out, hc_conv_spec spec, float* dw,
                               float* dx, hc_stream stream) {
    return conv_backward_impl<float>(output_grad, g_rows, g_cols, w, w_rows, w_cols, cached_cols, c_rows, c_cols, in, out, spec, dw, dx, stream);
}
hc_status hc_conv_backward_f64(const double* output_grad, int64_t g_rows, int64_t g_cols, const double* w,
                               int64_t w_rows, int64_t w_cols, const double* cached_cols, int64_t c_rows,
                               int64_t c_cols, const hc_psh* in, const hc_psh* out, hc_conv_spec spec, double* dw,
                               double* dx, hc_stream stream) {
    return conv_backward_impl<double>(output_grad, g_rows, g_cols, w, w_rows, w_cols, cached_cols, c_rows, c_cols, in, out, spec, dw, dx, stream);
}

hc_status hc_max_pool_f32(const hc_psh* in, const float* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, float* result, int32_t* switches, hc_stream stream) {
    return max_pool_impl<float>(in, data, data_rows, data_cols, out, spec, result, switches, stream);
}
hc_status hc_max_pool_f64(const hc_psh* in, const double* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, double* result, int32_t* switches, hc_stream stream) {
    return max_pool_impl<double>(in, data, data_rows, data_cols, out, spec, result, switches, stream);
}

hc_status hc_avg_pool_f32(const hc_psh* in, const float* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, float* result, hc_stream stream) {
    return avg_pool_impl<float>(in, data, data_rows, data_cols, out, spec, result, stream);
}
hc_status hc_avg_pool_f64(const hc_psh* in, const double* data, int64_t data_rows, int64_t data_cols, const hc_psh* out,
                          hc_conv_spec spec, double* result, hc_stream stream) {
    return avg_pool_impl<double>(in, data, data_rows, data_cols, out, spec, result, stream);
}

hc_status hc_max_unpool_f32(const float* coarse_data, int64_t c_rows, int64_t c_cols, const int32_t* switches,
                            int64_t s_rows, int64_t s_cols, const hc_psh* fine, const hc_psh* coarse,
                            hc_conv_spec spec, float* result, hc_stream stream) {
    return max_unpool_impl<float>(coarse_data, c_rows, c_cols, switches, s_rows, s_cols, fine, coarse, spec, result, stream);
}
hc_status hc_max_unpool_f64(const double* coarse_data, int64_t c_rows, int64_t c_cols, const int32_t* switches,
                            int64_t s_rows, int64_t s_cols, const hc_psh* fine, const hc_psh* coarse,
                            hc_conv_spec spec, double* result, hc_stream stream) {
    return max_unpool_impl<double>(coarse_data, c_rows, c_cols, switches, s_rows, s_cols, fine, coarse, spec, result, stream);
}

hc_status hc_avg_unpool_f32(const float* coarse_data, int64_t c_rows, int64_t c_cols, const hc_psh* fine,
                            const hc_psh* coarse, hc_conv_spec spec, float* result, hc_stream stream) {
    return avg_unpool_impl<float>(coarse_data, c_rows, c_cols, fine, coarse, spec, result, stream);
}
hc_status hc_avg_unpool_f64(const double* coarse_data, int64_t c_rows, int64_t c_cols, const hc_psh* fine,
                            const hc_psh* coarse, hc_conv_spec spec, double* result, hc_stream stream) {
    return avg_unpool_impl<double>(coarse_data, c_rows, c_cols, fine, coarse, spec, result, stream);
}

hc_status hc_deconv_forward_f32(const hc_psh* coarse, const float* coarse_data, int64_t d_rows, int64_t d_cols,
                                const hc_psh* fine, const float* w, int64_t w_rows, int64_t w_cols,
                                hc_conv_spec spec, float* result, hc_stream stream) {
    return deconv_forward_impl<float>(coarse, coarse_data, d_rows, d_cols, fine, w, w_rows, w_cols, spec, result, stream);
}
hc_status hc_deconv_forward_f64(const hc_psh* coarse, const double* coarse_data, int64_t d_rows, int64_t d_cols,
                                const hc_psh* fine, const double* w, int64_t w_rows, int64_t w_cols,
                                hc_conv_spec spec, double* result, hc_stream stream) {
    return deconv_forward_impl<double>(coarse, coarse_data, d_rows, d_cols, fine, w, w_rows, w_cols, spec, result, stream);
}

hc_status hc_deconv_backward_f32(const float* fine_grad, int64_t g_rows, int64_t g_cols, const float* w,
                                 int64_t w_rows, int64_t w_cols, const float* cached_coarse, int64_t c_rows,
                                 int64_t c_cols, const hc_psh* coarse, const hc_psh* fine, hc_conv_spec spec,
                                 float* dw, float* dx, hc_stream stream) {
    return deconv_backward_impl<float>(fine_grad, g_rows, g_cols, w, w_rows, w_cols, cached_coarse, c_rows, c_cols, coarse, fine, spec, dw, dx, stream);
}
hc_status hc_deconv_backward_f64(const double* fine_grad, int64_t g_rows, int64_t g_cols, const double* w,
                                 int64_t w_rows, int64_t w_cols, const double* cached_coarse, int64_t c_rows,
                                 int64_t c_cols, const hc_psh* coarse, const hc_psh* fine, hc_conv_spec spec,
                                 double* dw, double* dx, hc_stream stream) {
    return deconv_backward_impl<double>(fine_grad, g_rows, g_cols, w, w_rows, w_cols, cached_coarse, c_rows, c_cols, coarse, fine, spec, dw, dx, stream);
}

hc_status hc_matmul_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k, int64_t cb, hc_stream stream) {
    return matmul_impl<float>(a, b, c, ra, k, cb, stream);
}
hc_status hc_matmul_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k, int64_t cb, hc_stream stream) {
    return matmul_impl<double>(a, b, c, ra, k, cb, stream);
}
hc_status hc_matmul_trans_a_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k, int64_t cb,
                                hc_stream stream) {
    return matmul_trans_a_impl<float>(a, b, c, ra, k, cb, stream);
}
hc_status hc_matmul_trans_a_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k, int64_t cb,
                                hc_stream stream) {
    return matmul_trans_a_impl<double>(a, b, c, ra, k, cb, stream);
}
hc_status hc_matmul_trans_b_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k, int64_t rb,
                                hc_stream stream) {
    return matmul_trans_b_impl<float>(a, b, c, ra, k, rb, stream);
}
hc_status hc_matmul_trans_b_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k, int64_t rb,
                                hc_stream stream) {
    return matmul_trans_b_impl<double>(a, b, c, ra, k, rb, stream);
}

}  // extern "C"
