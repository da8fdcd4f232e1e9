// conv_tc.cu — the native (voxel-major) fused hash-conv on 5th-gen tensor cores.
//
// Implicit GEMM: the hash2col column matrix is never materialised. For output
// voxel n and field row t the field map (K0, ops_ref.cu) gives the input column
// nbr[n][t] (or -1); the A operand of the GEMM is gathered straight from the
// voxel-major feature rows X[nbr][:] into shared memory with 16-byte cp.async
// (zero-fill for empty cells), laid out in the UMMA SWIZZLE_128B canonical form,
// and tcgen05.mma accumulates in TMEM.
//
//   forward        Y [n][co]  = sum_{t,ci} X[nbr[n][t]][ci] * W[co][t][ci]
//   backward-data  dX[g][ci]  = sum_{t,co} dY[nbr[g][t]][co] * W[co][26-t][ci]
//                  (stride 1: the same kernel with flipped/transposed weights;
//                   cnn_ops.cpp:217-232 computes col2hash(W^T dY), the same sum)
//   weight grad    dW[co][t][ci] = sum_n dY[n][co] * X[nbr[n][t]][ci]
//                  (reduction over voxels: split-K over CTAs, partials reduced in a
//                   fixed order -> deterministic; both operands MN-major)
//
// Numerics: bf16 operands, fp32 accumulation (TMEM), fp32 or bf16 outputs.
// Tolerance-level parity against the double oracle (tests/test_conv_tc.py).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "hashconv_b200_native.h"
#include "hc_internal.h"
#include "hc_launch.cuh"
#include "tc_common.cuh"

namespace hcb {

namespace {

using bf16 = __nv_bfloat16;
using namespace tc;

constexpr int BM = 128;          // voxels (GEMM M) per CTA tile
constexpr int BK = 64;           // K elements (bf16) per pipeline stage = one 128 B row
constexpr int kProducers = 128;  // warps 0-3: cp.async producers, then epilogue
constexpr int kThreads = 160;    // + warp 4: TMEM allocator and MMA issuer

__host__ __device__ constexpr int tmem_cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256; }

template <int BN>
struct FwdCfg {
    static constexpr int STAGES = BN <= 64 ? 4 : 3;
    static constexpr int A_BYTES = BM * 128;      // 16 KB
    static constexpr int B_BYTES = BN * 128;      // BN rows of 128 B
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int MAX_TAPS = 27;
    static constexpr int SMEM = 1024 /*align slack*/ + STAGES * STAGE_BYTES + BM * MAX_TAPS * 4 + 256;
};

__device__ __forceinline__ void store_row(float* dst, const float (&v)[16]) {
#pragma unroll
    for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
}
__device__ __forceinline__ void store_row(bf16* dst, const float (&v)[16]) {
    uint32_t p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        p[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(dst) = make_uint4(p[0], p[1], p[2], p[3]);
    *reinterpret_cast<uint4*>(dst + 8) = make_uint4(p[4], p[5], p[6], p[7]);
}

// ====================================================================== gather-GEMM
// Y[m][0:BN] = sum_k A[m][k] * Wp[0:BN][k],  A[m][k] = X[nbr[m][k / C]][k % C] (0 if -1)
// One CTA per 128-row tile. K = taps*C (C % 8 == 0), Kp = K rounded up to 64.
template <int BN, typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    k_gather_gemm(const int* __restrict__ nbr, int taps, long long rows, const bf16* __restrict__ X, int C,
                  const bf16* __restrict__ Wp, int Kp, OutT* __restrict__ Y) {
    using Cfg = FwdCfg<BN>;
    constexpr int S = Cfg::STAGES;
    constexpr int LAG = S - 1;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_base = smem;
    int* nbr_s = reinterpret_cast<int*>(smem + S * Cfg::STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES + BM * Cfg::MAX_TAPS * 4);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 1);

    const int tid = threadIdx.x, warp = tid >> 5;
    const long long m0 = (long long)blockIdx.x * BM;
    const int K = taps * C;
    const int nkb = Kp / BK;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S), done = smem_u32(bars + 2 * S);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, kProducers);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(done, 1);
        mbar_init_fence();
    }
    if (warp == 4) tmem_alloc(smem_u32(tmem_slot), tmem_cols(BN));
    // stage this tile's field-map rows (coalesced)
    for (int i = tid; i < BM * taps; i += kThreads) {
        const long long r = m0 + i / taps;
        nbr_s[i] = r < rows ? __ldg(nbr + m0 * taps + i) : -1;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        // ---------------- producers: gather A rows and W rows into the ring
        const int c = tid & 7;      // 16-byte chunk within a 128-byte row
        const int r0 = tid >> 3;    // first row handled (then +16 per step)
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % S;
            if (kb >= S) mbar_wait(empty0 + 8 * s, ((kb / S) - 1) & 1);
            uint8_t* A = stage_base + s * Cfg::STAGE_BYTES;
            uint8_t* B = A + Cfg::A_BYTES;
            const int k = kb * BK + c * 8;
            const bool kin = k < K;
            const int t = kin ? k / C : 0;
            const int ci = kin ? k - t * C : 0;
#pragma unroll
            for (int j = 0; j < BM / 16; ++j) {
                const int r = r0 + 16 * j;
                const int g = kin ? nbr_s[r * taps + t] : -1;
                const bf16* src = g >= 0 ? X + (long long)g * C + ci : X;
                cp_async16(smem_u32(A + sw128_offset(r, c)), src, g >= 0 ? 16u : 0u);
            }
#pragma unroll
            for (int j = 0; j < BN / 16; ++j) {
                const int r = r0 + 16 * j;
                cp_async16(smem_u32(B + sw128_offset(r, c)), Wp + (long long)r * Kp + kb * BK + c * 8, 16u);
            }
            cp_async_commit();
            if (kb >= LAG) {
                cp_async_wait<LAG>();
                fence_proxy_async();
                mbar_arrive(full0 + 8 * ((kb - LAG) % S));
            }
        }
        cp_async_wait<0>();
        fence_proxy_async();
        for (int kb = std::max(0, nkb - LAG); kb < nkb; ++kb) mbar_arrive(full0 + 8 * (kb % S));

        // ---------------- epilogue: TMEM -> registers -> Y rows
        mbar_wait(done, 0);
        tc_fence_after();
        const int row = warp * 32 + (int)lane_id();
        const long long m = m0 + row;
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
            tmem_ld_wait();
            float f[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
            if (m < rows) store_row(Y + m * BN + c0, f);
        }
    } else if (tid == 4 * 32) {
        // ---------------- MMA issuer (single thread)
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, false, false);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % S;
            mbar_wait(full0 + 8 * s, (kb / S) & 1);
            tc_fence_after();
            const uint32_t a = smem_u32(stage_base + s * Cfg::STAGE_BYTES);
            const uint32_t b = a + Cfg::A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
                mma_bf16(tmem, sw128_desc(a + kk * 32, 16, 1024), sw128_desc(b + kk * 32, 16, 1024), idesc,
                         (kb | kk) != 0);
            mma_commit(empty0 + 8 * s);
        }
        mma_commit(done);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, tmem_cols(BN));
    }
}

// ====================================================================== weight gradient
// Partial[split][m][co] = sum over this split's voxels n of A[m][n] * B[co][n]
//   A[m][n] = X[nbr[n][m / C]][m % C]  (m = t*C + ci; MN-major: 128 B rows per voxel)
//   B[co][n] = dY[n][co]               (MN-major; C_out < 64 zero-padded to 64)
template <int NB>  // N tile = padded C_out (64, 128 or 256)
struct DwCfg {
    static constexpr int KB = 64;                  // voxels per stage
    static constexpr int STAGES = NB <= 64 ? 4 : 3;
    static constexpr int A_BYTES = 2 * KB * 128;   // two 64-wide MN blocks (M = 128)
    static constexpr int B_BYTES = (NB / 64) * KB * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;
};

template <int NB>
__global__ void __launch_bounds__(kThreads, 1)
    k_gather_dw(const int* __restrict__ nbr, int taps, long long rows, const bf16* __restrict__ X, int C,
                const bf16* __restrict__ dY, int Cout, int kb_per_split, float* __restrict__ partial, int Mtot) {
    using Cfg = DwCfg<NB>;
    constexpr int S = Cfg::STAGES;
    constexpr int LAG = S - 1;
    constexpr int KB = Cfg::KB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 1);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int mt = blockIdx.x, split = blockIdx.y;
    const long long total_kb = (rows + KB - 1) / KB;
    const long long kb_begin = (long long)split * kb_per_split;
    const int nkb = (int)std::max<long long>(0, std::min<long long>(kb_per_split, total_kb - kb_begin));
    const int K = taps * C;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S), done = smem_u32(bars + 2 * S);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, kProducers);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(done, 1);
        mbar_init_fence();
    }
    if (warp == 4) tmem_alloc(smem_u32(tmem_slot), tmem_cols(NB));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        const int c = tid & 7;
        const int q0 = tid >> 3;  // 0..15
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % S;
            if (kb >= S) mbar_wait(empty0 + 8 * s, ((kb / S) - 1) & 1);
            uint8_t* A = smem + s * Cfg::STAGE_BYTES;
            uint8_t* B = A + Cfg::A_BYTES;
            const long long n0 = (kb_begin + kb) * KB;
            // A: 2 MN blocks x 64 voxel rows x 8 chunks = 1024 chunks, 8 per thread
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int q = q0 + 16 * j;        // 0..127 = (block, voxel row)
                const int blk = q >> 6, r = q & 63;
                const int mm = mt * BM + blk * 64 + c * 8;
                const long long n = n0 + r;
                int g = -1, ci = 0;
                if (mm < K && n < rows) {
                    const int t = mm / C;
                    ci = mm - t * C;
                    g = __ldg(nbr + n * taps + t);
                }
                const bf16* src = g >= 0 ? X + (long long)g * C + ci : X;
                cp_async16(smem_u32(A + blk * (KB * 128) + sw128_offset(r, c)), src, g >= 0 ? 16u : 0u);
            }
            // B: NB/64 blocks x 64 voxel rows x 8 chunks
#pragma unroll
            for (int j = 0; j < (NB / 64) * 4; ++j) {
                const int q = q0 + 16 * j;
                const int blk = q >> 6, r = q & 63;
                const int co = blk * 64 + c * 8;
                const long long n = n0 + r;
                const bool ok = co < Cout && n < rows;
                const bf16* src = ok ? dY + n * Cout + co : dY;
                cp_async16(smem_u32(B + blk * (KB * 128) + sw128_offset(r, c)), src, ok ? 16u : 0u);
            }
            cp_async_commit();
            if (kb >= LAG) {
                cp_async_wait<LAG>();
                fence_proxy_async();
                mbar_arrive(full0 + 8 * ((kb - LAG) % S));
            }
        }
        cp_async_wait<0>();
        fence_proxy_async();
        for (int kb = std::max(0, nkb - LAG); kb < nkb; ++kb) mbar_arrive(full0 + 8 * (kb % S));

        // epilogue: row m = (t,ci) index, columns co
        const int row = warp * 32 + (int)lane_id();
        float* dst = partial + ((long long)split * Mtot + (long long)mt * BM + row) * NB;
        if (nkb == 0) {
#pragma unroll
            for (int c0 = 0; c0 < NB; c0 += 4) *reinterpret_cast<float4*>(dst + c0) = make_float4(0, 0, 0, 0);
        } else {
            mbar_wait(done, 0);
            tc_fence_after();
#pragma unroll
            for (int c0 = 0; c0 < NB; c0 += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
                tmem_ld_wait();
                float f[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
                store_row(dst + c0, f);
            }
        }
    } else if (tid == 4 * 32 && nkb > 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(BM, NB, true, true);
        constexpr uint32_t LBO = KB * 128;  // next 64-wide MN block
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % S;
            mbar_wait(full0 + 8 * s, (kb / S) & 1);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + s * Cfg::STAGE_BYTES);
            const uint32_t b = a + Cfg::A_BYTES;
#pragma unroll
            for (int kk = 0; kk < KB / 16; ++kk)  // 16 voxels = two 8-row atoms per MMA
                mma_bf16(tmem, sw128_desc(a + kk * 2048, LBO, 1024), sw128_desc(b + kk * 2048, LBO, 1024), idesc,
                         (kb | kk) != 0);
            mma_commit(empty0 + 8 * s);
        }
        mma_commit(done);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, tmem_cols(NB));
    }
}

// dW_ref[co][ci*taps + t] = sum_split partial[split][t*C + ci][co]  (fixed split order)
__global__ void k_reduce_dw(const float* __restrict__ partial, int splits, int Mtot, int NB, int taps, int C,
                            int Cout, float* __restrict__ dw) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // over Cout * C * taps (ref order)
    const long long total = (long long)Cout * C * taps;
    if (i >= total) return;
    const int co = (int)(i / (C * taps));
    const int rem = (int)(i % (C * taps));
    const int ci = rem / taps, t = rem % taps;
    const long long m = (long long)t * C + ci;
    float acc = 0.0f;
    for (int s = 0; s < splits; ++s) acc += partial[((long long)s * Mtot + m) * NB + co];
    dw[i] = acc;
}

// ====================================================================== layout helpers
// W_ref[co][ci*taps + t] (fp32, kernel weights layout cnn_ops.hpp:21-27) ->
//   forward:  Wp[co][t*C_in + ci]           (bf16, K padded to Kp with zeros)
//   backward: Wp[ci][t*C_out + co] = W_ref[co][ci*taps + (taps-1-t)]
__global__ void k_pack_w(const float* __restrict__ w, int cout, int cin, int taps, int flip, int Kp,
                         bf16* __restrict__ wp) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int rows = flip ? cin : cout;
    if (i >= (long long)rows * Kp) return;
    const int r = (int)(i / Kp), k = (int)(i % Kp);
    float v = 0.0f;
    if (!flip) {
        if (k < taps * cin) {
            const int t = k / cin, ci = k % cin;
            v = w[(long long)r * cin * taps + ci * taps + t];
        }
    } else {
        if (k < taps * cout) {
            const int t = k / cout, co = k % cout;
            v = w[(long long)co * cin * taps + r * taps + (taps - 1 - t)];
        }
    }
    wp[i] = __float2bfloat16_rn(v);
}

// channel-major fp32 (C x N) -> voxel-major bf16 (N x C), tiled transpose
__global__ void k_to_voxel_major(const float* __restrict__ in, long long C, long long N, bf16* __restrict__ out) {
    __shared__ float tile[32][33];
    const long long n0 = (long long)blockIdx.x * 32, c0 = (long long)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long c = c0 + i, n = n0 + threadIdx.x;
        tile[i][threadIdx.x] = (c < C && n < N) ? in[c * N + n] : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long n = n0 + i, c = c0 + threadIdx.x;
        if (c < C && n < N) out[n * C + c] = __float2bfloat16_rn(tile[threadIdx.x][i]);
    }
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }

// voxel-major (N x C, fp32/bf16) -> channel-major fp32 (C x N)
template <typename T>
__global__ void k_to_channel_major(const T* __restrict__ in, long long N, long long C, float* __restrict__ out) {
    __shared__ float tile[32][33];
    const long long n0 = (long long)blockIdx.x * 32, c0 = (long long)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long n = n0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (c < C && n < N) ? to_f<T>(in[n * C + c]) : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long c = c0 + i, n = n0 + threadIdx.x;
        if (c < C && n < N) out[c * N + n] = tile[threadIdx.x][i];
    }
}

// ====================================================================== launchers
template <int BN, typename OutT>
void launch_gg(const int* nbr, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, OutT* Y,
               cudaStream_t s) {
    auto kern = k_gather_gemm<BN, OutT>;
    const int smem = FwdCfg<BN>::SMEM;
    static bool attr = false;  // per instantiation
    if (!attr) {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
        attr = true;
    }
    kern<<<(unsigned)((rows + BM - 1) / BM), kThreads, smem, s>>>(nbr, taps, rows, X, C, Wp, Kp, Y);
    launched("conv gather-GEMM (tcgen05)");
}

template <typename OutT>
void gather_gemm(const int* nbr, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, int N,
                 OutT* Y, cudaStream_t s) {
    switch (N) {
        case 16: launch_gg<16>(nbr, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 32: launch_gg<32>(nbr, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 64: launch_gg<64>(nbr, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 128: launch_gg<128>(nbr, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 256: launch_gg<256>(nbr, taps, rows, X, C, Wp, Kp, Y, s); break;
        default: throw std::invalid_argument("native conv: output channels must be 16, 32, 64, 128 or 256");
    }
}

int dw_nb(int cout) { return cout <= 64 ? 64 : cout <= 128 ? 128 : 256; }

struct DwPlan {
    int nb, mt, splits, kbps;
    long long partial_floats;
};

DwPlan dw_plan(long long rows, int taps, int cin, int cout) {
    DwPlan p{};
    p.nb = dw_nb(cout);
    p.mt = (taps * cin + BM - 1) / BM;
    const long long total_kb = (rows + 63) / 64;
    int want = std::max(1, (148 * 2 + p.mt - 1) / p.mt);  // ~2 CTAs per SM overall
    want = (int)std::min<long long>(want, std::max<long long>(1, total_kb));
    p.kbps = (int)((total_kb + want - 1) / want);
    p.splits = (int)((total_kb + p.kbps - 1) / p.kbps);
    p.partial_floats = (long long)p.splits * p.mt * BM * p.nb;
    return p;
}

template <int NB>
void launch_dw(const DwPlan& p, const int* nbr, int taps, long long rows, const bf16* X, int C, const bf16* dY,
               int Cout, float* partial, cudaStream_t s) {
    auto kern = k_gather_dw<NB>;
    const int smem = DwCfg<NB>::SMEM;
    static bool attr = false;
    if (!attr) {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr");
        attr = true;
    }
    dim3 g((unsigned)p.mt, (unsigned)p.splits);
    kern<<<g, kThreads, smem, s>>>(nbr, taps, rows, X, C, dY, Cout, p.kbps, partial, p.mt * BM);
    launched("conv dW gather-GEMM (tcgen05)");
}

void check_native(int cin, int cout, int taps) {
    if (cin <= 0 || cin % 8 != 0) throw std::invalid_argument("native conv: input channels must be a multiple of 8");
    if (cout <= 0 || cout % 8 != 0) throw std::invalid_argument("native conv: output channels must be a multiple of 8");
    if (taps < 1 || taps > 27) throw std::invalid_argument("native conv: 1..27 field taps supported");
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

int64_t hc_native_packed_k(int32_t c, int32_t taps) { return ((int64_t)c * taps + 63) / 64 * 64; }

hc_status hc_native_pack_weights(const float* w_ref, int32_t c_out, int32_t c_in, int32_t taps, int32_t backward,
                                 void* w_packed, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        const int rows = backward ? c_in : c_out;
        const long long Kp = hc_native_packed_k(backward ? c_out : c_in, taps);
        const long long n = rows * Kp;
        k_pack_w<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(w_ref, c_out, c_in, taps, backward, (int)Kp,
                                                                   static_cast<bf16*>(w_packed));
        launched("pack weights");
    });
}

hc_status hc_native_gather_gemm(const int32_t* fmap, int64_t n_out, int32_t taps, const void* x, int32_t c_in,
                                const void* w_packed, int32_t c_out, void* y, hc_dtype y_dtype, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (n_out <= 0) return;
        const int Kp = (int)hc_native_packed_k(c_in, taps);
        cudaStream_t s = as_stream(stream);
        if (y_dtype == HC_DTYPE_F32)
            gather_gemm<float>(fmap, taps, n_out, static_cast<const bf16*>(x), c_in, static_cast<const bf16*>(w_packed),
                               Kp, c_out, static_cast<float*>(y), s);
        else
            gather_gemm<bf16>(fmap, taps, n_out, static_cast<const bf16*>(x), c_in, static_cast<const bf16*>(w_packed),
                              Kp, c_out, static_cast<bf16*>(y), s);
    });
}

size_t hc_native_dw_workspace(int64_t n_out, int32_t taps, int32_t c_in, int32_t c_out) {
    const DwPlan p = dw_plan(n_out, taps, c_in, c_out);
    return (size_t)p.partial_floats * sizeof(float);
}

hc_status hc_native_conv_dw(const int32_t* fmap, int64_t n_out, int32_t taps, const void* x, int32_t c_in,
                            const void* dy, int32_t c_out, float* dw_ref, void* workspace, size_t ws_bytes,
                            hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (c_out > 256) throw std::invalid_argument("native conv: dW supports up to 256 output channels");
        cudaStream_t s = as_stream(stream);
        const DwPlan p = dw_plan(n_out, taps, c_in, c_out);
        if (ws_bytes < (size_t)p.partial_floats * sizeof(float))
            throw std::invalid_argument("native conv: dW workspace too small");
        if (n_out <= 0) {
            cuda_check(cudaMemsetAsync(dw_ref, 0, sizeof(float) * c_out * c_in * taps, s), "memset");
            return;
        }
        float* part = static_cast<float*>(workspace);
        const bf16* X = static_cast<const bf16*>(x);
        const bf16* DY = static_cast<const bf16*>(dy);
        switch (p.nb) {
            case 64: launch_dw<64>(p, fmap, taps, n_out, X, c_in, DY, c_out, part, s); break;
            case 128: launch_dw<128>(p, fmap, taps, n_out, X, c_in, DY, c_out, part, s); break;
            default: launch_dw<256>(p, fmap, taps, n_out, X, c_in, DY, c_out, part, s); break;
        }
        const long long total = (long long)c_out * c_in * taps;
        k_reduce_dw<<<grid_for(total, 256), 256, 0, s>>>(part, p.splits, p.mt * BM, p.nb, taps, c_in, c_out, dw_ref);
        launched("dW split reduction");
    });
}

hc_status hc_native_to_voxel_major(const float* ref, int64_t c, int64_t n, void* out, hc_stream stream) {
    return guard([&] {
        if (c <= 0 || n <= 0) return;
        dim3 g((unsigned)((n + 31) / 32), (unsigned)((c + 31) / 32)), b(32, 8);
        k_to_voxel_major<<<g, b, 0, as_stream(stream)>>>(ref, c, n, static_cast<bf16*>(out));
        launched("to voxel-major");
    });
}

hc_status hc_native_to_channel_major(const void* native, hc_dtype dtype, int64_t n, int64_t c, float* out,
                                     hc_stream stream) {
    return guard([&] {
        if (c <= 0 || n <= 0) return;
        dim3 g((unsigned)((n + 31) / 32), (unsigned)((c + 31) / 32)), b(32, 8);
        if (dtype == HC_DTYPE_F32)
            k_to_channel_major<float><<<g, b, 0, as_stream(stream)>>>(static_cast<const float*>(native), n, c, out);
        else
            k_to_channel_major<bf16><<<g, b, 0, as_stream(stream)>>>(static_cast<const bf16*>(native), n, c, out);
        launched("to channel-major");
    });
}

}  // extern "C"
