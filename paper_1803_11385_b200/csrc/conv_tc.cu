// conv_tc.cu — the native (voxel-major) fused hash-conv on 5th-gen tensor cores.
//
// Implicit GEMM: the hash2col column matrix is never materialised. For output
// voxel n and field row t the field map (K0, ops_ref.cu) gives the input column
// nbr(n,t) (or -1); the gathered operand is copied straight from the voxel-major
// feature rows X[nbr][:] into shared memory with 16-byte cp.async (zero-fill for
// empty cells) in the UMMA SWIZZLE_128B canonical form, the dense operand (packed
// weights, or dY for the weight gradient) arrives by 2-D TMA, and tcgen05.mma
// accumulates in TMEM.
//
//   forward        Y [n][co]  = sum_{t,ci} X[nbr(n,t)][ci] * W[co][t][ci]
//   backward-data  dX[g][ci]  = sum_{t,co} dY[nbr(g,t)][co] * W[co][26-t][ci]
//                  (stride 1: the same kernel with flipped/transposed weights;
//                   cnn_ops.cpp:217-232 computes col2hash(W^T dY), the same sum)
//   weight grad    dW[co][t][ci] = sum_n dY[n][co] * X[nbr(n,t)][ci]
//                  (cnn_ops.cpp:228 matmul_trans_b; reduction over voxels: split-K over
//                   CTAs, partials reduced in a fixed order -> deterministic)
//
// Both kernels are persistent and warp-specialised:
//   producers  — warps that issue the gathers; per stage each thread does one shared
//                load of the tile's field-map entry (the map block of a 128-voxel tile is
//                staged by one bulk copy a tile ahead) and one cp.async per 16-byte chunk;
//                the stage completes on the mbarrier when the copies land
//                (cp.async.mbarrier.arrive.noinc), so no producer ever blocks on its own
//                copies. Stage/phase cursors and the (tap, channel) cursor advance
//                incrementally — no divisions on the issue path.
//   TMA        — one thread loads the dense operand of each stage (forward: its own warp).
//   MMA        — one thread issues tcgen05.mma (M128 x N x K16) and commits the stage.
//   epilogue   — one warpgroup drains double-buffered TMEM accumulators (forward).
// Long waits use mbarrier.try_wait with a suspend-time hint, so idle warps sleep
// instead of stealing issue slots from the producers (the round-1 profile showed
// ~30% of all issued instructions were try_wait spins).
//
// Numerics: bf16 operands, fp32 accumulation (TMEM), fp32 or bf16 outputs.
// Tolerance-level parity against the double oracle (tests/test_conv_tc.py).
#include <cuda.h>  // CUtensorMap / enums only; the encoder comes from cudaGetDriverEntryPoint
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "hashconv_b200_native.h"
#include "hc_internal.h"
#include "hc_launch.cuh"
#include "x2_layout.cuh"
#include "tc_common.cuh"
#include "tma_host.h"

namespace hcb {
namespace {

using bf16 = __nv_bfloat16;
using namespace tc;

#ifdef HCB_WAIT_SPIN  // A/B: plain try_wait spins for the long waits too
#define mbar_wait_sleep mbar_wait
#endif
#ifdef HCB_NO_PROXY_FENCE  // A/B only (not a valid memory-model protocol): measures the fence's cost
#define fence_proxy_async() ((void)0)
#endif

constexpr int BM = 128;  // voxels per forward tile (GEMM M) / (t,ci) rows per dW m-tile
constexpr int BK = 64;   // K elements (bf16) per stage = one 128-byte row
constexpr int kMaxTaps = 27;
constexpr int kNbrBytes = kMaxTaps * BM * 4;  // 13.5 KB field-map block per tile

// Split-row layout (x2_layout.cuh: x2_block, x2_pos, split2): a 64-wide K stage holds one plane of
// 64 channels and its hi and lo stages are adjacent (k_conv_fwd_x2 shares their weight tile).

__host__ __device__ constexpr int tmem_cols(int n) {
    return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512;
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "sm count");
    }
    return n;
}

// ---------------------------------------------------------------------- TMA descriptors
EncodeTiled encoder() { return tma_encoder(); }

// 2-D bf16 tensor [rows][inner] (row pitch `pitch` bytes), box = box_rows x 64 elements
// (one 128-byte swizzle span), SWIZZLE_128B, out-of-bounds elements read as zero.
CUtensorMap map2d(const void* base, uint64_t inner, uint64_t rows, uint64_t pitch, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {pitch};
    const cuuint32_t box[2] = {64, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

// Row-major [rows][cols] output for the epilogue's TMA stores: box = box_rows x box_cols
// (16 channels = 32 / 64 bytes: SWIZZLE_32B / 64B staging), rows past `rows` are clipped.
CUtensorMap map_out(const void* base, bool fp32, uint64_t cols, uint64_t rows, uint32_t box_cols, uint32_t box_rows) {
    CUtensorMap m;
    const uint64_t es = fp32 ? 4 : 2;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * es};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t ess[2] = {1, 1};
    const CUresult r = encoder()(&m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                 const_cast<void*>(base), dims, strides, box, ess, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 fp32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled (output) failed (" + std::to_string((int)r) + ")");
    return m;
}

// 16 channels of row r (0..31) -> its 32 (bf16) or 64 (fp32) bytes of the staging box, in the
// TMA SWIZZLE_32B / SWIZZLE_64B layout (16-byte chunk k stored at k ^ (r>>2 & 1) resp.
// k ^ (r>>1 & 3)), so a warp's 16-byte stores spread over all banks (4 wavefronts per
// instruction instead of 8 with plain 32-byte rows).
__device__ __forceinline__ void stage_row16(uint8_t* box, int r, const float (&v)[16], bf16*) {
    uint32_t p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        p[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    uint4* row = reinterpret_cast<uint4*>(box + r * 32);
    const int x = (r >> 2) & 1;
    row[0 ^ x] = make_uint4(p[0], p[1], p[2], p[3]);
    row[1 ^ x] = make_uint4(p[4], p[5], p[6], p[7]);
}
__device__ __forceinline__ void stage_row16(uint8_t* box, int r, const float (&v)[16], float*) {
    float4* row = reinterpret_cast<float4*>(box + r * 64);
    const int x = (r >> 1) & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) row[i ^ x] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}

__device__ __forceinline__ void store_row(float* dst, const float (&v)[16]) {
#pragma unroll
    for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
}


// ---------------------------------------------------------------------- batch-norm statistics
// The forward epilogue can emit, per 128-row tile and output channel, the tile's sum and its
// centred sum of squares (BN statistics from the conv epilogue instead of two
// extra passes over Y; cnn_ops.cpp:455-466 takes the mean and the centred variance in double).
// hc_native_bn_relu_forward_tiles merges the tiles with Chan's parallel formula in double in a
// fixed order, so the result is the two-pass statistic up to fp32 rounding inside a tile.
//
// Sum over a warp's 32 lanes of 16 values per lane in 16 shuffles (recursive halving): after
// the call, lane l holds the total of channel (l >> 1) & 15.
__device__ __forceinline__ float warp_sum16(float (&v)[16], int lane) {
#pragma unroll
    for (int w = 8, off = 16; w >= 1; w >>= 1, off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            const float send = up ? v[i] : v[w + i];
            const float keep = up ? v[w + i] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Tile statistics of one 16-channel chunk: f = this lane's row (rows >= `count` are padding and
// excluded), q = the warp's lane quadrant (rows q*32 ...). red: 2 x [4][16] floats of shared
// memory (buffer `buf` alternates per chunk). Named barrier 1 over the 4 epilogue warps.
__device__ __forceinline__ void tile_stats16(const float (&f)[16], bool valid, int count, int q, int lane, float* red,
                                             float2* out) {
    float v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = valid ? f[e] : 0.0f;
    const int ch = (lane >> 1) & 15;
    float* r1 = red;       // [4][16] warp sums
    float* r2 = red + 64;  // [4][16] warp centred squares
    const float s1 = warp_sum16(v, lane);
    if ((lane & 1) == 0) r1[q * 16 + ch] = s1;
    named_sync(1, 128);
    const float inv = 1.0f / (float)count;
    float tot = 0.0f;  // lane < 16: the tile sum of channel `lane` (read before r1 can be reused)
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const float t = ((r1[e] + r1[16 + e]) + r1[32 + e]) + r1[48 + e];
        if (e == lane) tot = t;
        const float d = f[e] - t * inv;
        v[e] = valid ? d * d : 0.0f;
    }
    const float s2 = warp_sum16(v, lane);
    if ((lane & 1) == 0) r2[q * 16 + ch] = s2;
    named_sync(1, 128);
    // r1 may be overwritten by the next chunk from here on (a warp passes this barrier only after
    // its own reads); r2 is rewritten only after the next chunk's first barrier
    if (q == 0 && lane < 16) out[lane] = make_float2(tot, ((r2[lane] + r2[16 + lane]) + r2[32 + lane]) + r2[48 + lane]);
}

// Per-launch target of the epilogue statistics (hc_native_gather_gemm*_stats set it around
// the launch; the launchers pass it to the kernels): [tiles][c_out] float2 {sum, M2}.
thread_local float2* g_tile_stats = nullptr;
struct TileStatsScope {
    explicit TileStatsScope(float2* p) { g_tile_stats = p; }
    ~TileStatsScope() { g_tile_stats = nullptr; }
};

// ====================================================================== forward gather-GEMM
// Y[m][0:BN] = sum_k A[m][k] * Wp[0:BN][k],  A[m][k] = X[nbr(m, k / C)][k % C] (0 if -1)
// CPS resident CTAs per SM (1: one deep ring; 2: two shallower rings), PW producer warps.
template <int BN, int CPS, int PW, int OUT_BYTES = 2>
struct FwdCfg {
    static constexpr int A_BYTES = BM * 128;  // 16 KB
    static constexpr int B_BYTES = BN * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int NBR = 2 * kNbrBytes;
    // epilogue staging: per epilogue warp EPI_BUFS buffers of 32 rows x 16 channels
    static constexpr int EPI_BUFS = (OUT_BYTES == 2 && BN < 256) ? 2 : 1;  // BN=256 keeps a 4-stage ring
    static constexpr int EPI_BUF = 32 * 16 * OUT_BYTES;
    static constexpr int EPI = 4 * EPI_BUFS * EPI_BUF;
    static constexpr int BUDGET = (CPS == 2 ? 113 : 226) * 1024 - 1024 - 320 - NBR - EPI - 1024;  // - stats scratch
#ifndef HCB_FWD_MAXSTAGES
#define HCB_FWD_MAXSTAGES 10
#endif
    static constexpr int STAGES = BUDGET / STAGE_BYTES > HCB_FWD_MAXSTAGES ? HCB_FWD_MAXSTAGES : BUDGET / STAGE_BYTES;
    static constexpr int PRODUCERS = PW * 32;      // warps 0..PW-1
    static constexpr int THREADS = PW * 32 + 192;  // + epilogue warps PW..PW+3, MMA warp PW+4, TMA warp PW+5
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + NBR + EPI + 320;
};

// SUMH (split-precision forward, hc_native_gather_gemm_x2): the B tile holds two weight planes
// (rows [0, BN/2) = hi, [BN/2, BN) = lo) and the gathered rows two feature planes (K offsets
// [0, C/2) = hi, [C/2, C) = lo of every C-wide row); the epilogue adds the two accumulator halves,
// and K16 chunks of the lo feature plane issue N = BN/2 (the lo x lo product is dropped when
// skip_lolo, leaving hi.hi + hi.lo + lo.hi).
template <int BN, int CPS, int PW, typename OutT, bool SUMH = false>
__global__ void __launch_bounds__(FwdCfg<BN, CPS, PW, sizeof(OutT)>::THREADS, CPS)
    k_conv_fwd(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap ymap,
               const int* __restrict__ fmap, int taps, long long rows, const bf16* __restrict__ X, int C, int nkb,
               int tiles, int skip_lolo /* SUMH: plane block g, 0 = keep lo x lo */, float2* __restrict__ stats) {
    __shared__ float red_s[128];  // epilogue BN statistics scratch (tile_stats16)
    using Cfg = FwdCfg<BN, CPS, PW, sizeof(OutT)>;
    constexpr int NP = Cfg::PRODUCERS;
    constexpr int S = Cfg::STAGES;
    constexpr int RS = NP / 8;  // row stride between one producer thread's rows
    constexpr int J = BM / RS;  // rows per producer thread per stage
    static_assert(BM % RS == 0 && S >= 2, "producer / ring shape");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    int* nbr_s = reinterpret_cast<int*>(smem + S * Cfg::STAGE_BYTES);  // [2][taps][128]
    uint8_t* epi_s = smem + S * Cfg::STAGE_BYTES + Cfg::NBR;           // [4 warps][EPI_BUFS][32][16]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES + Cfg::NBR + Cfg::EPI);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 6);
    int* nbr_cnt = reinterpret_cast<int*>(tmem_slot + 2);  // warps done with each map buffer

    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
    const uint32_t tfull0 = smem_u32(bars + 2 * S), tempty0 = smem_u32(bars + 2 * S + 2);
    const uint32_t nfull0 = smem_u32(bars + 2 * S + 4);
    const uint32_t nbr_bytes = (uint32_t)(taps * BM * 4);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, NP + 1);  // NP cp.async arrivals + the TMA expect_tx arrival
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull0 + 8 * a, 1);
            mbar_init(tempty0 + 8 * a, 128);
            mbar_init(nfull0 + 8 * a, 1);
            nbr_cnt[a] = 0;
        }
        mbar_init_fence();
    }
    if (warp == PW + 4) tmem_alloc(smem_u32(tmem_slot), tmem_cols(2 * BN));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < PW) {
        // ---------------- producers
        // thread (q, c): 16-byte chunk c of the J CONSECUTIVE rows q*J .. q*J+J-1, so its map
        // entries are one or two 16-byte shared loads instead of J scalar ones (a warp's
        // cp.async still covers 4 whole rows: the 4 q of the warp at the same j)
        const int c = tid & 7;
        const int r0 = (tid >> 3) * J;
        static_assert(J % 4 == 0, "map entries are loaded 4 at a time");
        uint32_t doff[J];
#pragma unroll
        for (int j = 0; j < J; ++j) doff[j] = sw128_offset(r0 + j, c);
        const int t0 = (c * 8) / C, ci0 = c * 8 - t0 * C;
        const uint32_t row_bytes = (uint32_t)C * 2;
        auto request = [&](int tile, int buf) {
            mbar_arrive_expect_tx(nfull0 + 8 * buf, nbr_bytes);
            bulk_g2s(smem_u32(nbr_s + buf * kMaxTaps * BM), fmap + (long long)tile * taps * BM, nbr_bytes,
                     nfull0 + 8 * buf);
        };
        if (tid == 0) {
            if (blockIdx.x < tiles) request(blockIdx.x, 0);
            if (blockIdx.x + gridDim.x < tiles) request(blockIdx.x + gridDim.x, 1);
        }
        int s = 0;
        uint32_t ph = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int buf = i & 1;
            mbar_wait_sleep(nfull0 + 8 * buf, (uint32_t)((i >> 1) & 1));
            const uint32_t nb = smem_u32(nbr_s + buf * kMaxTaps * BM + r0);
            int t = t0, ci = ci0;
            for (int kb = 0; kb < nkb; ++kb) {
                // field-map entries first (independent shared loads, batched), then the copies
                int g[J];
                if (t < taps) {  // k = t*C + ci < K
#pragma unroll
                    for (int j = 0; j < J; j += 4) {
                        const int4 v = ld_shared_v4(nb + (t * BM + j) * 4);
                        g[j] = v.x, g[j + 1] = v.y, g[j + 2] = v.z, g[j + 3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < J; ++j) g[j] = -1;
                }
                mbar_wait_sleep(empty0 + 8 * s, ph ^ 1);
                const uint32_t A = sbase + s * Cfg::STAGE_BYTES;
                const char* xs = reinterpret_cast<const char*>(X + ci);
#ifndef HCB_NO_GATHER  // A/B only: the pipeline without the gathers (MMA / issue bound)
#pragma unroll
                for (int j = 0; j < J; ++j) cp_async16_row(A + doff[j], xs, g[j], row_bytes);
#else
                if (g[0] == -12345) cp_async16_row(A + doff[0], xs, g[0], row_bytes);
#endif
                cp_async_arrive_noinc(full0 + 8 * s);
                ci += BK;
                while (ci >= C) {
                    ci -= C;
                    ++t;
                }
                if (++s == S) {
                    s = 0;
                    ph ^= 1;
                }
            }
            // this warp is past the tile's map block; the last warp to get here refills it
            // with tile i+2 (no CTA-wide barrier: producers never wait for each other)
            __syncwarp();
            if ((tid & 31) == 0 && atomicAdd(&nbr_cnt[buf], 1) == PW - 1) {
                nbr_cnt[buf] = 0;
                if (tile + 2 * (int)gridDim.x < tiles) request(tile + 2 * gridDim.x, buf);
            }
        }
    } else if (warp < PW + 4) {
        // ---------------- epilogue warpgroup: TMEM -> registers -> shared staging -> TMA store.
        // Row-per-thread global stores would cost 32 L1 wavefronts per instruction (one line
        // per lane) on the same LSU pipe the gathers need; staged 32 x 16 boxes leave by TMA.
        const int q = warp & 3;  // TMEM lane quadrant of this warp
        const int lane = (int)lane_id();
        uint8_t* stage = epi_s + q * (Cfg::EPI_BUFS * Cfg::EPI_BUF);
        int nb_issued = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int acc = i & 1;
            mbar_wait_sleep(tfull0 + 8 * acc, (uint32_t)((i >> 1) & 1));
            tc_fence_after();
            const int r0 = tile * BM + q * 32;
            constexpr int BO = SUMH ? BN / 2 : BN;  // output channels
#pragma unroll
            for (int c0 = 0; c0 < BO; c0 += 16) {
                uint32_t v[16];
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c0;
                tmem_ld16(ta, v);
                float f[16];
                if constexpr (SUMH) {
                    uint32_t u[16];
                    tmem_ld16(ta + BO, u);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]) + __uint_as_float(u[e]);
                } else {
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]);
                }
                if (stats)  // BN statistics of the fp32 values before the output rounding
                    tile_stats16(f, r0 + lane < rows, (int)min(128LL, rows - (long long)tile * BM), q, lane, red_s,
                                 stats + (long long)tile * BO + c0);
                uint8_t* buf = stage + (nb_issued % Cfg::EPI_BUFS) * Cfg::EPI_BUF;
                if (nb_issued >= Cfg::EPI_BUFS) {  // that buffer's previous store has been read
                    if (lane == 0) bulk_wait_read<Cfg::EPI_BUFS - 1>();
                    __syncwarp();
                }
                stage_row16(buf, lane, f, (OutT*)nullptr);
                fence_proxy_async();  // generic smem writes -> TMA (async proxy) reads
                __syncwarp();
                if (lane == 0) {
                    tma_store2d(&ymap, smem_u32(buf), c0, r0);
                    bulk_commit();
                }
                ++nb_issued;
            }
            tc_fence_before();
            mbar_arrive(tempty0 + 8 * acc);
        }
        if (lane == 0) bulk_wait<0>();  // the last stores complete before the CTA retires
        __syncwarp();
    } else if (tid == (PW + 5) * 32) {
        // ---------------- weight-tile loader (single thread): one 2-D TMA per stage
        int s = 0;
        uint32_t ph = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait_sleep(empty0 + 8 * s, ph ^ 1);
                mbar_arrive_expect_tx(full0 + 8 * s, Cfg::B_BYTES);
                tma_load2d(sbase + s * Cfg::STAGE_BYTES + Cfg::A_BYTES, &wmap, kb * BK, 0, full0 + 8 * s);
                if (++s == S) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == PW + 4) {
        // ---------------- MMA issuer: warp-uniform loop, one elected lane issues
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, false, false);
        constexpr uint32_t idesc_h = idesc_bf16_f32(BM, SUMH ? BN / 2 : BN, false, false);
        const uint64_t a0 = sw128_desc(sbase, 16, 1024), b0 = sw128_desc(sbase + Cfg::A_BYTES, 16, 1024);
        const int g2 = skip_lolo;  // SUMH: plane block g (0: keep lo x lo); row offset kp is lo iff kp % 2g >= g
        int s = 0;
        uint32_t ph = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int acc = i & 1;
            mbar_wait(tempty0 + 8 * acc, (uint32_t)(((i >> 1) & 1) ^ 1));
            tc_fence_after();
            const uint32_t d = tmem + acc * BN;
            int kpos = 0;  // K offset of the stage inside its C-wide row (SUMH)
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(full0 + 8 * s, ph);
                fence_proxy_async();  // cp.async (generic proxy) writes -> tcgen05 operand reads
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t so = (uint64_t)((s * Cfg::STAGE_BYTES) >> 4);  // descriptor start-address units
                    if constexpr (SUMH) {
                        int kp = kpos;  // offset inside the current 2g-wide [hi | lo] block
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk) {
                            const bool lo = g2 && kp >= g2;
                            mma_bf16(d, a0 + so + 2 * kk, b0 + so + 2 * kk, lo ? idesc_h : idesc, (kb | kk) != 0);
                            kp += 16;
                            if (kp >= 2 * g2) kp -= 2 * g2;
                        }
                    } else {
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            mma_bf16(d, a0 + so + 2 * kk, b0 + so + 2 * kk, idesc, (kb | kk) != 0);
                    }
                    mma_commit(empty0 + 8 * s);
                }
                if constexpr (SUMH) {
                    if (g2) {
                        kpos += BK;
                        while (kpos >= 2 * g2) kpos -= 2 * g2;
                    }
                }
                __syncwarp();
                if (++s == S) {
                    s = 0;
                    ph ^= 1;
                }
            }
            if (elect_one()) mma_commit(tfull0 + 8 * acc);
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == PW + 4) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, tmem_cols(2 * BN));
    }
}

// ====================================================================== split-precision forward, shared weight ring
// k_conv_fwd_x2: the SUMH forward for rows interleaved at 64 channels (C_in a multiple of 64:
// row = [hi c0..63 | lo c0..63 | hi c64..127 | lo c64..127 ...]), so every hi stage is followed
// by the lo stage of the same 64 channels, whose weight slice is identical (the packed operand
// repeats it). The weight tiles therefore live in their own ring, one per (hi, lo) pair: half the
// TMA loads and L2 weight traffic of k_conv_fwd<SUMH>, and a weight tile is requested two A
// stages further ahead. NBUF field-map buffers (1 frees 13.5 KB for a deeper A ring).
//   hi stage: D[:, 0:BN] += A_hi . [W_hi; W_lo]^T  (N = BN)      lo stage: D[:, 0:BN/2] += A_lo . W_hi^T
template <int BN, int CPS, int PW, int SA, int SB, int NBUF>
struct FwdX2Cfg {
    static constexpr int A_BYTES = BM * 128;
    static constexpr int B_BYTES = BN * 128;
    static constexpr int NBR = NBUF * kNbrBytes;
    static constexpr int EPI = 4 * 32 * 16 * 4;  // fp32 staging, one 32 x 16 box per epilogue warp
    static constexpr int THREADS = PW * 32 + 192;
    static constexpr int SMEM = 1024 + SA * A_BYTES + SB * B_BYTES + NBR + EPI + 512;
    static_assert(SMEM <= (CPS == 2 ? 113 : 226) * 1024, "shared memory budget");
};

template <int BN, int CPS, int PW, int SA, int SB, int NBUF>
__global__ void __launch_bounds__(FwdX2Cfg<BN, CPS, PW, SA, SB, NBUF>::THREADS, CPS)
    k_conv_fwd_x2(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap ymap,
                  const int* __restrict__ fmap, int taps, const bf16* __restrict__ X, int C, int nkb, int tiles,
                  long long rows, float2* __restrict__ stats) {
    __shared__ float red_s[128];  // epilogue BN statistics scratch (tile_stats16)
    using Cfg = FwdX2Cfg<BN, CPS, PW, SA, SB, NBUF>;
    constexpr int NP = PW * 32;
    constexpr int RS = NP / 8;
    constexpr int J = BM / RS;
    constexpr int BO = BN / 2;  // output channels
    static_assert(BM % RS == 0 && J % 4 == 0 && SA >= 2 && SB >= 1, "producer / ring shape");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bsm = smem + SA * Cfg::A_BYTES;
    int* nbr_s = reinterpret_cast<int*>(bsm + SB * Cfg::B_BYTES);
    uint8_t* epi_s = reinterpret_cast<uint8_t*>(nbr_s) + Cfg::NBR;
    uint64_t* bars = reinterpret_cast<uint64_t*>(epi_s + Cfg::EPI);
    // bars: afull[SA] aempty[SA] bfull[SB] bempty[SB] tfull[2] tempty[2] nfull[NBUF]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * SA + 2 * SB + 4 + NBUF);
    int* nbr_cnt = reinterpret_cast<int*>(tmem_slot + 2);

    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t sbase = smem_u32(smem), bbase = smem_u32(bsm);
    const uint32_t afull0 = smem_u32(bars), aempty0 = smem_u32(bars + SA);
    const uint32_t bfull0 = smem_u32(bars + 2 * SA), bempty0 = smem_u32(bars + 2 * SA + SB);
    const uint32_t tfull0 = smem_u32(bars + 2 * SA + 2 * SB), tempty0 = tfull0 + 16;
    const uint32_t nfull0 = tfull0 + 32;
    const uint32_t nbr_bytes = (uint32_t)(taps * BM * 4);

    if (tid == 0) {
        for (int s = 0; s < SA; ++s) {
            mbar_init(afull0 + 8 * s, NP);
            mbar_init(aempty0 + 8 * s, 1);
        }
        for (int s = 0; s < SB; ++s) {
            mbar_init(bfull0 + 8 * s, 1);
            mbar_init(bempty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull0 + 8 * a, 1);
            mbar_init(tempty0 + 8 * a, 128);
        }
        for (int a = 0; a < NBUF; ++a) {
            mbar_init(nfull0 + 8 * a, 1);
            nbr_cnt[a] = 0;
        }
        mbar_init_fence();
    }
    if (warp == PW + 4) tmem_alloc(smem_u32(tmem_slot), tmem_cols(2 * BN));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < PW && NBUF == 0) {
        // ---------------- producers, map entries straight from global memory (NBUF = 0): each
        // thread loads its J entries of the next tap (2 x 16 bytes, L1-shared by the 8 threads of
        // a row group) one tap ahead, so no shared map block is needed and its 13.5 KB become a
        // fourth A stage
        const int c = tid & 7;
        const int r0 = (tid >> 3) * J;
        uint32_t doff[J];
#pragma unroll
        for (int j = 0; j < J; ++j) doff[j] = sw128_offset(r0 + j, c);
        const uint32_t row_bytes = (uint32_t)C * 2;
        const int spt = C / BK;  // stages per tap (C >= 128: a 64-wide stage never crosses a tap)
        int s = 0;
        uint32_t ph = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const int* mt = fmap + (long long)tile * taps * BM + r0;
            int gn[J];
#pragma unroll
            for (int j = 0; j < J; j += 4) {
                const int4 v = __ldg(reinterpret_cast<const int4*>(mt + j));
                gn[j] = v.x, gn[j + 1] = v.y, gn[j + 2] = v.z, gn[j + 3] = v.w;
            }
            for (int t = 0; t < taps; ++t) {
                int g[J];
#pragma unroll
                for (int j = 0; j < J; ++j) g[j] = gn[j];
                if (t + 1 < taps) {
#pragma unroll
                    for (int j = 0; j < J; j += 4) {
                        const int4 v = __ldg(reinterpret_cast<const int4*>(mt + (t + 1) * BM + j));
                        gn[j] = v.x, gn[j + 1] = v.y, gn[j + 2] = v.z, gn[j + 3] = v.w;
                    }
                }
                for (int k = 0; k < spt; ++k) {
                    mbar_wait_sleep(aempty0 + 8 * s, ph ^ 1);
                    const uint32_t A = sbase + s * Cfg::A_BYTES;
                    const char* xs = reinterpret_cast<const char*>(X + k * BK + c * 8);
#pragma unroll
                    for (int j = 0; j < J; ++j) cp_async16_row(A + doff[j], xs, g[j], row_bytes);
                    cp_async_arrive_noinc(afull0 + 8 * s);
                    if (++s == SA) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp < PW) {
        // ---------------- producers (as k_conv_fwd: J consecutive rows x one 16-byte chunk)
        const int c = tid & 7;
        const int r0 = (tid >> 3) * J;
        uint32_t doff[J];
#pragma unroll
        for (int j = 0; j < J; ++j) doff[j] = sw128_offset(r0 + j, c);
        const uint32_t row_bytes = (uint32_t)C * 2;
        auto request = [&](int tile, int buf) {
            mbar_arrive_expect_tx(nfull0 + 8 * buf, nbr_bytes);
            bulk_g2s(smem_u32(nbr_s + buf * kMaxTaps * BM), fmap + (long long)tile * taps * BM, nbr_bytes,
                     nfull0 + 8 * buf);
        };
        if (tid == 0)
            for (int b = 0; b < NBUF; ++b)
                if (blockIdx.x + b * gridDim.x < tiles) request(blockIdx.x + b * gridDim.x, b);
        int s = 0;
        uint32_t ph = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            constexpr int NB1 = NBUF > 0 ? NBUF : 1;  // (this branch runs only with NBUF > 0)
            const int buf = NB1 == 1 ? 0 : i % NB1;
            mbar_wait_sleep(nfull0 + 8 * buf, (uint32_t)((i / NB1) & 1));
            const uint32_t nb = smem_u32(nbr_s + buf * kMaxTaps * BM + r0);
            int t = 0, ci = c * 8;  // C >= 128: a 64-wide stage never crosses a tap
            for (int kb = 0; kb < nkb; ++kb) {
                int g[J];
                if (t < taps) {
#pragma unroll
                    for (int j = 0; j < J; j += 4) {
                        const int4 v = ld_shared_v4(nb + (t * BM + j) * 4);
                        g[j] = v.x, g[j + 1] = v.y, g[j + 2] = v.z, g[j + 3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < J; ++j) g[j] = -1;
                }
                mbar_wait_sleep(aempty0 + 8 * s, ph ^ 1);
                const uint32_t A = sbase + s * Cfg::A_BYTES;
                const char* xs = reinterpret_cast<const char*>(X + ci);
#ifndef HCB_NO_GATHER
#pragma unroll
                for (int j = 0; j < J; ++j) cp_async16_row(A + doff[j], xs, g[j], row_bytes);
#else
                if (g[0] == -12345) cp_async16_row(A + doff[0], xs, g[0], row_bytes);
#endif
                cp_async_arrive_noinc(afull0 + 8 * s);
                ci += BK;
                if (ci >= C) {
                    ci -= C;
                    ++t;
                }
                if (++s == SA) {
                    s = 0;
                    ph ^= 1;
                }
            }
            __syncwarp();
            if ((tid & 31) == 0 && atomicAdd(&nbr_cnt[buf], 1) == PW - 1) {
                nbr_cnt[buf] = 0;
                if (tile + NBUF * (int)gridDim.x < tiles) request(tile + NBUF * gridDim.x, buf);
            }
        }
    } else if (warp < PW + 4) {
        // ---------------- epilogue: D[:, co] + D[:, BO + co] -> fp32 -> staging -> TMA store
        const int q = warp & 3;
        const int lane = (int)lane_id();
        uint8_t* stage = epi_s + q * (32 * 16 * 4);
        int i = 0, issued = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int acc = i & 1;
            mbar_wait_sleep(tfull0 + 8 * acc, (uint32_t)((i >> 1) & 1));
            tc_fence_after();
            const int r0 = tile * BM + q * 32;
#pragma unroll
            for (int c0 = 0; c0 < BO; c0 += 16) {
                uint32_t v[16], u[16];
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c0;
                tmem_ld16(ta, v);
                tmem_ld16(ta + BO, u);
                tmem_ld_wait();
                float f[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]) + __uint_as_float(u[e]);
                if (stats)
                    tile_stats16(f, r0 + lane < rows, (int)min(128LL, rows - (long long)tile * BM), q, lane, red_s,
                                 stats + (long long)tile * BO + c0);
                if (issued) {  // the staging box's previous store has been read
                    if (lane == 0) bulk_wait_read<0>();
                    __syncwarp();
                }
                stage_row16(stage, lane, f, (float*)nullptr);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    tma_store2d(&ymap, smem_u32(stage), c0, r0);
                    bulk_commit();
                }
                issued = 1;
            }
            tc_fence_before();
            mbar_arrive(tempty0 + 8 * acc);
        }
        if (lane == 0) bulk_wait<0>();
        __syncwarp();
    } else if (tid == (PW + 5) * 32) {
        // ---------------- weight loader: one [W_hi; W_lo] tile per (hi, lo) stage pair
        int s = 0;
        uint32_t ph = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            for (int kb = 0; kb < nkb; kb += 2) {
                mbar_wait_sleep(bempty0 + 8 * s, ph ^ 1);
#ifdef HCB_NO_BLOAD  // A/B only (wrong results): weight tiles loaded once, then reused
                if (tile != (int)blockIdx.x || kb >= 2 * SB) { mbar_arrive(bfull0 + 8 * s); goto next_w; }
#endif
                mbar_arrive_expect_tx(bfull0 + 8 * s, Cfg::B_BYTES);
                tma_load2d(bbase + s * Cfg::B_BYTES, &wmap, kb * BK, 0, bfull0 + 8 * s);
#ifdef HCB_NO_BLOAD
            next_w:
#endif
                if (++s == SB) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == PW + 4) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, false, false);
        constexpr uint32_t idesc_h = idesc_bf16_f32(BM, BO, false, false);
        const uint64_t a0 = sw128_desc(sbase, 16, 1024), b0 = sw128_desc(bbase, 16, 1024);
        int sa = 0, sb = 0;
        uint32_t pha = 0, phb = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int acc = i & 1;
            mbar_wait(tempty0 + 8 * acc, (uint32_t)(((i >> 1) & 1) ^ 1));
            tc_fence_after();
            const uint32_t d = tmem + acc * BN;
            for (int kb = 0; kb < nkb; kb += 2) {
                mbar_wait(bfull0 + 8 * sb, phb);
                const uint64_t bo = (uint64_t)((sb * Cfg::B_BYTES) >> 4);
#pragma unroll
                for (int half = 0; half < 2; ++half) {  // hi stage (N = BN), then lo stage (N = BN/2)
                    mbar_wait(afull0 + 8 * sa, pha);
                    fence_proxy_async();
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t ao = (uint64_t)((sa * Cfg::A_BYTES) >> 4);
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            mma_bf16(d, a0 + ao + 2 * kk, b0 + bo + 2 * kk, half ? idesc_h : idesc,
                                     (kb | half | kk) != 0);
                        mma_commit(aempty0 + 8 * sa);
                        if (half) mma_commit(bempty0 + 8 * sb);
                    }
                    __syncwarp();
                    if (++sa == SA) {
                        sa = 0;
                        pha ^= 1;
                    }
                }
                if (++sb == SB) {
                    sb = 0;
                    phb ^= 1;
                }
            }
            if (elect_one()) mma_commit(tfull0 + 8 * acc);
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == PW + 4) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, tmem_cols(2 * BN));
    }
}

// ====================================================================== weight gradient
// Partial[split][m][co] = sum over this split's voxels n of A[m][n] * B[co][n]
//   A[m][n] = X[nbr(n, m / C)][m % C]   (m = t*C + ci; MN-major: one 128-byte gathered row
//                                        per voxel and 64-wide MN block)
//   B[co][n] = dY[n][co]                 (MN-major; 2-D TMA of 64 voxel rows per block,
//                                        C_out < 64 zero-filled out of bounds)
// Grid = CTA slots of the SM count (DwGroups): a group owns up to 512/(NB*CPS) m-tiles whose
// fp32 accumulators (NB TMEM columns each) stay resident for the CTA's whole voxel range,
// so each dY stage is loaded once and feeds all of them (the previous one-m-tile-per-
// CTA plan re-read dY mt = 14 times at C=64).
// Split plan, passed by value: group g owns m-tiles [m_begin[g], m_begin[g+1]) and CTAs
// [cta_begin[g], cta_begin[g+1]). Its voxel range is cut into nchunk[g] chunks of tps[g] voxel
// tiles; CTA k of the group runs chunks [k*cpc[g], (k+1)*cpc[g]) back to back, draining its
// TMEM accumulators into one partial slot per chunk (a chunk is one accumulation chain: the
// split-precision path bounds it to keep the tensor core's fp32 accumulation within 1e-5).
//   tri (split precision, c_out >= 32, default): units of 128 (t, ci) rows; the hi-plane m-tile
//     multiplies [dY_hi | dY_lo] (N = 2 c_out), the lo-plane m-tile dY_hi only (N = c_out), so the
//     negligible lo.lo product is never computed (3 products instead of 4); each epilogue lane sums
//     its own row, rpm = 128 rows x c_out. For 32 < c_out <= 64 (tshared) the lo-plane m-tile
//     accumulates into the hi.dY_hi columns — 2 c_out TMEM columns per unit, two units per CTA,
//     half the dY loads — and the lane sums (hi.dY_hi + lo.dY_hi) + hi.dY_lo; otherwise lo.dY_hi
//     keeps its own c_out columns and the sum is (hi.dY_hi + hi.dY_lo) + lo.dY_hi.
// Partials start at part_begin[g] (floats), laid out [chunk][m-tile][rpm][pcols]:
//   plain: rpm = 128 (t,ci) rows of the row width C, pcols = NB.
//   pair (split precision, hc_native_conv_dw_x2): X rows are [hi | lo] (C = 2 c), dY rows
//     [hi | lo] (2 c_out); m-tile j's 64-row blocks are the hi and the lo plane of the same 64
//     (t, ci) rows j*64 .. j*64+63 of taps x c, so the epilogue adds the four plane products
//     (lanes r and 64 + r, columns co and c_out + co) and writes rpm = 64 rows x c_out.
constexpr int kMaxGroups = 64;
struct DwGroups {
    int groups;
    int pair, rpm, pcols;
    int nacc;  // accumulator buffers per CTA (2: chunk drains overlap the next chunk's MMAs)
    int shift[kMaxGroups];  // chunk c of group g covers tiles [c*tps - shift, (c+1)*tps - shift) (clipped):
                            // groups alternate between 0 and tps/2, so the two CTAs an SM holds (of
                            // different groups) drain their accumulators at different times
    int tshared;  // tri: the lo-plane m-tile accumulates into the hi.dY_hi columns (c_out <= 64)
    int strided;  // 1: CTA k of a group runs chunks k, k + n, k + 2n ... (n = the group's CTAs), so
                  // the whole grid sweeps the voxels together and the groups' gathers of X and
                  // loads of dY hit L2; 0: contiguous runs of cpc chunks
    int m_begin[kMaxGroups + 1];
    int cta_begin[kMaxGroups + 1];
    int tps[kMaxGroups];
    int nchunk[kMaxGroups];
    int cpc[kMaxGroups];
    long long part_begin[kMaxGroups];
};

// NT = field-map taps one buffer holds: a CTA stages only the taps its m-tiles touch
// (C=64, 4 m-tiles: 9 of 27), which leaves shared memory for a deeper A ring.
template <int NB, int PW, int CPS = 1, int NT = kMaxTaps>
struct DwCfg {
    static constexpr int KB = 64;                      // voxels per stage
    static constexpr int A_BYTES = 2 * KB * 128;       // two 64-wide MN blocks (M = 128)
    static constexpr int B_BYTES = (NB / 64) * KB * 128;
#ifndef HCB_DW_BSTAGES
#define HCB_DW_BSTAGES 2
#endif
    static constexpr int BSTAGES = HCB_DW_BSTAGES;
    static constexpr int NBR = 2 * NT * BM * 4;
    static constexpr int XCH = 64 * 20 * 4;  // pair-mode epilogue exchange: 64 rows x 16 (+4 pad) floats
    static constexpr int BUDGET = (CPS == 2 ? 113 : 226) * 1024 - 1024 - 512 - 1024 - NBR - BSTAGES * B_BYTES - XCH;
    static constexpr int STAGES = BUDGET / A_BYTES > 10 ? 10 : BUDGET / A_BYTES;
    static constexpr int PRODUCERS = PW * 32;
    // + MMA / TMEM warp PW, dY TMA warp PW+1, epilogue warps PW+2 .. PW+5 (TMEM lane quadrants)
    static constexpr int THREADS = PRODUCERS + 64 + 128;
    static constexpr int TMEM_COLS = 512 / CPS;  // per CTA (CPS resident CTAs per SM)
    static constexpr int SMEM = 1024 + STAGES * A_BYTES + BSTAGES * B_BYTES + NBR + XCH + 1024 + 512;
};

template <int NB, int PW, int CPS, int NT>
__global__ void __launch_bounds__(DwCfg<NB, PW, CPS, NT>::THREADS, CPS)
    k_conv_dw(const __grid_constant__ CUtensorMap dymap, const int* __restrict__ fmap, int taps, long long rows,
              const bf16* __restrict__ X, int C, const DwGroups grp_tab, int tiles, float* __restrict__ partial) {
    using Cfg = DwCfg<NB, PW, CPS, NT>;
    constexpr int S = Cfg::STAGES, BS = Cfg::BSTAGES;
    constexpr int NP = Cfg::PRODUCERS;
    constexpr int RS = NP / 8;
    constexpr int J = 128 / RS;  // rows (of 128 = 2 blocks x 64 voxels) per thread per stage
    static_assert(128 % RS == 0 && RS <= 64, "producer shape");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bsm = smem + S * Cfg::A_BYTES;
    int* nbr_s = reinterpret_cast<int*>(bsm + BS * Cfg::B_BYTES);
    float* xch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(nbr_s) + Cfg::NBR);
    int* tab = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(xch) + Cfg::XCH);  // [m-tile][2 blocks][8 chunks]
    uint64_t* bars = reinterpret_cast<uint64_t*>(tab + 256);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 2 * BS + 6);
    int* nbr_cnt = reinterpret_cast<int*>(tmem_slot + 2);

    const int tid = threadIdx.x, warp = tid >> 5;
    int grp = 0;  // this CTA's m-tile group, and its run of chunks inside the group
    while (grp + 1 < grp_tab.groups && (int)blockIdx.x >= grp_tab.cta_begin[grp + 1]) ++grp;
    const int m0 = grp_tab.m_begin[grp];
    const int nm = grp_tab.m_begin[grp + 1] - m0;
    const int tps = grp_tab.tps[grp];
    const int kcta = (int)blockIdx.x - grp_tab.cta_begin[grp];
    const int nct = grp_tab.cta_begin[grp + 1] - grp_tab.cta_begin[grp];
    const int nchunk = grp_tab.nchunk[grp];
    const int chunk0 = grp_tab.strided ? kcta : kcta * grp_tab.cpc[grp];
    const int cstride = grp_tab.strided ? nct : 1;
    const int nch = grp_tab.strided ? (kcta < nchunk ? (nchunk - kcta + nct - 1) / nct : 0)
                                    : max(0, min(grp_tab.cpc[grp], nchunk - chunk0));
    // this CTA's chunks are chunk0 + j * cstride; chunk c covers [c*tps - sh, (c+1)*tps - sh) within
    // [0, tiles): all hold tps tiles but the group's first (tps - sh) and last ones
    const int sh = grp_tab.shift[grp];
    auto cstart = [&](int c) { return max(0, c * tps - sh); };
    auto cend = [&](int c) { return min(tiles, (c + 1) * tps - sh); };
    const int len0 = nch > 0 ? cend(chunk0) - cstart(chunk0) : 0;  // this CTA's first chunk
    const int ntl = nch == 0 ? 0 : nch == 1 ? len0
                  : len0 + (nch - 2) * tps + (cend(chunk0 + (nch - 1) * cstride) - cstart(chunk0 + (nch - 1) * cstride));
    auto tile_of = [&](int lt) {
        if (lt < len0) return cstart(chunk0) + lt;
        const int r = lt - len0;
        return cstart(chunk0 + (1 + r / tps) * cstride) + r % tps;
    };
    const int pair = grp_tab.pair;    // 0 plain, 1 pair (split precision, 4 products), 2 tri (3 products)
    const int Co = pair ? C / 2 : C;  // channels of one plane
    const int RPM = pair == 1 ? 64 : 128;  // (t, ci) rows per m-tile (tri: per unit)
    const int nmt = pair == 2 ? 2 * nm : nm;  // m-tiles the producers fill / the MMA consumes per stage
    const int pco = grp_tab.pcols;             // tri: c_out (one plane)
    const int K = taps * Co;
    const uint32_t sbase = smem_u32(smem), bbase = smem_u32(bsm);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
    const uint32_t bfull0 = smem_u32(bars + 2 * S), bempty0 = smem_u32(bars + 2 * S + BS);
    // done[b] / drained[b]: accumulator buffer b (nacc = 2: chunk c uses buffer c & 1, so the epilogue
    // drains one chunk while the MMA accumulates the next)
    const uint32_t nfull0 = smem_u32(bars + 2 * S + 2 * BS), done0 = nfull0 + 16, drained0 = nfull0 + 32;
    const int nacc = grp_tab.nacc;
    // taps [t_lo, t_lo + ntb) cover this CTA's (t, ci) rows; only they are staged
    const int t_lo = (m0 * RPM) / Co;
    const int ntb = min(NT, (min(K, (m0 + nm) * RPM) - 1) / Co - t_lo + 1);
    const uint32_t nbr_bytes = (uint32_t)(ntb * BM * 4);

    for (int e = tid; e < nmt * 16; e += blockDim.x) {
        const int blk = (e / 8) & 1;
        int m, plane;
        if (pair == 2) {  // m-tile 2u = hi plane, 2u + 1 = lo plane of unit u's 128 rows
            m = (m0 + e / 32) * 128 + blk * 64 + (e & 7) * 8;
            plane = (e / 16) & 1;
        } else if (pair == 1) {
            m = (m0 + e / 16) * 64 + (e & 7) * 8;
            plane = blk;
        } else {
            m = (m0 + e / 16) * 128 + blk * 64 + (e & 7) * 8;
            plane = 0;
        }
        tab[e] = m < K ? ((m / Co - t_lo) << 16) | (pair ? x2_pos(m % Co, plane, x2_block(Co)) : m % Co) : -1;
    }
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, NP);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int s = 0; s < BS; ++s) {
            mbar_init(bfull0 + 8 * s, 1);
            mbar_init(bempty0 + 8 * s, 1);
        }
        mbar_init(nfull0, 1);
        mbar_init(nfull0 + 8, 1);
        nbr_cnt[0] = nbr_cnt[1] = 0;
        for (int b = 0; b < 2; ++b) {
            mbar_init(done0 + 8 * b, 1);
            mbar_init(drained0 + 8 * b, 128);
        }
        mbar_init_fence();
    }
    if (warp == PW) tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < PW) {
        // ---------------- producers
        const int c = tid & 7;
        // thread (q, c): chunk c of the J consecutive rows q*J .. q*J+J-1 of the stage's 128
        // (block, voxel) rows — all in one 64-wide MN block, so one (tap, channel) entry per
        // stage and the J map entries as 16-byte shared loads
        const int q = tid >> 3;
        static_assert(J % 4 == 0 && 64 % J == 0, "rows of a thread stay in one MN block");
        const int blk = (q * J) >> 6, v0 = (q * J) & 63;
        const uint32_t row_bytes = (uint32_t)C * 2;
        const uint32_t tab_s = smem_u32(tab) + (blk * 8 + c) * 4;
        uint32_t doff[J];
#pragma unroll
        for (int j = 0; j < J; ++j) doff[j] = blk * (Cfg::KB * 128) + sw128_offset(v0 + j, c);
        auto request = [&](int lt, int buf) {
            mbar_arrive_expect_tx(nfull0 + 8 * buf, nbr_bytes);
            bulk_g2s(smem_u32(nbr_s + buf * NT * BM), fmap + ((long long)tile_of(lt) * taps + t_lo) * BM, nbr_bytes,
                     nfull0 + 8 * buf);
        };
        if (tid == 0) {
            if (ntl > 0) request(0, 0);
            if (ntl > 1) request(1, 1);
        }
        int s = 0;
        uint32_t ph = 0;
        for (int lt = 0; lt < ntl; ++lt) {
            const int buf = lt & 1;
            mbar_wait_sleep(nfull0 + 8 * buf, (uint32_t)((lt >> 1) & 1));
            const uint32_t nb = smem_u32(nbr_s + buf * NT * BM);
            for (int h = 0; h < 2; ++h) {
                const uint32_t nbh = nb + h * 64 * 4;
                for (int mi = 0; mi < nmt; ++mi) {
                    const int e = ld_shared_s32(tab_s + mi * 64);
                    int g[J];
                    if (e >= 0) {
#pragma unroll
                        for (int j = 0; j < J; j += 4) {
                            const int4 w = ld_shared_v4(nbh + ((e >> 16) * BM + v0 + j) * 4);
                            g[j] = w.x, g[j + 1] = w.y, g[j + 2] = w.z, g[j + 3] = w.w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < J; ++j) g[j] = -1;
                    }
                    mbar_wait_sleep(empty0 + 8 * s, ph ^ 1);
                    const uint32_t A = sbase + s * Cfg::A_BYTES;
                    const char* xs = reinterpret_cast<const char*>(X + (e & 0xffff));
#ifndef HCB_NO_GATHER
#pragma unroll
                    for (int j = 0; j < J; ++j) cp_async16_row(A + doff[j], xs, g[j], row_bytes);
#else
                    if (g[0] == -12345) cp_async16_row(A + doff[0], xs, g[0], row_bytes);
#endif
                    cp_async_arrive_noinc(full0 + 8 * s);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
            __syncwarp();
            if ((tid & 31) == 0 && atomicAdd(&nbr_cnt[buf], 1) == PW - 1) {
                nbr_cnt[buf] = 0;
                if (lt + 2 < ntl) request(lt + 2, buf);
            }
        }
    } else if (tid == (PW + 1) * 32) {
        // ---------------- dY loader (own warp: a producer thread blocking on the B ring
        // would stall its A rows and with them every stage)
        int bs = 0;
        uint32_t bph = 0;
        for (int lt = 0; lt < ntl; ++lt)
            for (int h = 0; h < 2; ++h) {
                mbar_wait_sleep(bempty0 + 8 * bs, bph ^ 1);
#ifdef HCB_NO_BLOAD  // A/B only (wrong results): dY tiles loaded once, then reused
                if (lt >= 1) { mbar_arrive(bfull0 + 8 * bs); goto next_b; }
#endif
                {
                mbar_arrive_expect_tx(bfull0 + 8 * bs, Cfg::B_BYTES);
                const int n0 = tile_of(lt) * BM + h * 64;
#pragma unroll
                for (int cb = 0; cb < NB / 64; ++cb)
                    tma_load2d(bbase + bs * Cfg::B_BYTES + cb * (Cfg::KB * 128), &dymap, cb * 64, n0,
                               bfull0 + 8 * bs);
                }
#ifdef HCB_NO_BLOAD
            next_b:
#endif
                if (++bs == BS) {
                    bs = 0;
                    bph ^= 1;
                }
            }
    } else if (warp == PW && ntl > 0) {
        // ---------------- MMA issuer: warp-uniform loop, one elected lane issues. Each chunk
        // starts a fresh accumulation (after the epilogue drained the previous chunk) and
        // ends with a commit to `done`.
        constexpr uint32_t idesc = idesc_bf16_f32(BM, NB, true, true);
        constexpr uint32_t LBO = Cfg::KB * 128;  // next 64-wide MN block
        const uint64_t a0 = sw128_desc(sbase, LBO, 1024), b0 = sw128_desc(bbase, LBO, 1024);
        // tri: the lo m-tile multiplies dY_hi only (N = c_out); with c_out >= 128 the dY tile's
        // 64-wide blocks alternate hi / lo, so its hi blocks are two blocks apart
        const uint32_t idesc_lo = pair == 2 ? idesc_bf16_f32(BM, pco, true, true) : idesc;
        const uint32_t idesc_hi = pair == 2 ? idesc_bf16_f32(BM, 2 * pco, true, true) : idesc;  // [dY_hi | dY_lo]
        const uint64_t b0_lo = sw128_desc(bbase, pco >= 128 ? 2 * LBO : LBO, 1024);
        // tri: c_out <= 64 -> the lo-plane m-tile accumulates into the hi.dY_hi columns (its D columns are the
        // hi channels 0 .. c_out - 1, the first half of the [dY_hi | dY_lo] row), 2 c_out columns per unit;
        // wider: dY_hi's 64-blocks are not contiguous there, so lo.dY_hi keeps its own c_out columns
        const bool tshared = pair == 2 && grp_tab.tshared;
        const int ucols = pair == 2 ? (tshared ? 2 * pco : 3 * pco) : NB;  // accumulator columns per m-tile / unit
        int s = 0, bs = 0;
        uint32_t ph = 0, bph = 0;
        int cl = 0, ci = 0;  // tile index inside the chunk, chunk index
        int clen = len0;     // tiles of the current chunk
        for (int lt = 0; lt < ntl; ++lt) {
            const int ab = nacc == 2 ? (ci & 1) : 0;  // accumulator buffer of this chunk
            if (cl == 0 && ci >= nacc) {                 // its previous chunk has been drained
                const int prev = ci - nacc;
                mbar_wait(drained0 + 8 * ab, (uint32_t)((nacc == 2 ? prev >> 1 : prev) & 1));
                tc_fence_after();
            }
            const uint32_t acc0 = tmem + ab * nm * ucols;
            for (int h = 0; h < 2; ++h) {
                mbar_wait(bfull0 + 8 * bs, bph);
                const uint64_t bo = (uint64_t)((bs * Cfg::B_BYTES) >> 4);
                for (int mi = 0; mi < nmt; ++mi) {
                    mbar_wait(full0 + 8 * s, ph);
                    fence_proxy_async();
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t ao = (uint64_t)((s * Cfg::A_BYTES) >> 4);
                        const bool lo = pair == 2 && (mi & 1);
                        const uint32_t d = pair == 2 ? acc0 + (mi >> 1) * ucols + (lo && !tshared ? 2 * pco : 0)
                                                     : acc0 + mi * NB;
                        const uint64_t bd = (lo ? b0_lo : b0) + bo;
                        const uint32_t id = lo ? idesc_lo : idesc_hi;
                        // a shared lo accumulator (tshared) always adds: the unit's hi m-tile stage, issued
                        // first, zero-initialises those columns at the chunk's first K step
                        const bool first = (cl | h) == 0 && !(lo && tshared);
#pragma unroll
                        for (int kk = 0; kk < Cfg::KB / 16; ++kk)  // 16 voxels = two 8-row atoms per MMA
                            mma_bf16(d, a0 + ao + 128 * kk, bd + 128 * kk, id, !(first && kk == 0));
                        mma_commit(empty0 + 8 * s);
                    }
                    __syncwarp();
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (elect_one()) mma_commit(bempty0 + 8 * bs);
                __syncwarp();
                if (++bs == BS) {
                    bs = 0;
                    bph ^= 1;
                }
            }
            if (++cl == clen || lt == ntl - 1) {
                if (elect_one()) mma_commit(done0 + 8 * ab);
                __syncwarp();
                cl = 0;
                ++ci;
                const int c = chunk0 + ci * cstride;
                clen = cend(c) - cstart(c);
            }
        }
    } else if (warp >= PW + 2) {
        // ---------------- epilogue warps: TMEM lane quadrant q = warp & 3, row = q*32 + lane.
        const int q = warp & 3;
        const int row = q * 32 + (int)lane_id();
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
        for (int c = 0; c < nch; ++c) {
            const int ab = nacc == 2 ? (c & 1) : 0;
            mbar_wait_sleep(done0 + 8 * ab, (uint32_t)((nacc == 2 ? c >> 1 : c) & 1));
            const bool tsh = pair == 2 && grp_tab.tshared;  // as the MMA issuer's tshared
            const int uc = pair == 2 ? (tsh ? 2 * pco : 3 * pco) : NB;
            const uint32_t tqa = tq + ab * nm * uc;
            tc_fence_after();
            const long long slot = chunk0 + (long long)c * cstride;
            if (pair == 2) {
                // tri: lane = (t, ci) row of the unit; fixed order (hi.dY_hi + hi.dY_lo) + lo.dY_hi
                const int g = x2_block(pco);
                for (int u = 0; u < nm; ++u) {
                    float* dst = partial + grp_tab.part_begin[grp] + ((slot * nm + u) * BM + row) * pco;
                    const uint32_t tu = tqa + u * uc;
                    for (int c0 = 0; c0 < pco; c0 += 16) {
                        uint32_t a[16], b[16], l[16];
                        tmem_ld16(tu + x2_pos(c0, 0, g), a);
                        tmem_ld16(tu + x2_pos(c0, 1, g), b);
                        if (!tsh) tmem_ld16(tu + 2 * pco + c0, l);
                        tmem_ld_wait();
                        float f[16];
                        if (tsh) {  // (hi.dY_hi + lo.dY_hi) + hi.dY_lo
#pragma unroll
                            for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(a[e]) + __uint_as_float(b[e]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                f[e] = (__uint_as_float(a[e]) + __uint_as_float(b[e])) + __uint_as_float(l[e]);
                        }
                        store_row(dst + c0, f);
                    }
                }
            } else if (pair) {
                // lanes 64..127 (lo plane rows) hand their column sums to lanes 0..63 through a
                // 64 x 16 shared exchange; fixed order (hi.hi + hi.lo) + (lo.hi + lo.lo)
                const int r = row & 63;
                const int pc = grp_tab.pcols;  // c_out (a multiple of 16)
                float* x = xch + r * 20;
                for (int mi = 0; mi < nm; ++mi) {
                    float* dst = partial + grp_tab.part_begin[grp] + ((slot * nm + mi) * 64 + r) * pc;
                    for (int c0 = 0; c0 < pc; c0 += 16) {
                        uint32_t a[16], b[16];  // dY planes interleave like X's (x2_pos)
                        tmem_ld16(tqa + mi * NB + x2_pos(c0, 0, x2_block(pc)), a);
                        tmem_ld16(tqa + mi * NB + x2_pos(c0, 1, x2_block(pc)), b);
                        tmem_ld_wait();
                        float f[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(a[e]) + __uint_as_float(b[e]);
                        if (row >= 64) {
#pragma unroll
                            for (int e = 0; e < 16; e += 4)
                                *reinterpret_cast<float4*>(x + e) = make_float4(f[e], f[e + 1], f[e + 2], f[e + 3]);
                        }
                        named_sync(1, 128);
                        if (row < 64) {
#pragma unroll
                            for (int e = 0; e < 16; e += 4) {
                                const float4 v = *reinterpret_cast<const float4*>(x + e);
                                f[e] += v.x, f[e + 1] += v.y, f[e + 2] += v.z, f[e + 3] += v.w;
                            }
                            store_row(dst + c0, f);
                        }
                        named_sync(1, 128);
                    }
                }
            } else {
                for (int mi = 0; mi < nm; ++mi) {
                    float* dst = partial + grp_tab.part_begin[grp] + ((slot * nm + mi) * BM + row) * NB;
#pragma unroll
                    for (int c0 = 0; c0 < NB; c0 += 16) {
                        uint32_t v[16];
                        tmem_ld16(tqa + mi * NB + c0, v);
                        tmem_ld_wait();
                        float f[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]);
                        store_row(dst + c0, f);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(drained0 + 8 * ab);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == PW) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, Cfg::TMEM_COLS);
    }
}

// Sum over the voxel splits of one (m, n) partial: lane j of 8 takes splits j, j+8, ...
__device__ __forceinline__ float split_lane_sum(const float* __restrict__ partial, const DwGroups& grp_tab,
                                                long long m, int n, int j) {
    const int rpm = grp_tab.rpm, pc = grp_tab.pcols;
    const int mtile = (int)(m / rpm), row = (int)(m % rpm);
    int g = 0;
    while (g + 1 < grp_tab.groups && mtile >= grp_tab.m_begin[g + 1]) ++g;
    const int nm = grp_tab.m_begin[g + 1] - grp_tab.m_begin[g];
    const int splits = grp_tab.nchunk[g];
    const float* p = partial + grp_tab.part_begin[g] + ((long long)(mtile - grp_tab.m_begin[g]) * rpm + row) * pc + n;
    const long long stride = (long long)nm * rpm * pc;
    float acc = 0.0f;
#ifndef HCB_REDUCE_UNROLL
#define HCB_REDUCE_UNROLL 8
#endif
    constexpr int U = HCB_REDUCE_UNROLL;  // loads in flight per lane (the sum order is unchanged)
    int s = j;
    for (; s + 8 * (U - 1) < splits; s += 8 * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = p[(long long)(s + 8 * u) * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    for (; s < splits; s += 8) acc += p[(long long)s * stride];
    return acc;
}

// dW_ref[co][ci*taps + t] = sum_split partial[split][t*C + ci][co]  (fixed order).
// Block = 32 consecutive (m, co) outputs x 8 split lanes: lane j sums splits j, j+8, ...,
// then the 8 lane sums are added in lane order -> deterministic, 8x the loads in flight of
// a thread-per-output loop (hundreds of splits at small C).
// (C, Cout): the GEMM's (possibly zero-padded) channels; (cin_r, cout_r): the written dW's.
__global__ void __launch_bounds__(256) k_reduce_dw(const float* __restrict__ partial, const DwGroups grp_tab,
                                                  int taps, int C, int Cout, float* __restrict__ dw, int cin_r,
                                                  int cout_r) {
    __shared__ float red[8][33];
    const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;
    const long long i = blockIdx.x * 32LL + lane;  // over (taps*C) x Cout
    const long long total = (long long)taps * C * Cout;
    float acc = 0.0f;
    long long m = 0;
    int co = 0;
    if (i < total) {
        m = i / Cout;
        co = (int)(i - m * Cout);
        acc = split_lane_sum(partial, grp_tab, m, co, j);
    }
    red[j][lane] = acc;
    __syncthreads();
    if (j == 0 && i < total) {
        float v = red[0][lane];
#pragma unroll
        for (int k = 1; k < 8; ++k) v += red[k][lane];
        const int t = (int)(m / C), ci = (int)(m - (long long)t * C);
        if (ci < cin_r && co < cout_r) dw[(long long)co * cin_r * taps + (long long)ci * taps + t] = v;
    }
}

// Row-major [n][taps] (layout 0) or tap-major [taps][n] (layout 1) -> tile-major
// [ceil(n/128)][taps][128] with -1 padding (the layout both kernels consume).
__global__ void k_retile(const int* __restrict__ src, int layout, long long n, int taps, int* __restrict__ dst) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // over padded n x taps (tile-major)
    const long long padded = (n + 127) / 128 * 128;
    if (i >= padded * taps) return;
    const long long tile = i / (taps * 128);
    const int rem = (int)(i - tile * taps * 128);
    const int t = rem / 128;
    const long long col = tile * 128 + (rem & 127);
    int v = -1;
    if (col < n) v = layout == 0 ? src[col * taps + t] : src[(long long)t * n + col];
    dst[i] = v;
}

// ====================================================================== layout helpers
// W_ref[co][ci*taps + t] (fp32, kernel weights layout cnn_ops.hpp:21-27) ->
//   mode 0 (forward):    Wp[co][t*C_in + ci]  = W_ref[co][ci*taps + t]   (bf16, K padded to Kp)
//   mode 1 (backward):   Wp[ci][t*C_out + co] = W_ref[co][ci*taps + (taps-1-t)]
//   mode 2 (transpose):  Wp[ci][t*C_out + co] = W_ref[co][ci*taps + t]   (deconvolution, W^T)
__global__ void k_pack_w(const float* __restrict__ w, int cout, int cin, int taps, int mode, int Kp,
                         bf16* __restrict__ wp) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int rows = mode ? cin : cout;
    if (i >= (long long)rows * Kp) return;
    const int r = (int)(i / Kp), k = (int)(i % Kp);
    float v = 0.0f;
    if (mode == 0) {
        if (k < taps * cin) {
            const int t = k / cin, ci = k % cin;
            v = w[(long long)r * cin * taps + ci * taps + t];
        }
    } else {
        if (k < taps * cout) {
            const int t = k / cout, co = k % cout;
            v = w[(long long)co * cin * taps + r * taps + (mode == 1 ? taps - 1 - t : t)];
        }
    }
    wp[i] = __float2bfloat16_rn(v);
}

// Split precision: an fp32 value v is carried as two bf16 planes hi = rn(v), lo = rn(v - hi)
// (|v - hi - lo| <= 2^-17 |v|); the products hi.hi + hi.lo + lo.hi (+ lo.lo) accumulate in fp32.

// Weights in the split layout: rows [0, R) the hi plane, [R, 2R) the lo plane of the mode's
// matrix (as k_pack_w); each tap's K segment is [hi features | lo features] (2 Ck wide) with
// the same weight value in both halves, so row q, segment p multiplies plane q by plane p.
// (cout, cin): the reference weight matrix; (cout_p, cin_p) >= them: the zero-padded operand.
__global__ void k_pack_w_x2(const float* __restrict__ w, int cout, int cin, int taps, int mode, int Kp2,
                            bf16* __restrict__ wp, int cout_p, int cin_p) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int rows = mode ? cin_p : cout_p;
    if (i >= 2LL * rows * Kp2) return;
    const int rr = (int)(i / Kp2), k = (int)(i % Kp2);
    const int q = rr >= rows, r = rr - q * rows;
    const int ck = mode ? cout_p : cin_p;
    const int g = x2_block(ck);
    float v = 0.0f;
    if (k < taps * 2 * ck) {
        const int t = k / (2 * ck);
        const int kr = k - t * 2 * ck;                     // position inside the tap's row
        const int c = (kr / (2 * g)) * g + kr % g;         // channel (either plane)
        const int co = mode ? c : r, ci = mode ? r : c;
        if (co < cout && ci < cin)
            v = w[(long long)co * cin * taps + ci * taps + (mode == 1 ? taps - 1 - t : t)];
    }
    bf16 hi, lo;
    split2(v, hi, lo);
    wp[i] = q ? lo : hi;
}

// channel-major fp32 (C rows of stride ld) -> split voxel-major rows [N][2Cp] bf16 =
// [hi(0..Cp-1) | lo(0..Cp-1)], channels C..Cp-1 zero (padding to the tensor-core tile set)
__global__ void k_split_cm(const float* __restrict__ in, long long C, long long N, long long ld, long long Cp,
                           bf16* __restrict__ out) {
    __shared__ float tile[32][33];
    const long long n0 = (long long)blockIdx.x * 32, c0 = (long long)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long c = c0 + i, n = n0 + threadIdx.x;
        tile[i][threadIdx.x] = (c < C && n < N) ? in[c * ld + n] : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long n = n0 + i, c = c0 + threadIdx.x;
        if (c < Cp && n < N) {
            bf16 hi, lo;
            split2(tile[threadIdx.x][i], hi, lo);
            const int g = x2_block((int)Cp);
            out[n * 2 * Cp + x2_pos((int)c, 0, g)] = hi;
            out[n * 2 * Cp + x2_pos((int)c, 1, g)] = lo;
        }
    }
}

// voxel-major fp32 [N][C] (C % 4 == 0) -> split rows [N][2C] bf16
__global__ void k_split_vm(const float4* __restrict__ in, long long N, int C, bf16* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // over N * C/4
    const int c4 = C / 4;
    if (i >= N * c4) return;
    const long long n = i / c4;
    const int c = (int)(i - n * c4) * 4;
    const float4 v = in[i];
    bf16 h[4], l[4];
    split2(v.x, h[0], l[0]);
    split2(v.y, h[1], l[1]);
    split2(v.z, h[2], l[2]);
    split2(v.w, h[3], l[3]);
    bf16* row = out + n * 2 * C;
    const int g = x2_block(C);
    *reinterpret_cast<uint2*>(row + x2_pos(c, 0, g)) = *reinterpret_cast<uint2*>(h);
    *reinterpret_cast<uint2*>(row + x2_pos(c, 1, g)) = *reinterpret_cast<uint2*>(l);
}

// Transposed field map for the deconvolution (cnn_ops.cpp:408-419, col2hash of W^T D):
// from the conv map pmap [n_coarse][taps] (fine column of coarse voxel p's field row t)
// build tmap [ceil(n_fine/128)][taps][128] (tile-major): tmap[g][t] = the coarse voxel
// whose field holds fine voxel g at row t, or -1. (g, t) determines p uniquely
// (p*S - pad = g - offset(t)), so the scatter has no conflicts; tmap pre-filled with -1.
__global__ void k_transpose_map(const int* __restrict__ pmap, long long nc, int taps, int* __restrict__ tmap) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nc * taps) return;
    const int g = pmap[i];
    if (g < 0) return;
    const int t = (int)(i % taps);
    tmap[((long long)(g >> 7) * taps + t) * 128 + (g & 127)] = (int)(i / taps);
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
__global__ void k_to_channel_major(const T* __restrict__ in, long long N, long long C, float* __restrict__ out,
                                   long long ld) {  // ld: input row stride (>= C)
    __shared__ float tile[32][33];
    const long long n0 = (long long)blockIdx.x * 32, c0 = (long long)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long n = n0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (c < C && n < N) ? to_f<T>(in[n * ld + c]) : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long c = c0 + i, n = n0 + threadIdx.x;
        if (c < C && n < N) out[c * N + n] = tile[threadIdx.x][i];
    }
}


// ====================================================================== launchers
// Forward variant: HCB_FWD_CPS = CTAs per SM (2: BN <= 64 only, so both CTAs'
// double-buffered accumulators fit TMEM; 1: one deep ring), HCB_FWD_PW = producer warps
// (2, 4 or 8).
template <int BN, int CPS, int PW, typename OutT, bool SUMH = false>
void launch_fwd(const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, OutT* Y,
                cudaStream_t s, int skip_lolo = 0) {
    using Cfg = FwdCfg<BN, CPS, PW, sizeof(OutT)>;
    auto kern = k_conv_fwd<BN, CPS, PW, OutT, SUMH>;
    smem_optin(kern, Cfg::SMEM);
    const CUtensorMap wm = map2d(Wp, (uint64_t)Kp, (uint64_t)BN, (uint64_t)Kp * 2, BN);
    const int tiles = (int)((rows + BM - 1) / BM);
    const int grid = std::min(tiles, CPS * num_sms());
    const CUtensorMap ym = map_out(Y, sizeof(OutT) == 4, (uint64_t)(SUMH ? BN / 2 : BN), (uint64_t)rows, 16, 32);
    kern<<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(wm, ym, fmap, taps, rows, X, C, Kp / BK, tiles, skip_lolo, g_tile_stats);
    launched(SUMH ? "conv gather-GEMM, split precision (tcgen05)" : "conv gather-GEMM (tcgen05)");
}

template <int BN, typename OutT>
void launch_fwd_bn(const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, OutT* Y,
                   cudaStream_t s) {
    // Defaults measured on B200 at 256^3 x 8 shells (scripts/gpu_ab.sh): two CTAs per SM
    // with 4 producer warps each wherever both CTAs' accumulators fit (BN <= 64), else one
    // CTA with 4 producer warps.
    static const int cps = env_int("HCB_FWD_CPS", 2);
    static const int pw = env_int("HCB_FWD_PW", 4);
    if constexpr (BN <= 64) {
        if (cps == 2) {
            if (pw == 2) return launch_fwd<BN, 2, 2>(fmap, taps, rows, X, C, Wp, Kp, Y, s);
            if (pw == 8) return launch_fwd<BN, 2, 8>(fmap, taps, rows, X, C, Wp, Kp, Y, s);
            return launch_fwd<BN, 2, 4>(fmap, taps, rows, X, C, Wp, Kp, Y, s);
        }
    }
    if (pw == 4) return launch_fwd<BN, 1, 4>(fmap, taps, rows, X, C, Wp, Kp, Y, s);
    launch_fwd<BN, 1, 8>(fmap, taps, rows, X, C, Wp, Kp, Y, s);
}

// Split-precision forward: BN = 2 x output channels (hi and lo weight planes), fp32 output.
// Two CTAs per SM where both CTAs' double-buffered accumulators fit TMEM (BN <= 128; C 64->64:
// 1.35 vs 1.66 ms with one CTA and a deeper ring), else one (HCB_X2_CPS=1 forces it).
template <int BN>
void launch_fwd_x2(const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, float* Y,
                   cudaStream_t s, int skip_lolo) {
    static const int cps = env_int("HCB_X2_CPS", BN <= 128 ? 2 : 1);
    static const int pw = env_int("HCB_X2_PW", 4);
    if constexpr (BN <= 128) {
        if (cps == 2 && pw == 8) return launch_fwd<BN, 2, 8, float, true>(fmap, taps, rows, X, C, Wp, Kp, Y, s, skip_lolo);
        if (cps == 2 && pw == 2) return launch_fwd<BN, 2, 2, float, true>(fmap, taps, rows, X, C, Wp, Kp, Y, s, skip_lolo);
        if (cps == 2) return launch_fwd<BN, 2, 4, float, true>(fmap, taps, rows, X, C, Wp, Kp, Y, s, skip_lolo);
    }
    launch_fwd<BN, 1, 4, float, true>(fmap, taps, rows, X, C, Wp, Kp, Y, s, skip_lolo);
}

template <int BN, int CPS, int PW, int SA, int SB, int NBUF>
void launch_fwd_x2s(const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, float* Y,
                    cudaStream_t s) {
    using Cfg = FwdX2Cfg<BN, CPS, PW, SA, SB, NBUF>;
    auto kern = k_conv_fwd_x2<BN, CPS, PW, SA, SB, NBUF>;
    smem_optin(kern, Cfg::SMEM);
    const CUtensorMap wm = map2d(Wp, (uint64_t)Kp, (uint64_t)BN, (uint64_t)Kp * 2, BN);
    const int tiles = (int)((rows + BM - 1) / BM);
    const int grid = std::min(tiles, CPS * num_sms());
    const CUtensorMap ym = map_out(Y, true, (uint64_t)(BN / 2), (uint64_t)rows, 16, 32);
    kern<<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(wm, ym, fmap, taps, X, C, Kp / BK, tiles, rows, g_tile_stats);
    launched("conv gather-GEMM, split precision, shared weight ring (tcgen05)");
}

// C_in a multiple of 64 (rows interleaved per 64 channels): the shared-weight-ring kernel.
// HCB_X2_RING: 0 = the generic SUMH kernel, 1 = (A 2, B 2, 2 map buffers), 2 = (A 3, B 2, 1 map buffer),
// 8 (default) = (A 4, B 2, map entries from global one tap ahead; 1-2% faster than 2 at C 64->64).
// 3-7: deeper rings / one CTA per SM / 8 producer warps, all measured slower.
bool conv_fwd_x2_shared(const int* fmap, int taps, long long rows, const bf16* X, int C2, const bf16* Wp, int Kp,
                        int N2, float* Y, cudaStream_t s) {
    static const int ring = env_int("HCB_X2_RING", 8);
    if (ring == 0 || (C2 / 2) % 64 != 0) return false;
    if (N2 == 128) {
        if (ring == 3) launch_fwd_x2s<128, 2, 4, 2, 3, 1>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else if (ring == 4) launch_fwd_x2s<128, 1, 4, 8, 2, 2>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else if (ring == 5) launch_fwd_x2s<128, 1, 8, 8, 2, 2>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else if (ring == 6) launch_fwd_x2s<128, 1, 8, 9, 3, 1>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else if (ring == 7) launch_fwd_x2s<128, 2, 8, 3, 2, 1>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else if (ring == 8 && Kp / BK == taps * (C2 / BK))  // map from global, 4-deep A ring
            launch_fwd_x2s<128, 2, 4, 4, 2, 0>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else if (ring == 2 || ring == 8) launch_fwd_x2s<128, 2, 4, 3, 2, 1>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else launch_fwd_x2s<128, 2, 4, 2, 2, 2>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        return true;
    }
    if (N2 == 64) {
        if (ring == 8 && Kp / BK == taps * (C2 / BK)) launch_fwd_x2s<64, 2, 4, 4, 2, 0>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else if (ring == 2 || ring == 8) launch_fwd_x2s<64, 2, 4, 3, 2, 1>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        else launch_fwd_x2s<64, 2, 4, 2, 2, 2>(fmap, taps, rows, X, C2, Wp, Kp, Y, s);
        return true;
    }
    return false;
}

void conv_fwd_x2(const int* fmap, int taps, long long rows, const bf16* X, int C2, const bf16* Wp, int Kp, int N2,
                 float* Y, cudaStream_t s) {
    if (conv_fwd_x2_shared(fmap, taps, rows, X, C2, Wp, Kp, N2, Y, s)) return;
    static const int keep_lolo = env_int("HCB_X2_LOLO", 0);
    const int g = x2_block(C2 / 2);
    const int skip = (!keep_lolo && g % 16 == 0) ? g : 0;  // the lo plane's K16 chunks issue N = BN/2
    switch (N2) {
        case 32: launch_fwd_x2<32>(fmap, taps, rows, X, C2, Wp, Kp, Y, s, skip); break;
        case 64: launch_fwd_x2<64>(fmap, taps, rows, X, C2, Wp, Kp, Y, s, skip); break;
        case 128: launch_fwd_x2<128>(fmap, taps, rows, X, C2, Wp, Kp, Y, s, skip); break;
        case 256: launch_fwd_x2<256>(fmap, taps, rows, X, C2, Wp, Kp, Y, s, skip); break;
        default: throw std::invalid_argument("native conv (split precision): output channels must be 16, 32, 64 or 128");
    }
}

template <typename OutT>
void conv_fwd(const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, int N, OutT* Y,
              cudaStream_t s) {
    switch (N) {
        case 16: launch_fwd_bn<16>(fmap, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 32: launch_fwd_bn<32>(fmap, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 64: launch_fwd_bn<64>(fmap, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 128: launch_fwd_bn<128>(fmap, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 256: launch_fwd_bn<256>(fmap, taps, rows, X, C, Wp, Kp, Y, s); break;
        default: throw std::invalid_argument("native conv: output channels must be 16, 32, 64, 128 or 256");
    }
}

int dw_nb(int cout) { return cout <= 64 ? 64 : cout <= 128 ? 128 : 256; }

// Split plan: m-tiles are grouped so each group's accumulators fit TMEM (m-tiles * NB <=
// 512 / CPS columns) and the groups' CTAs fill the SMs x CPS slots. Deterministic for a
// given SM count.
// HCB_DW_CPS = resident dW CTAs per SM (2, default: 256 TMEM columns each, NB <= 128 —
// two independent pipelines per SM measured 11% faster at C=64; 1: 512 columns).
int dw_cps(int nb) {
    static const int env = env_int("HCB_DW_CPS", 2);
    return (env == 2 && nb <= 128) ? 2 : 1;
}

struct DwPlan {
    int nb, mt, cps, ctas, tiles, max_taps;
    DwGroups g;
    long long partial_floats;
};

// max_tps > 0 caps a split's voxel tiles (the length of one TMEM accumulation chain).
// pair: split precision — cin / cout are the channels of one plane, the GEMM runs on rows of
// 2 cin (X) and 2 cout (dY) with 64 (t, ci) rows x both planes per m-tile (DwGroups).
// mode (split precision): 1 = pair (four plane products per m-tile), 2 = tri (three products:
// units of 128 (t, ci) rows, a hi m-tile against [dY_hi | dY_lo] and a lo m-tile against dY_hi).
int x2_dw_mode() {
    static const int v = env_int("HCB_X2_DW_TRI", 1) ? 2 : 1;
    return v;
}

DwPlan dw_plan(long long rows, int taps, int cin, int cout, int max_tps = 0, bool pair = false) {
    DwPlan p{};
    // tri needs c_out >= 32 to pay (C 16: 0.50 ms tri vs 0.43 pair; C 32: 0.62 vs 0.68; C 64: 1.46 vs 1.62)
    const int mode = pair ? (cout >= 32 ? x2_dw_mode() : 1) : 0;
    const int rpm = mode == 1 ? 64 : BM;
    p.nb = dw_nb(pair ? 2 * cout : cout);
    p.mt = (taps * cin + rpm - 1) / rpm;  // m-tiles (tri: units of a hi and a lo m-tile)
    p.cps = dw_cps(p.nb);
    p.tiles = (int)((rows + BM - 1) / BM);
    // pair mode with chunked accumulation: HCB_DW_DBUF=1 keeps two accumulator sets per CTA (the
    // epilogue drains one chunk while the next accumulates) at half the m-tiles per CTA
    static const int dbuf_env = env_int("HCB_DW_DBUF", 0);
    // tri: [hi.dY_hi + lo.dY_hi | hi.dY_lo] (c_out <= 64, shared) or + a separate lo.dY_hi (wider)
    static const int tshared_env = env_int("HCB_DW_TRI_SHARED", 1);
    const bool tshared = mode == 2 && cout > 32 && cout <= 64 && tshared_env;  // C 64: 1.47 -> 1.42 ms; C 32 slower (0.68 vs 0.67)
    const int unit_cols = mode == 2 ? (tshared ? 2 * cout : 3 * cout) : p.nb;
    const int nacc = (pair && max_tps > 0 && dbuf_env && 512 / (unit_cols * p.cps * 2) >= 1) ? 2 : 1;
    const int cap = std::min(mode == 2 ? 8 : 16, 512 / (unit_cols * p.cps * nacc));  // m-tiles (units) per CTA
    const int G = (p.mt + cap - 1) / cap;  // -> every group has <= cap m-tiles
    if (cap < 1 || G > kMaxGroups)
        throw std::invalid_argument("native conv: dW supports at most " + std::to_string(kMaxGroups * std::max(cap, 0) * BM) +
                                    " (taps x input channels) rows at " + std::to_string(cout) + " output channels");
    const int slots = num_sms() * p.cps;
    DwGroups& g = p.g;
    g.groups = G;
    g.pair = mode;
    g.tshared = tshared ? 1 : 0;
    g.nacc = nacc;
    static const int strided = env_int("HCB_DW_STRIDED", 1);
    g.strided = strided;
    g.rpm = rpm;
    g.pcols = pair ? cout : p.nb;
    // Few groups (C_out <= 64): CTAs proportional to each group's m-tiles, so groups of
    // 4 and 3 m-tiles finish together (C=64: 0.667 -> 0.607 ms). Many groups (C_out >= 128,
    // 14+ groups re-reading dY): equal voxel splits in lockstep, so one range's dY tile and
    // gathered rows are shared through L2 by all groups (proportional splits lose that
    // alignment: C=128 1.51 -> 2.0 ms); the imbalance of 2-vs-1 m-tile groups is small there.
    const bool proportional = G <= 4;
    const int eq_want = std::max(1, std::min(p.tiles, slots / G));
    long long part = 0;
    g.m_begin[0] = 0;
    g.cta_begin[0] = 0;
    for (int i = 0; i < G; ++i) {
        g.m_begin[i + 1] = (int)((long long)p.mt * (i + 1) / G);
        const int mg = g.m_begin[i + 1] - g.m_begin[i];
        int want = eq_want;
        if (proportional) {
            const int end = (int)((long long)slots * g.m_begin[i + 1] / p.mt);
            want = std::max(1, std::min(p.tiles, end - g.cta_begin[i]));
        }
        g.tps[i] = std::max(1, (p.tiles + want - 1) / want);  // tiles per CTA ...
        if (max_tps > 0) g.tps[i] = std::min(g.tps[i], max_tps);  // ... cut into chunks of <= max_tps
        static const int phase = env_int("HCB_DW_PHASE", 1);
        // half-chunk phase shift of odd groups: C 128 5.45 -> 5.29 ms; with the shared tri accumulator
        // (C 64, 7 groups) it costs 3% (1.31 -> 1.35), so not there
        g.shift[i] = (phase && strided && max_tps > 0 && !tshared && (i & 1) && g.tps[i] >= 2 && p.tiles > g.tps[i])
                         ? g.tps[i] / 2 : 0;
        g.nchunk[i] = std::max(1, (p.tiles + g.shift[i] + g.tps[i] - 1) / g.tps[i]);
        g.cpc[i] = (g.nchunk[i] + want - 1) / want;
        g.cta_begin[i + 1] = g.cta_begin[i] + (g.nchunk[i] + g.cpc[i] - 1) / g.cpc[i];
        g.part_begin[i] = part;
        part += (long long)g.nchunk[i] * mg * rpm * g.pcols;
    }
    p.ctas = g.cta_begin[G];
    p.partial_floats = part;
    p.max_taps = 0;  // widest tap range any group's m-tiles touch
    for (int i = 0; i < G; ++i) {
        const int lo = g.m_begin[i] * rpm / cin;
        const int hi = (std::min(taps * cin, g.m_begin[i + 1] * rpm) - 1) / cin;
        p.max_taps = std::max(p.max_taps, hi - lo + 1);
    }
    return p;
}

template <int NB, int PW, int CPS, int NT = kMaxTaps>
void launch_dw_pw(const DwPlan& p, const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* dY,
                  int Cout, float* partial, cudaStream_t s) {
    using Cfg = DwCfg<NB, PW, CPS, NT>;
    auto kern = k_conv_dw<NB, PW, CPS, NT>;
    smem_optin(kern, Cfg::SMEM);
    // dY [rows][Cout] bf16: boxes of 64 voxels x 64 channels; channels >= Cout and voxels
    // >= rows are out of bounds -> zero.
    const CUtensorMap dm = map2d(dY, (uint64_t)Cout, (uint64_t)rows, (uint64_t)Cout * 2, 64);
    kern<<<p.ctas, Cfg::THREADS, Cfg::SMEM, s>>>(dm, fmap, taps, rows, X, C, p.g, p.tiles, partial);
    launched("conv dW gather-GEMM (tcgen05)");
}

// HCB_DW_PW = producer warps of the dW kernel (2/4/8 with 2 CTAs per SM, default 4;
// 4/8 with one, default 8). Measured on B200 (scripts/gpu_ab.sh).
template <int NB>
void launch_dw(const DwPlan& p, const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* dY,
               int Cout, float* partial, cudaStream_t s) {
    static const int pw = env_int("HCB_DW_PW", p.cps == 2 ? 4 : 8);
    if constexpr (NB <= 128) {
        if (p.cps == 2) {
            if (pw == 2) return launch_dw_pw<NB, 2, 2>(p, fmap, taps, rows, X, C, dY, Cout, partial, s);
            if (pw == 8) return launch_dw_pw<NB, 8, 2>(p, fmap, taps, rows, X, C, dY, Cout, partial, s);
            static const int small_map = env_int("HCB_DW_SMALLMAP", 1);
            if (small_map && p.max_taps <= 9) return launch_dw_pw<NB, 4, 2, 9>(p, fmap, taps, rows, X, C, dY, Cout, partial, s);
            return launch_dw_pw<NB, 4, 2>(p, fmap, taps, rows, X, C, dY, Cout, partial, s);
        }
    }
    if (pw == 4) return launch_dw_pw<NB, 4, 1>(p, fmap, taps, rows, X, C, dY, Cout, partial, s);
    launch_dw_pw<NB, 8, 1>(p, fmap, taps, rows, X, C, dY, Cout, partial, s);
}

void check_native(int cin, int cout, int taps) {
    if (cin <= 0 || cin % 8 != 0) throw std::invalid_argument("native conv: input channels must be a multiple of 8");
    if (cout <= 0 || cout % 8 != 0) throw std::invalid_argument("native conv: output channels must be a multiple of 8");
    if (taps < 1 || taps > 27) throw std::invalid_argument("native conv: 1..27 field taps supported");
}

// The kernels consume the tile-major map; the row-major / tap-major layouts are
// re-tiled into stream-ordered scratch first.
struct TiledMap {
    const int* p;
    Scratch* tmp;
    TiledMap(const int32_t* fmap, int32_t layout, long long n, int taps, cudaStream_t s) : p(fmap), tmp(nullptr) {
        if (layout == 2) return;
        if (layout != 0 && layout != 1) throw std::invalid_argument("native conv: unknown field-map layout");
        const long long total = (n + 127) / 128 * 128 * taps;
        tmp = new Scratch((size_t)total * 4, s);
        k_retile<<<grid_for(total, 256), 256, 0, s>>>(fmap, layout, n, taps, tmp->as<int>());
        launched("field map re-tile");
        p = tmp->as<int>();
    }
    ~TiledMap() { delete tmp; }
    TiledMap(const TiledMap&) = delete;
    TiledMap& operator=(const TiledMap&) = delete;
};

int x2_dw_tps() {
    // One TMEM accumulation chain covers at most HCB_X2_DW_TPS voxel tiles (default 32 = 4096
    // voxels): the tensor core's fp32 accumulation over hundreds of thousands of products
    // drifts past the 1e-5 contract (256^3 x 8, C 64: 9e-5 unbounded, 7.5e-6 at 64 tiles,
    // 4.3e-6 at 32, 3.4e-6 at 16), the fixed-order split reduction does not.
    static const int v = env_int("HCB_X2_DW_TPS", 32);
    return v;
}

}  // namespace

// ---------------------------------------------------------------- reference-signature FAST route
// conv_forward / conv_backward (cnn_ops.cpp:206-232) in HC_MATH_FAST on a stride-1 layer over
// one structure: the fused split-precision implicit GEMM instead of hash2col + 3xTF32 GEMMs over
// the materialised column matrix. Reference layout in and out; channels zero-padded to the
// tile set inside.
static int tile_ch(int c) { return c <= 16 ? 16 : c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : 256; }

bool fused_x2_eligible(const hc_psh* in, const hc_psh* out, hc_conv_spec sp, int taps) {
    static const int on = env_int("HCB_FAST_FUSED", 1);
    return on && in == out && sp.stride == 1 && taps >= 1 && taps <= kMaxTaps && sp.in_channels > 0 &&
           sp.out_channels > 0 && tile_ch(sp.in_channels) <= 128 && tile_ch(sp.out_channels) <= 128;
}

namespace {
struct FusedMap {
    Scratch buf;
    FusedMap(const hc_psh* in, hc_conv_spec sp, int taps, long long N, cudaStream_t s)
        : buf((size_t)((N + 127) / 128) * 128 * taps * 4, s) {
        const hc_status st = hc_field_map_tiled(in, in, sp, buf.as<int32_t>(), reinterpret_cast<hc_stream>(s));
        if (st != HC_OK) throw std::runtime_error(hc_last_error());
    }
};
void split_cm(const float* src, long long C, long long N, long long ld, long long Cp, bf16* out, cudaStream_t s) {
    dim3 g((unsigned)((N + 31) / 32), (unsigned)((Cp + 31) / 32)), b(32, 8);
    k_split_cm<<<g, b, 0, s>>>(src, C, N, ld, Cp, out);
    launched("split fp32 -> bf16 hi/lo planes");
}
void pack_x2(const float* w, int cout, int cin, int taps, int mode, int cout_p, int cin_p, bf16* wp, int Kp2,
             cudaStream_t s) {
    const long long n = 2LL * (mode ? cin_p : cout_p) * Kp2;
    k_pack_w_x2<<<grid_for(n, 256), 256, 0, s>>>(w, cout, cin, taps, mode, Kp2, wp, cout_p, cin_p);
    launched("pack weights (split precision)");
}
void to_cm(const float* y, long long N, long long C, long long ld, float* out, cudaStream_t s) {
    dim3 g((unsigned)((N + 31) / 32), (unsigned)((C + 31) / 32)), b(32, 8);
    k_to_channel_major<float><<<g, b, 0, s>>>(y, N, C, out, ld);
    launched("to channel-major");
}
}  // namespace

void fused_conv_forward_f32(const hc_psh* in, const float* data, const float* w, hc_conv_spec sp, int taps,
                            long long N, float* result, cudaStream_t s) {
    const int cin = sp.in_channels, cout = sp.out_channels, cin_p = tile_ch(cin), cout_p = tile_ch(cout);
    const FusedMap fm(in, sp, taps, N, s);
    const int Kp2 = (int)hc_native_packed_k_x2(cin_p, taps);
    Scratch xs((size_t)N * 2 * cin_p * 2, s), wp((size_t)2 * cout_p * Kp2 * 2, s), y((size_t)N * cout_p * 4, s);
    split_cm(data, cin, N, N, cin_p, xs.as<bf16>(), s);
    pack_x2(w, cout, cin, taps, 0, cout_p, cin_p, wp.as<bf16>(), Kp2, s);
    conv_fwd_x2(fm.buf.as<int>(), taps, N, xs.as<bf16>(), 2 * cin_p, wp.as<bf16>(), Kp2, 2 * cout_p, y.as<float>(), s);
    to_cm(y.as<float>(), N, cout, cout_p, result, s);
}

// conv_backward's input is not passed (only the cached column matrix): for a stride-1 field
// over one structure the centre field row of column n IS input column n (the voxel itself,
// always present), so X = cached_cols rows c * taps + (taps - 1) / 2.
void fused_conv_backward_f32(const float* dy, const float* w, const float* cols, const hc_psh* in, hc_conv_spec sp,
                             int taps, long long N, float* dw, float* dx, cudaStream_t s) {
    const int cin = sp.in_channels, cout = sp.out_channels, cin_p = tile_ch(cin), cout_p = tile_ch(cout);
    const FusedMap fm(in, sp, taps, N, s);
    const int Kp2 = (int)hc_native_packed_k_x2(cout_p, taps);
    Scratch xs((size_t)N * 2 * cin_p * 2, s), dys((size_t)N * 2 * cout_p * 2, s);
    Scratch wp((size_t)2 * cin_p * Kp2 * 2, s), dxp((size_t)N * cin_p * 4, s);
    split_cm(cols + (long long)((taps - 1) / 2) * N, cin, N, (long long)taps * N, cin_p, xs.as<bf16>(), s);
    split_cm(dy, cout, N, N, cout_p, dys.as<bf16>(), s);
    const DwPlan p = dw_plan(N, taps, cin_p, cout_p, x2_dw_tps(), true);
    Scratch part((size_t)p.partial_floats * 4, s);
    const int C2 = 2 * cin_p, Co2 = 2 * cout_p;
    switch (p.nb) {
        case 64: launch_dw<64>(p, fm.buf.as<int>(), taps, N, xs.as<bf16>(), C2, dys.as<bf16>(), Co2, part.as<float>(), s); break;
        case 128: launch_dw<128>(p, fm.buf.as<int>(), taps, N, xs.as<bf16>(), C2, dys.as<bf16>(), Co2, part.as<float>(), s); break;
        default: launch_dw<256>(p, fm.buf.as<int>(), taps, N, xs.as<bf16>(), C2, dys.as<bf16>(), Co2, part.as<float>(), s); break;
    }
    const long long total = (long long)cout_p * cin_p * taps;
    k_reduce_dw<<<grid_for(total, 32), 256, 0, s>>>(part.as<float>(), p.g, taps, cin_p, cout_p, dw, cin, cout);
    launched("dW split reduction (split precision)");
    pack_x2(w, cout, cin, taps, 1, cout_p, cin_p, wp.as<bf16>(), Kp2, s);
    conv_fwd_x2(fm.buf.as<int>(), taps, N, dys.as<bf16>(), Co2, wp.as<bf16>(), Kp2, 2 * cin_p, dxp.as<float>(), s);
    to_cm(dxp.as<float>(), N, cin, cin_p, dx, s);
}

}  // namespace hcb

using namespace hcb;

extern "C" {

int64_t hc_native_packed_k(int32_t c, int32_t taps) { return ((int64_t)c * taps + 63) / 64 * 64; }

hc_status hc_native_pack_weights(const float* w_ref, int32_t c_out, int32_t c_in, int32_t taps, int32_t backward,
                                 void* w_packed, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (backward < 0 || backward > 2) throw std::invalid_argument("native conv: pack mode must be 0, 1 or 2");
        const int rows = backward ? c_in : c_out;
        const long long Kp = hc_native_packed_k(backward ? c_out : c_in, taps);
        const long long n = rows * Kp;
        k_pack_w<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(w_ref, c_out, c_in, taps, backward, (int)Kp,
                                                                   static_cast<bf16*>(w_packed));
        launched("pack weights");
    });
}

hc_status hc_native_transpose_map(const int32_t* pmap, int64_t n_coarse, int32_t taps, int64_t n_fine,
                                  int32_t* tmap_tiled, hc_stream stream) {
    return guard([&] {
        if (taps < 1 || taps > 27) throw std::invalid_argument("native conv: 1..27 field taps supported");
        cudaStream_t s = as_stream(stream);
        const long long total = (n_fine + 127) / 128 * 128 * taps;
        if (total > 0) cuda_check(cudaMemsetAsync(tmap_tiled, 0xFF, sizeof(int32_t) * total, s), "memset");
        if (n_coarse <= 0) return;
        k_transpose_map<<<grid_for(n_coarse * taps, 256), 256, 0, s>>>(pmap, n_coarse, taps, tmap_tiled);
        launched("transposed field map");
    });
}

hc_status hc_native_gather_gemm(const int32_t* fmap, int32_t fmap_layout, int64_t n_out, int32_t taps,
                                const void* x, int32_t c_in, const void* w_packed, int32_t c_out, void* y,
                                hc_dtype y_dtype, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (n_out <= 0) return;
        cudaStream_t s = as_stream(stream);
        const int Kp = (int)hc_native_packed_k(c_in, taps);
        const TiledMap fm(fmap, fmap_layout, n_out, taps, s);
        const bf16* X = static_cast<const bf16*>(x);
        const bf16* W = static_cast<const bf16*>(w_packed);
        if (y_dtype == HC_DTYPE_F32)
            conv_fwd<float>(fm.p, taps, n_out, X, c_in, W, Kp, c_out, static_cast<float*>(y), s);
        else
            conv_fwd<bf16>(fm.p, taps, n_out, X, c_in, W, Kp, c_out, static_cast<bf16*>(y), s);
    });
}

size_t hc_native_dw_workspace(int64_t n_out, int32_t taps, int32_t c_in, int32_t c_out) {
    size_t r = 0;  // 0 = unsupported shape (hc_native_conv_dw reports why)
    const hc_status st = guard([&] { r = (size_t)dw_plan(n_out, taps, c_in, c_out).partial_floats * sizeof(float); });
    return st == HC_OK ? r : 0;
}

hc_status hc_native_conv_dw(const int32_t* fmap, int32_t fmap_layout, int64_t n_out, int32_t taps, const void* x,
                            int32_t c_in, const void* dy, int32_t c_out, float* dw_ref, void* workspace,
                            size_t ws_bytes, hc_stream stream) {
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
        const TiledMap fm(fmap, fmap_layout, n_out, taps, s);
        const bf16* X = static_cast<const bf16*>(x);
        const bf16* DY = static_cast<const bf16*>(dy);
        switch (p.nb) {
            case 64: launch_dw<64>(p, fm.p, taps, n_out, X, c_in, DY, c_out, part, s); break;
            case 128: launch_dw<128>(p, fm.p, taps, n_out, X, c_in, DY, c_out, part, s); break;
            default: launch_dw<256>(p, fm.p, taps, n_out, X, c_in, DY, c_out, part, s); break;
        }
        const long long total = (long long)c_out * c_in * taps;
        k_reduce_dw<<<grid_for(total, 32), 256, 0, s>>>(part, p.g, taps, c_in, c_out, dw_ref, c_in, c_out);
        launched("dW split reduction");
    });
}

// ---------------------------------------------------------------- split precision (fp32-accurate)
int64_t hc_native_packed_k_x2(int32_t c, int32_t taps) { return ((int64_t)2 * c * taps + 63) / 64 * 64; }

hc_status hc_native_split(const float* src, int32_t channel_major, int64_t c, int64_t n, void* out,
                          hc_stream stream) {
    return guard([&] {
        if (c <= 0 || c % 4 != 0) throw std::invalid_argument("native split: channels must be a positive multiple of 4");
        if (n <= 0) return;
        cudaStream_t s = as_stream(stream);
        bf16* o = static_cast<bf16*>(out);
        if (channel_major) {
            dim3 g((unsigned)((n + 31) / 32), (unsigned)((c + 31) / 32)), b(32, 8);
            k_split_cm<<<g, b, 0, s>>>(src, c, n, n, c, o);
        } else {
            const long long total = n * (c / 4);
            k_split_vm<<<grid_for(total, 256), 256, 0, s>>>(reinterpret_cast<const float4*>(src), n, (int)c, o);
        }
        launched("split fp32 -> bf16 hi/lo planes");
    });
}

// Forward and flipped (dX) operands of one layer in one launch (blockIdx.y selects the mode);
// the dX operand may be zero-padded to c_in_bwd >= c_in input channels (the tile set starts at 16).
__global__ void k_pack_w_x2_fb(const float* __restrict__ w, int cout, int cin, int taps, int Kf, int Kb, int cin_bwd,
                               bf16* __restrict__ wf, bf16* __restrict__ wb) {
    const bool b = blockIdx.y == 1;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int rows = b ? cin_bwd : cout;
    const int Kp2 = b ? Kb : Kf;
    if (i >= 2LL * rows * Kp2) return;
    const int rr = (int)(i / Kp2), k = (int)(i % Kp2);
    const int q = rr >= rows, r = rr - q * rows;
    const int ck = b ? cout : cin;  // K-side channels of this operand
    const int g = x2_block(ck);
    float v = 0.0f;
    if (k < taps * 2 * ck) {
        const int t = k / (2 * ck);
        const int kr = k - t * 2 * ck;
        const int c = (kr / (2 * g)) * g + kr % g;
        const int co = b ? c : r, ci = b ? r : c;
        if (co < cout && ci < cin) v = w[(long long)co * cin * taps + ci * taps + (b ? taps - 1 - t : t)];
    }
    bf16 hi, lo;
    split2(v, hi, lo);
    (b ? wb : wf)[i] = q ? lo : hi;
}

hc_status hc_native_pack_weights_x2_fb(const float* w_ref, int32_t c_out, int32_t c_in, int32_t taps,
                                       int32_t c_in_bwd, void* w_fwd, void* w_bwd, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (c_in_bwd < c_in || c_in_bwd % 8) throw std::invalid_argument("native conv: c_in_bwd must be >= c_in, % 8");
        const long long Kf = hc_native_packed_k_x2(c_in, taps), Kb = hc_native_packed_k_x2(c_out, taps);
        const long long n = std::max(2LL * c_out * Kf, 2LL * c_in_bwd * Kb);
        const dim3 grid((unsigned)grid_for(n, 256), 2);
        k_pack_w_x2_fb<<<grid, 256, 0, as_stream(stream)>>>(w_ref, c_out, c_in, taps, (int)Kf, (int)Kb, c_in_bwd,
                                                            static_cast<bf16*>(w_fwd), static_cast<bf16*>(w_bwd));
        launched("pack weights fwd + dX (split precision)");
    });
}

hc_status hc_native_pack_weights_x2(const float* w_ref, int32_t c_out, int32_t c_in, int32_t taps, int32_t mode,
                                    void* w_packed, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (mode < 0 || mode > 2) throw std::invalid_argument("native conv: pack mode must be 0, 1 or 2");
        const int rows = mode ? c_in : c_out;
        const long long Kp2 = hc_native_packed_k_x2(mode ? c_out : c_in, taps);
        const long long n = 2LL * rows * Kp2;
        k_pack_w_x2<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(w_ref, c_out, c_in, taps, mode, (int)Kp2,
                                                                      static_cast<bf16*>(w_packed), c_out, c_in);
        launched("pack weights (split precision)");
    });
}

hc_status hc_native_gather_gemm_stats(const int32_t* fmap, int32_t fmap_layout, int64_t n_out, int32_t taps,
                                      const void* x, int32_t c_in, const void* w_packed, int32_t c_out, void* y,
                                      hc_dtype y_dtype, float* tile_stats, hc_stream stream) {
    const TileStatsScope scope(reinterpret_cast<float2*>(tile_stats));
    return hc_native_gather_gemm(fmap, fmap_layout, n_out, taps, x, c_in, w_packed, c_out, y, y_dtype, stream);
}

hc_status hc_native_gather_gemm_x2_stats(const int32_t* fmap, int32_t fmap_layout, int64_t n_out, int32_t taps,
                                         const void* x_split, int32_t c_in, const void* w_packed_x2, int32_t c_out,
                                         float* y, float* tile_stats, hc_stream stream) {
    const TileStatsScope scope(reinterpret_cast<float2*>(tile_stats));
    return hc_native_gather_gemm_x2(fmap, fmap_layout, n_out, taps, x_split, c_in, w_packed_x2, c_out, y, stream);
}

hc_status hc_native_gather_gemm_x2(const int32_t* fmap, int32_t fmap_layout, int64_t n_out, int32_t taps,
                                   const void* x_split, int32_t c_in, const void* w_packed_x2, int32_t c_out,
                                   float* y, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (c_out > 128) throw std::invalid_argument("native conv (split precision): at most 128 output channels");
        if (n_out <= 0) return;
        cudaStream_t s = as_stream(stream);
        const int Kp2 = (int)hc_native_packed_k_x2(c_in, taps);
        const TiledMap fm(fmap, fmap_layout, n_out, taps, s);
        conv_fwd_x2(fm.p, taps, n_out, static_cast<const bf16*>(x_split), 2 * c_in,
                    static_cast<const bf16*>(w_packed_x2), Kp2, 2 * c_out, y, s);
    });
}

size_t hc_native_dw_workspace_x2(int64_t n_out, int32_t taps, int32_t c_in, int32_t c_out) {
    size_t r = 0;
    const hc_status st = guard([&] {
        const DwPlan p = dw_plan(n_out, taps, c_in, c_out, x2_dw_tps(), true);
        r = (size_t)p.partial_floats * sizeof(float);
    });
    return st == HC_OK ? r : 0;
}

hc_status hc_native_conv_dw_x2(const int32_t* fmap, int32_t fmap_layout, int64_t n_out, int32_t taps,
                               const void* x_split, int32_t c_in, const void* dy_split, int32_t c_out, float* dw_ref,
                               void* workspace, size_t ws_bytes, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (c_out > 128) throw std::invalid_argument("native conv (split precision): dW supports up to 128 output channels");
        cudaStream_t s = as_stream(stream);
        if (n_out <= 0) {
            cuda_check(cudaMemsetAsync(dw_ref, 0, sizeof(float) * c_out * c_in * taps, s), "memset");
            return;
        }
        const int C2 = 2 * c_in, Co2 = 2 * c_out;
        if (c_out % 16 != 0) throw std::invalid_argument("native conv (split precision): dW output channels must be a multiple of 16");
        const DwPlan p = dw_plan(n_out, taps, c_in, c_out, x2_dw_tps(), true);
        if (ws_bytes < (size_t)p.partial_floats * sizeof(float))
            throw std::invalid_argument("native conv: dW workspace too small");
        float* part = static_cast<float*>(workspace);
        const TiledMap fm(fmap, fmap_layout, n_out, taps, s);
        const bf16* X = static_cast<const bf16*>(x_split);
        const bf16* DY = static_cast<const bf16*>(dy_split);
        switch (p.nb) {
            case 64: launch_dw<64>(p, fm.p, taps, n_out, X, C2, DY, Co2, part, s); break;
            case 128: launch_dw<128>(p, fm.p, taps, n_out, X, C2, DY, Co2, part, s); break;
            default: launch_dw<256>(p, fm.p, taps, n_out, X, C2, DY, Co2, part, s); break;
        }
        const long long total = (long long)c_out * c_in * taps;
        k_reduce_dw<<<grid_for(total, 32), 256, 0, s>>>(part, p.g, taps, c_in, c_out, dw_ref, c_in, c_out);
        launched("dW split reduction (split precision)");
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
            k_to_channel_major<float><<<g, b, 0, as_stream(stream)>>>(static_cast<const float*>(native), n, c, out, c);
        else
            k_to_channel_major<bf16><<<g, b, 0, as_stream(stream)>>>(static_cast<const bf16*>(native), n, c, out, c);
        launched("to channel-major");
    });
}

}  // extern "C"
