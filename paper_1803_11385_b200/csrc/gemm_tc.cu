// gemm_tc.cu — the reference-layout contraction on 5th-gen tensor cores: conv_forward's
// matmul, conv_backward's matmul_trans_b (dW) and matmul_trans_a (column gradient)
// (gemm.cpp:14-69, cnn_ops.cpp:206-232) over the MATERIALISED fp32 column matrix, as
// tcgen05.mma kind::tf32 with both operands staged by 2-D TMA straight from the row-major
// fp32 matrices (no layout pass, no conversion pass in HBM).
//
// Every product is computed as tiles of C^T: the MMA's M (128 TMEM lanes) runs along C's
// contiguous column index (voxels, or column-matrix rows for dW), the MMA's N (BN <= 64)
// along C's rows (output channels), so the epilogue's tcgen05.ld registers go out as
// 128-byte coalesced stores (32 consecutive floats per warp instruction):
//
//   nn  C[ra][cb] = A[ra][K] * B[K][cb]     MMA-A <- B (MN-major)  MMA-B <- A (K-major)
//   nt  C[ra][cb] = A[ra][K] * B[cb][K]^T   MMA-A <- B (K-major)   MMA-B <- A (K-major)
//   tn  C[ra][cb] = A[K][ra]^T * B[K][cb]   MMA-A <- B (MN-major)  MMA-B <- A (MN-major)
//
// Precision. HC_MATH_FAST runs 3xTF32: with hi = x with the low 13 mantissa bits cleared
// (exact in tf32) and lo = x - hi (exact in fp32, |lo| < 2^-10 |x|), D += lo_a*hi_b +
// hi_a*lo_b + hi_a*hi_b keeps the fp32 bar of the FFMA path (<= 1e-5 normwise vs double;
// the dropped lo*lo term is ~2^-20 relative). The B200 tensor core reads an fp32 operand
// as tf32 by TRUNCATION (measured: products of raw and of explicitly truncated operands are
// bit-identical, pinned by tests/test_gemm_tc.py), so the raw TMA tile already is hi and
// only lo is written (a second shared-memory tile); -DHCB_TF32_EXPLICIT_HI writes hi too.
// HC_MATH_TF32 is the single-pass product (~1e-3). (Rejected: splitting small operands
// once in HBM and loading their lo planes by TMA — slower for matmul_trans_a at C >= 64.)
//
// Warp roles (192 threads): warp 0 TMA, warp 1 MMA issue (elect.sync), warps 2-5 split
// the tiles (3xTF32) and drain TMEM in the epilogue. The long-K product (dW, K = voxels)
// is split over CTAs; partials are reduced in a fixed order -> deterministic.
// Eligibility: 16-byte aligned bases and row pitches (inner dimensions % 4 == 0); other
// shapes take the FFMA kernels (gemm_fast.cu).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "hc_internal.h"
#include "hc_launch.cuh"
#include "tc_common.cuh"
#include "tma_host.h"

namespace hcb {
namespace {

using namespace tc;

constexpr int BM = 128;         // C columns per tile (TMEM lanes)
constexpr int BKF = 32;         // fp32 K elements per stage = one 128-byte swizzle row
#ifndef HCB_GEMM_EW
#define HCB_GEMM_EW 4  // A/B: 8 warps measured slower (fwd 3.33 -> 3.53 ms at C=64)
#endif
constexpr int kEW = HCB_GEMM_EW;           // split / epilogue warps (4 or 8)
constexpr int kEpi = kEW * 32;             // their threads
constexpr int kThreads = 64 + kEpi;        // + TMA warp + MMA warp
constexpr int kBlk = 8;         // stages (8 x 32 = 256 K) per TMEM accumulation block

template <int BN, int SPLIT>
struct GCfg {
    static constexpr int A_BYTES = BM * 128;
    static constexpr int B_BYTES = BN * 128;
    static constexpr int RAW = A_BYTES + B_BYTES;
    static constexpr int STAGE = RAW * (SPLIT >= 3 ? 2 : 1);  // raw (= hi) + lo
    // SPLIT 5: only the A tile is split in shared memory; B's lo plane arrives by TMA
    static constexpr int CVT = SPLIT == 5 ? A_BYTES : RAW;        // bytes the split warps convert
    static constexpr int TX = SPLIT == 5 ? RAW + B_BYTES : RAW;   // TMA bytes per stage
    // two CTAs per SM when two rings of >= 2 stages fit, else one CTA with a deeper ring
    static constexpr int BUDGET = 2 * STAGE <= 104 * 1024 ? 104 * 1024 : 200 * 1024;
    static constexpr int S = BUDGET / STAGE < 8 ? BUDGET / STAGE : 8;
    static constexpr int SMEM = S * STAGE + 1024;
    static constexpr int CTAS = BUDGET == 104 * 1024 ? 2 : 1;  // resident per SM
    static_assert(S >= 2, "ring too shallow");
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void split_tf32(uint32_t x, uint32_t& hi, uint32_t& lo) {
    hi = x & 0xFFFFE000u;
    lo = __float_as_uint(__fsub_rn(__uint_as_float(x), __uint_as_float(hi)));
}

// Tile t of the grid-stride loop: n-tile fastest (the CTAs working at the same time share
// the MMA-A operand — e.g. dY's voxel block in matmul_trans_a — through L2), then m-tile,
// then K split.
struct Tile {
    long long m0, n0, kb, z;  // kb: first 32-wide K block
    int nk;
};
__device__ __forceinline__ Tile tile_at(long long t, long long tiles_n, long long tiles_m, int BN, long long K,
                                        long long k_chunk) {
    Tile r;
    const long long ny = t % tiles_n, mx = (t / tiles_n) % tiles_m;
    r.z = t / (tiles_n * tiles_m);
    r.m0 = mx * BM;
    r.n0 = ny * BN;
    // K splits are interleaved: split z takes 32-wide K blocks z, z + splits, ... so the
    // splits running side by side read adjacent 128-byte segments of the same rows (DRAM
    // page locality for the long-K product); k_chunk = number of splits
    const long long nb = (K + BKF - 1) / BKF;
    r.kb = r.z;
    r.nk = (int)((nb - r.z + k_chunk - 1) / k_chunk);
    return r;
}

// Persistent: each CTA walks tiles t = blockIdx.x, +gridDim.x, ...; the stage ring, the
// stage phases and the two TMEM accumulation buffers run on across tiles, so a tile's
// epilogue overlaps the next tile's loads and MMAs.
template <bool AMN, bool BMN, int BN, int SPLIT>
__global__ void __launch_bounds__(kThreads, GCfg<BN, SPLIT>::CTAS) k_gemm_tf32(const __grid_constant__ CUtensorMap amap,
                                                        const __grid_constant__ CUtensorMap bmap,
                                                        const __grid_constant__ CUtensorMap blomap,
                                                        float* __restrict__ C, long long ra, long long cb, long long K,
                                                        long long k_chunk, long long split_stride, long long tiles_n,
                                                        long long tiles_m, long long ntiles) {
    using Cfg = GCfg<BN, SPLIT>;
    constexpr int S = Cfg::S;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[3 * S + 4];
    __shared__ uint32_t tmem_slot;
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t full0 = smem_u32(&bars[0]), cvt0 = smem_u32(&bars[S]), empty0 = smem_u32(&bars[2 * S]),
                   tfull0 = smem_u32(&bars[3 * S]), tempty0 = smem_u32(&bars[3 * S + 2]);
    const int warp = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(cvt0 + 8 * s, kEpi);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            mbar_init(tempty0 + 8 * b, kEpi);
        }
        mbar_init_fence();
    }
    if (warp == 1) tmem_alloc(smem_u32(&tmem_slot), 2 * BN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane_id() == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const Tile T = tile_at(t, tiles_n, tiles_m, BN, K, k_chunk);
                for (int i = 0; i < T.nk; ++i) {
                    mbar_wait(empty0 + 8 * s, ph ^ 1);
                    mbar_arrive_expect_tx(full0 + 8 * s, Cfg::TX);
                    const int k0 = (int)((T.kb + (long long)i * k_chunk) * BKF);
                    const uint32_t a = sbase + s * Cfg::STAGE, b = a + Cfg::A_BYTES;
                    if (AMN) {
#pragma unroll
                        for (int j = 0; j < BM / 32; ++j)
                            tma_load2d(a + j * 4096, &amap, (int)T.m0 + 32 * j, k0, full0 + 8 * s);
                    } else {
                        tma_load2d(a, &amap, k0, (int)T.m0, full0 + 8 * s);
                    }
                    if (BMN) {
#pragma unroll
                        for (int j = 0; j < BN / 32; ++j)
                            tma_load2d(b + j * 4096, &bmap, (int)T.n0 + 32 * j, k0, full0 + 8 * s);
                    } else {
                        tma_load2d(b, &bmap, k0, (int)T.n0, full0 + 8 * s);
                    }
                    if constexpr (SPLIT == 5) {  // B's pre-split lo plane into the lo region
                        static_assert(!BMN, "SPLIT 5 is for a K-major B operand");
                        tma_load2d(b + Cfg::RAW, &blomap, k0, (int)T.n0, full0 + 8 * s);
                    }
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = idesc_tf32_f32(BM, BN, AMN, BMN);
        // K-major (SWIZZLE_128B): one 128-byte row per M/N element, 8-row atoms (SBO 1 KB),
        // K step 32 B. MN-major (SWIZZLE_128B_BASE32B, the only MN-major form for tf32): 32
        // M/N elements per 128-byte row, one row per k, 4-row atoms (SBO 512 B), 32-wide M/N
        // blocks 4 KB apart (LBO), K step 8 rows = 1 KB.
        constexpr uint32_t A_STEP = AMN ? 64 : 2, B_STEP = BMN ? 64 : 2;  // 16-byte units per MMA
        const uint64_t ad = AMN ? sw128b32_desc(sbase, 4096, 512) : sw128_desc(sbase, 16, 1024);
        const uint64_t bd = BMN ? sw128b32_desc(sbase + Cfg::A_BYTES, 4096, 512)
                                : sw128_desc(sbase + Cfg::A_BYTES, 16, 1024);
        constexpr uint64_t LO = Cfg::RAW >> 4;
        int s = 0, blk = -1;
        uint32_t ph = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const Tile T = tile_at(t, tiles_n, tiles_m, BN, K, k_chunk);
            int in_blk = 0;
            for (int i = 0; i < T.nk; ++i) {
                if (in_blk == 0) {
                    ++blk;
                    if (blk >= 2) mbar_wait(tempty0 + 8 * (blk & 1), ((blk >> 1) - 1) & 1);  // drained
                }
                const int buf = blk & 1;
                mbar_wait(SPLIT >= 3 ? cvt0 + 8 * s : full0 + 8 * s, ph);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t d = tmem + buf * BN;
                    const uint64_t so = (uint64_t)((s * Cfg::STAGE) >> 4);
#pragma unroll
                    for (int kk = 0; kk < BKF / 8; ++kk) {
                        const uint64_t a = ad + so + A_STEP * kk, b = bd + so + B_STEP * kk;
                        if (SPLIT >= 3) {
                            mma_tf32(d, a + LO, b, idesc, (in_blk | kk) != 0);  // lo_a * hi_b
                            mma_tf32(d, a, b + LO, idesc, 1);                   // hi_a * lo_b
                            mma_tf32(d, a, b, idesc, 1);                        // hi_a * hi_b
                        } else {
                            mma_tf32(d, a, b, idesc, (in_blk | kk) != 0);
                        }
                    }
                    mma_commit(empty0 + 8 * s);
                    if (in_blk == kBlk - 1 || i == T.nk - 1) mma_commit(tfull0 + 8 * buf);
                }
                __syncwarp();
                if (++s == S) {
                    s = 0;
                    ph ^= 1;
                }
                if (++in_blk == kBlk) in_blk = 0;
            }
        }
    } else {
        // ---------------- split (3xTF32) + epilogue warps
        // Two-level accumulation: the tensor core sums kBlk stages (256 K) into one of two TMEM
        // buffers, these warps add each finished block into fp32 registers with IEEE adds
        // (the tensor core's internal fp32 accumulation is not round-to-nearest; long chains
        // in TMEM alone miss the 1e-5 bar at K >= ~2000).
        const int t_id = threadIdx.x - 64;
        const int q = warp & 3;  // TMEM lane quadrant this warp may read
        // with 8 warps two share a quadrant and split the accumulator's columns
        constexpr int BNW = BN * 4 / kEW;
        const int cw = ((warp - 2) / 4) * BNW;
        float acc[BNW];
#pragma unroll
        for (int j = 0; j < BNW; ++j) acc[j] = 0.0f;
        // drain global block b; `last`: the final block of tile T -> store and reset
        auto drain = [&](int b, const Tile& T, bool last) {
            const int buf = b & 1;
            mbar_wait(tfull0 + 8 * buf, (b >> 1) & 1);  // spin: the MMA warp needs this buffer back soon
            tc_fence_after();
#pragma unroll
            for (int c0 = 0; c0 < BNW; c0 += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + buf * BN + cw + c0, v);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[c0 + j] = __fadd_rn(acc[c0 + j], __uint_as_float(v[j]));
            }
            tc_fence_before();
            mbar_arrive(tempty0 + 8 * buf);
            if (last) {
                const long long m = T.m0 + q * 32 + lane_id();
                if (m < cb) {
                    float* p = C + T.z * split_stride + (T.n0 + cw) * cb + m;
                    const int rows = (int)min((long long)BNW, ra - T.n0 - cw);
#pragma unroll
                    for (int j = 0; j < BNW; ++j) {
                        if (j < rows) __stcs(p, acc[j]);  // streaming: the output is not re-read here
                        p += cb;
                        asm volatile("" : "+l"(p));  // keep the address chain sequential (no 64 live pointers)
                    }
                }
#pragma unroll
                for (int j = 0; j < BNW; ++j) acc[j] = 0.0f;
            }
        };
        int blk = -1;
        if constexpr (SPLIT >= 3) {
            // convert stage by stage; once the first stage of block b+1 is converted, drain
            // block b (the MMA warp can finish b without more conversions). One drain call
            // site, so the BN-float accumulator is inlined once.
            int s = 0;
            uint32_t ph = 0;
            Tile prevT{}, curT{};
            bool prev_last = false, cur_last = false;
            long long t = blockIdx.x;
            Tile T{};
            if (t < ntiles) T = tile_at(t, tiles_n, tiles_m, BN, K, k_chunk);
            int i = 0;
            for (;;) {
                const bool have = t < ntiles;
                int dblk = -1;
                bool dlast = false;
                Tile dT{};
                if (have) {
                    const bool starts = (i % kBlk) == 0;
                    if (starts) {
                        prevT = curT;
                        prev_last = cur_last;
                        curT = T;
                        cur_last = i + kBlk >= T.nk;
                        ++blk;
                    }
                    mbar_wait(full0 + 8 * s, ph);
                    const uint32_t raw = sbase + s * Cfg::STAGE;
#pragma unroll 4
                    for (int e = t_id; e < Cfg::CVT / 16; e += kEpi) {
                        const int4 v = ld_shared_v4(raw + 16 * e);
                        uint4 h, l;
                        split_tf32((uint32_t)v.x, h.x, l.x);
                        split_tf32((uint32_t)v.y, h.y, l.y);
                        split_tf32((uint32_t)v.z, h.z, l.z);
                        split_tf32((uint32_t)v.w, h.w, l.w);
#ifdef HCB_TF32_EXPLICIT_HI
                        st_shared_v4(raw + 16 * e, h);
#endif
                        st_shared_v4(raw + Cfg::RAW + 16 * e, l);
                    }
                    fence_proxy_async();
                    mbar_arrive(cvt0 + 8 * s);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                    if (starts && blk >= 1) {
                        dblk = blk - 1;
                        dT = prevT;
                        dlast = prev_last;
                    }
                    if (++i == T.nk) {
                        i = 0;
                        t += gridDim.x;
                        if (t < ntiles) T = tile_at(t, tiles_n, tiles_m, BN, K, k_chunk);
                    }
                } else if (blk >= 0) {
                    dblk = blk;
                    dT = curT;
                    dlast = cur_last;
                }
                if (dblk >= 0) drain(dblk, dT, dlast);
                if (!have) break;
            }
        } else {
            for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const Tile T = tile_at(t, tiles_n, tiles_m, BN, K, k_chunk);
                for (int i = 0; i < T.nk; i += kBlk) drain(++blk, T, i + kBlk >= T.nk);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 2 * BN);
    }
}

// fixed-order reduction of split partials: c = sum_z P[z] (z ascending)
__global__ void k_reduce_splits4(const float4* __restrict__ P, float4* __restrict__ Cout, long long n4, int splits) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n4) return;
    float4 s = P[i];
    for (int z = 1; z < splits; ++z) {
        const float4 p = P[(long long)z * n4 + i];
        s.x += p.x;
        s.y += p.y;
        s.z += p.z;
        s.w += p.w;
    }
    Cout[i] = s;
}

// fp32 row-major [outer][inner], box = box_outer x box_inner (box_inner * 4 = 128 B), SWIZZLE_128B
// (K-major operands) or SWIZZLE_128B_ATOM_32B (MN-major operands), out-of-bounds elements read as zero.
CUtensorMap fmap2d(const float* base, long long inner, long long outer, uint32_t box_inner, uint32_t box_outer,
                   bool mn_major) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    const cuuint64_t strides[1] = {(cuuint64_t)inner * 4};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = tma_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled (fp32) failed (" + std::to_string((int)r) + ")");
    return m;
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "sm count");
    }
    return n;
}

// opB: MMA-B source. MN-major: X[K][ra] (inner = ra), K-major: X[ra][K] (inner = K).
// opA: MMA-A source. MN-major: X[K][cb] (inner = cb), K-major: X[cb][K] (inner = K).
template <bool AMN, bool BMN, int BN, int SPLIT>
void launch(const float* asrc, const float* bsrc, float* C, long long ra, long long cb, long long K, cudaStream_t s,
            const float* blo = nullptr) {
    using Cfg = GCfg<BN, SPLIT>;
    auto kern = k_gemm_tf32<AMN, BMN, BN, SPLIT>;
    smem_optin(kern, Cfg::SMEM);
    const CUtensorMap am = AMN ? fmap2d(asrc, cb, K, 32, 32, true) : fmap2d(asrc, K, cb, 32, BM, false);
    const CUtensorMap bm = BMN ? fmap2d(bsrc, ra, K, 32, 32, true) : fmap2d(bsrc, K, ra, 32, BN, false);
    const CUtensorMap blm = SPLIT == 5 ? fmap2d(blo, K, ra, 32, BN, false) : bm;
    const long long tiles_m = (cb + BM - 1) / BM, tiles_n = (ra + BN - 1) / BN, tiles = tiles_m * tiles_n;
    const long long slots = (long long)Cfg::CTAS * sm_count();
    // long-K products with few output tiles (dW: K = voxels): split K over CTAs to fill one
    // wave exactly (no straggler wave); each split keeps >= 2048 K
    long long splits = 1;
    if (tiles < slots) splits = std::max<long long>(1, std::min<long long>(slots / tiles, K / 2048));
    const long long chunk = (K + splits - 1) / splits;  // K per split (interleaved 32-wide blocks)
    const long long ntiles = tiles * splits;
    // long tiles (K >= 512): one CTA per tile, the hardware scheduler balances them; short
    // tiles (matmul_trans_a, K = C_out): persistent CTAs, so per-CTA setup (barriers, TMEM
    // allocation) is paid once and a tile's epilogue overlaps the next tile's loads
    static const int persist = [] {
        const char* e = std::getenv("HCB_TC_PERSIST");  // A/B: 1 always, 0 never
        return e ? std::atoi(e) : -1;
    }();
    const bool long_tiles = chunk >= 512;
    const bool use_persist = persist == 1 || (persist != 0 && !long_tiles);
    const unsigned grid = (unsigned)(use_persist ? std::min<long long>(ntiles, slots) : ntiles);
    if (splits == 1) {
        kern<<<grid, kThreads, Cfg::SMEM, s>>>(am, bm, blm, C, ra, cb, K, splits, 0, tiles_n, tiles_m, ntiles);
        launched("gemm (tcgen05 tf32)");
        return;
    }
    const long long mn = ra * cb;  // % 4 == 0: cb % 4 == 0 by eligibility
    Scratch part(sizeof(float) * mn * splits, s);
    kern<<<grid, kThreads, Cfg::SMEM, s>>>(am, bm, blm, part.as<float>(), ra, cb, K, splits, mn, tiles_n, tiles_m,
                                           ntiles);
    k_reduce_splits4<<<grid_for(mn / 4, 256), 256, 0, s>>>(part.as<const float4>(), reinterpret_cast<float4*>(C),
                                                          mn / 4, (int)splits);
    launched("gemm (tcgen05 tf32, split-K)", 2);
}

// lo = x - tf32_trunc(x) elementwise (the small operand's pre-split plane for SPLIT 5)
__global__ void k_tf32_lo(const uint4* __restrict__ x, uint4* __restrict__ lo, long long n4) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n4) return;
    const uint4 v = x[i];
    uint4 h, l;
    split_tf32(v.x, h.x, l.x);
    split_tf32(v.y, h.y, l.y);
    split_tf32(v.z, h.z, l.z);
    split_tf32(v.w, h.w, l.w);
    lo[i] = l;
}

template <bool AMN, bool BMN>
void dispatch(const float* asrc, const float* bsrc, float* C, long long ra, long long cb, long long K, bool three,
              cudaStream_t s) {
    static const int presplit = [] {
        const char* e = std::getenv("HCB_TC_PRESPLIT_B");  // A/B: 0 splits B in shared memory too
        return e ? std::atoi(e) : 1;
    }();
    // matmul (conv forward): B = the weights, tiny next to the column matrix -> split it once
    // in HBM and stream its lo plane by TMA; the split warps then only convert A
    if constexpr (AMN && !BMN) {
        if (three && presplit && ra > 32) {
            const long long n = ra * K;  // K % 4 == 0 by eligibility
            Scratch lo(sizeof(float) * n, s);
            k_tf32_lo<<<grid_for(n / 4, 256), 256, 0, s>>>(reinterpret_cast<const uint4*>(bsrc), lo.as<uint4>(), n / 4);
            launched("tf32 lo plane (weights)");
            return launch<AMN, BMN, 64, 5>(asrc, bsrc, C, ra, cb, K, s, lo.as<float>());
        }
    }
    if (ra <= 32) {
        if (three) return launch<AMN, BMN, 32, 3>(asrc, bsrc, C, ra, cb, K, s);
        return launch<AMN, BMN, 32, 1>(asrc, bsrc, C, ra, cb, K, s);
    }
    // BN <= 64: the epilogue's fp32 register accumulator is BN floats per thread; wider C row
    // ranges are more n-tiles (consecutive CTAs, so their shared MMA-A tile stays in L2)
    if (three) return launch<AMN, BMN, 64, 3>(asrc, bsrc, C, ra, cb, K, s);
    launch<AMN, BMN, 64, 1>(asrc, bsrc, C, ra, cb, K, s);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

bool enabled() {
    static const int on = [] {
        const char* e = std::getenv("HCB_TC_GEMM");  // A/B: 0 forces the FFMA kernels
        return e ? std::atoi(e) : 1;
    }();
    return on != 0;
}

constexpr long long kMaxCoord = 1LL << 31;  // TMA coordinates are int32

}  // namespace

// Each returns false (nothing enqueued) when the shape is not TMA-eligible; the caller then
// uses the FFMA kernels. ra / cb / k as in gemm_fast.cu.

// matmul: c[ra x cb] = a[ra x k] * b[k x cb]
bool tc_gemm_nn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, bool three,
                cudaStream_t s) {
    if (!enabled() || ra <= 0 || cb <= 0 || k <= 0 || k % 4 || cb % 4 || !aligned16(a) || !aligned16(b) ||
        !aligned16(c) || cb >= kMaxCoord || k >= kMaxCoord || ra >= kMaxCoord)
        return false;
    dispatch<true, false>(b, a, c, ra, cb, k, three, s);
    return true;
}
// matmul_trans_a: c[k x cb] = a[ra x k]^T * b[ra x cb]   (contraction over ra)
bool tc_gemm_tn(const float* a, const float* b, float* c, long long ra, long long k, long long cb, bool three,
                cudaStream_t s) {
    if (!enabled() || ra <= 0 || cb <= 0 || k <= 0 || k % 4 || cb % 4 || !aligned16(a) || !aligned16(b) ||
        !aligned16(c) || cb >= kMaxCoord || k >= kMaxCoord || ra >= kMaxCoord)
        return false;
    dispatch<true, true>(b, a, c, k, cb, ra, three, s);
    return true;
}
// matmul_trans_b: c[ra x rb] = a[ra x k] * b[rb x k]^T
bool tc_gemm_nt(const float* a, const float* b, float* c, long long ra, long long k, long long rb, bool three,
                cudaStream_t s) {
    if (!enabled() || ra <= 0 || rb <= 0 || k <= 0 || k % 4 || rb % 4 || !aligned16(a) || !aligned16(b) ||
        !aligned16(c) || rb >= kMaxCoord || k >= kMaxCoord || ra >= kMaxCoord)
        return false;
    dispatch<false, false>(b, a, c, ra, rb, k, three, s);
    return true;
}

}  // namespace hcb
