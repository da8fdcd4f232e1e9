// conv_tma.cu — gather-GEMM with TMA tile::gather4 producers (sm_100a).
//
// Same contract as k_gather_gemm in conv_tc.cu (Y[n] = sum_{t,ci} X[nbr(n,t)][ci] *
// W[co][t][ci]), but the operand ring is filled by the Tensor Memory Accelerator:
//   * A (gathered feature rows): one `cp.async.bulk.tensor.2d...tile::gather4` per 4
//     output voxels — the tensor map views X as a 2-D [N][C] bf16 tensor with a
//     1 x 64-element box and SWIZZLE_128B, so each instruction lands four 128-byte rows
//     in the UMMA canonical layout; empty cells (nbr = -1) are out-of-bounds rows and
//     TMA zero-fills them. 32 instructions per 16 KB stage instead of ~1,000 16-byte
//     cp.async from 256 threads.
//   * B (packed weights): one 2-D tiled TMA load per stage.
//   * the tile's field-map block: one 1-D bulk copy per tile, double-buffered.
// One producer warp, one MMA thread, one epilogue warpgroup; persistent over tiles,
// double-buffered TMEM accumulators. Requires C % 64 == 0 (one tap per 64-wide K
// block, the TMA box = one full 128-byte row).
#include <cuda.h>  // CUtensorMap / enums only; the encoder comes from cudaGetDriverEntryPoint
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "hc_internal.h"
#include "hc_launch.cuh"
#include "tc_common.cuh"

namespace hcb {

namespace {

using bf16 = __nv_bfloat16;
using namespace tc;

constexpr int BM = 128, BK = 64, kMaxTaps = 27;
constexpr int kNbrBytes = kMaxTaps * BM * 4;

__host__ __device__ constexpr int cols_pow2(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
    static EncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!p || q != cudaDriverEntryPointSuccess) throw cuda_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiled>(p);
    }
    return fn;
}

// 2-D bf16 tensor [rows][inner] (row pitch `pitch` bytes), box = box_rows x box_inner,
// 128-byte swizzle, zero fill out of bounds.
CUtensorMap map2d(const void* base, uint64_t inner, uint64_t rows, uint64_t pitch, uint32_t box_inner,
                  uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {pitch};
    const cuuint32_t box[2] = {box_inner, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                            int r3, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void store_row16(float* dst, const float (&v)[16]) {
#pragma unroll
    for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
}
__device__ __forceinline__ void store_row16(bf16* dst, const float (&v)[16]) {
    uint32_t p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        p[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(dst) = make_uint4(p[0], p[1], p[2], p[3]);
    *reinterpret_cast<uint4*>(dst + 8) = make_uint4(p[4], p[5], p[6], p[7]);
}

template <int BN>
struct TmaCfg {
    static constexpr int A_BYTES = BM * 128;
    static constexpr int B_BYTES = BN * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = std::min(8, (226 * 1024 - 1280 - 2 * kNbrBytes) / STAGE_BYTES);
    static constexpr int THREADS = 192;  // warp 0 TMA producer, warp 1 MMA, warps 2-5 epilogue
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 2 * kNbrBytes + 256;
};

template <int BN, typename OutT>
__global__ void __launch_bounds__(TmaCfg<BN>::THREADS, 1)
    k_gather_gemm_tma(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
                      const int* __restrict__ fmap, int taps, long long rows, int C, int Kp,
                      OutT* __restrict__ Y, int tiles) {
    using Cfg = TmaCfg<BN>;
    constexpr int S = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    int* nbr_s = reinterpret_cast<int*>(smem + S * Cfg::STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES + 2 * kNbrBytes);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 6);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nkb = Kp / BK;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
    const uint32_t tfull0 = smem_u32(bars + 2 * S), tempty0 = smem_u32(bars + 2 * S + 2);
    const uint32_t nfull0 = smem_u32(bars + 2 * S + 4);
    const uint32_t nbr_bytes = (uint32_t)(taps * BM * 4);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull0 + 8 * a, 1);
            mbar_init(tempty0 + 8 * a, 128);
            mbar_init(nfull0 + 8 * a, 1);
        }
        mbar_init_fence();
    }
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), cols_pow2(2 * BN));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer warp
        auto request = [&](int tile, int buf) {
            mbar_arrive_expect_tx(nfull0 + 8 * buf, nbr_bytes);
            bulk_g2s(smem_u32(nbr_s + buf * kMaxTaps * BM), fmap + (long long)tile * taps * BM, nbr_bytes,
                     nfull0 + 8 * buf);
        };
        if (lane == 0) {
            if (blockIdx.x < tiles) request(blockIdx.x, 0);
            if (blockIdx.x + gridDim.x < tiles) request(blockIdx.x + gridDim.x, 1);
        }
        long long it = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int buf = i & 1;
            mbar_wait(nfull0 + 8 * buf, (uint32_t)((i >> 1) & 1));
            const int* nb = nbr_s + buf * kMaxTaps * BM + 4 * lane;
            for (int kb = 0; kb < nkb; ++kb, ++it) {
                const int s = (int)(it % S);
                if (it >= S) mbar_wait(empty0 + 8 * s, (uint32_t)(((it / S) + 1) & 1));
                const uint32_t A = smem_u32(smem + s * Cfg::STAGE_BYTES);
                if (lane == 0) mbar_arrive_expect_tx(full0 + 8 * s, Cfg::STAGE_BYTES);
                __syncwarp();
                const int k0 = kb * BK;
                const int t = k0 / C, c0 = k0 - t * C;
                const int4 g = *reinterpret_cast<const int4*>(nb + t * BM);  // rows 4*lane .. 4*lane+3
                tma_gather4(A + 4 * lane * 128, &xmap, c0, g.x, g.y, g.z, g.w, full0 + 8 * s);
                if (lane == 0) tma_load2d(A + Cfg::A_BYTES, &wmap, k0, 0, full0 + 8 * s);
            }
            __syncwarp();  // every lane has issued this tile's gathers (coordinates are operands)
            if (lane == 0 && tile + 2 * (int)gridDim.x < tiles) request(tile + 2 * gridDim.x, buf);
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, false, false);
            long long it = 0;
            int i = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
                const int acc = i & 1;
                if (i >= 2) mbar_wait(tempty0 + 8 * acc, (uint32_t)(((i >> 1) - 1) & 1));
                tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = (int)(it % S);
                    mbar_wait(full0 + 8 * s, (uint32_t)((it / S) & 1));
                    tc_fence_after();
                    const uint32_t a = smem_u32(smem + s * Cfg::STAGE_BYTES);
                    const uint32_t b = a + Cfg::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        mma_bf16(d, sw128_desc(a + kk * 32, 16, 1024), sw128_desc(b + kk * 32, 16, 1024), idesc,
                                 (kb | kk) != 0);
                    mma_commit(empty0 + 8 * s);
                }
                mma_commit(tfull0 + 8 * acc);
            }
        }
    } else {
        // ---------------- epilogue warpgroup (warps 2-5 -> TMEM lane quadrants 2,3,0,1)
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int acc = i & 1;
            mbar_wait(tfull0 + 8 * acc, (uint32_t)((i >> 1) & 1));
            tc_fence_after();
            const long long m = (long long)tile * BM + row;
#pragma unroll
            for (int c0 = 0; c0 < BN; c0 += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c0, v);
                tmem_ld_wait();
                float f[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]);
                if (m < rows) store_row16(Y + m * BN + c0, f);
            }
            tc_fence_before();
            mbar_arrive(tempty0 + 8 * acc);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, cols_pow2(2 * BN));
    }
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

template <int BN, typename OutT>
void launch(const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, OutT* Y,
            cudaStream_t s) {
    using Cfg = TmaCfg<BN>;
    auto kern = k_gather_gemm_tma<BN, OutT>;
    static bool attr = false;
    if (!attr) {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM), "smem attr");
        attr = true;
    }
    // The row extent of X is not part of the gather-GEMM contract (the field map only
    // holds valid columns or -1); -1 rows are out of bounds on the low side -> zeros.
    const CUtensorMap xm = map2d(X, (uint64_t)C, 0x7FFFFFFFull, (uint64_t)C * 2, BK, 1);
    const CUtensorMap wm = map2d(Wp, (uint64_t)Kp, (uint64_t)BN, (uint64_t)Kp * 2, BK, BN);
    const int tiles = (int)((rows + BM - 1) / BM);
    const int grid = std::min(tiles, sm_count());
    kern<<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(xm, wm, fmap, taps, rows, C, Kp, Y, tiles);
    launched("conv gather-GEMM (tcgen05, TMA gather4)");
}

}  // namespace

// Entry used by conv_tc.cu's dispatch: tile-major map, C % 64 == 0, N in {64,128,256}.
bool gather_gemm_tma_supported(int C, int N) {
    static int env = -1;
    if (env < 0) {
        // Off by default: correct, but on B200 the per-SM TMA unit serves 128-byte gather4
        // rows ~2.9x slower than 8 warps of 16-byte cp.async (C=64: 3.29 vs 1.14 ms,
        // profiles/ROUND1.md). HCB_FWD_TMA=1 selects it.
        const char* e = std::getenv("HCB_FWD_TMA");
        env = e ? (std::atoi(e) != 0) : 0;
    }
    return env && C % 64 == 0 && (N == 64 || N == 128 || N == 256);
}

template <typename OutT>
void gather_gemm_tma(const int* fmap, int taps, long long rows, const bf16* X, int C, const bf16* Wp, int Kp, int N,
                     OutT* Y, cudaStream_t s) {
    switch (N) {
        case 64: launch<64>(fmap, taps, rows, X, C, Wp, Kp, Y, s); break;
        case 128: launch<128>(fmap, taps, rows, X, C, Wp, Kp, Y, s); break;
        default: launch<256>(fmap, taps, rows, X, C, Wp, Kp, Y, s); break;
    }
}
template void gather_gemm_tma<float>(const int*, int, long long, const bf16*, int, const bf16*, int, int, float*,
                                     cudaStream_t);
template void gather_gemm_tma<bf16>(const int*, int, long long, const bf16*, int, const bf16*, int, int, bf16*,
                                    cudaStream_t);

}  // namespace hcb
