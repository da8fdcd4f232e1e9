// conv_tc.cu — the native (voxel-major) fused hash-conv on 5th-gen tensor cores.
//
// Implicit GEMM: the hash2col column matrix is never materialised. For output
// voxel n and field row t the field map (K0, ops_ref.cu) gives the input column
// nbr(n,t) (or -1); the A operand is gathered straight from the voxel-major
// feature rows X[nbr][:] into shared memory with 16-byte cp.async (zero-fill for
// empty cells), laid out in the UMMA SWIZZLE_128B canonical form, and
// tcgen05.mma accumulates in TMEM.
//
//   forward        Y [n][co]  = sum_{t,ci} X[nbr(n,t)][ci] * W[co][t][ci]
//   backward-data  dX[g][ci]  = sum_{t,co} dY[nbr(g,t)][co] * W[co][26-t][ci]
//                  (stride 1: the same kernel with flipped/transposed weights;
//                   cnn_ops.cpp:217-232 computes col2hash(W^T dY), the same sum)
//   weight grad    dW[co][t][ci] = sum_n dY[n][co] * X[nbr(n,t)][ci]
//                  (reduction over voxels: split-K over CTAs, partials reduced in a
//                   fixed order -> deterministic; both operands MN-major)
//
// Forward kernel: persistent, warp-specialised — 4 producer warps stream the
// gathered operand ring continuously across tiles (field-map entries are
// prefetched into registers two stages ahead, so no dependent load sits on the
// issue path), one elected thread issues tcgen05.mma, and a separate epilogue
// warpgroup drains double-buffered TMEM accumulators while the next tile's MMAs
// run.
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

// conv_tma.cu: the TMA tile::gather4 variant of the forward gather-GEMM
bool gather_gemm_tma_supported(int C, int N);
template <typename OutT>
void gather_gemm_tma(const int* fmap, int taps, long long rows, const __nv_bfloat16* X, int C,
                     const __nv_bfloat16* Wp, int Kp, int N, OutT* Y, cudaStream_t s);

namespace {

using bf16 = __nv_bfloat16;
using namespace tc;

constexpr int BM = 128;          // voxels (GEMM M) per tile
constexpr int BK = 64;           // K elements (bf16) per pipeline stage = one 128 B row
constexpr int kProducers = 128;  // warps 0-3

__host__ __device__ constexpr int tmem_cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }

// Field map access: element (n, t) at p[n*sn + t*st] (row-major [N][taps] or tap-major [taps][N]).
// Layouts: 0 row-major [N][taps], 1 tap-major [taps][N], 2 tile-major [N/128][taps][128].
struct FMap {
    const int* p;
    long long sn, st;
    int tiled, taps;
};
__device__ __forceinline__ int fm_ld(const FMap& f, long long n, int t) {
    if (f.tiled) return __ldg(f.p + ((n >> 7) * f.taps + t) * 128 + (n & 127));
    return __ldg(f.p + n * f.sn + (long long)t * f.st);
}

// Producers signal stage completion with cp.async.mbarrier.arrive.noinc (non-blocking)
// instead of wait_group + arrive. HCB_ASYNC_ARRIVE=0 selects the blocking form (A/B).
int async_arrive() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("HCB_ASYNC_ARRIVE");
        v = e ? (std::atoi(e) != 0) : 1;
    }
    return v;
}

// Producer warps of the bulk-staged forward kernel (8, or 4 with HCB_FWD_PW=4).
int fwd_pw() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("HCB_FWD_PW");
        v = (e && std::atoi(e) == 4) ? 4 : 8;
    }
    return v;
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

// ====================================================================== gather-GEMM (persistent)
// CPS = resident CTAs per SM: 2 (4-stage rings, twice the producer warps per SM)
// or 1 (one deep ring). Both fit ~200 KB of shared memory per SM.
// TILED: the field map is tile-major and each tile's 27x128 map block is brought into
// a double-buffered shared-memory slot by one bulk copy a tile ahead.
constexpr int kMaxTaps = 27;
constexpr int kNbrBytes = kMaxTaps * BM * 4;  // 13.5 KB per buffer

template <int BN, int CPS, bool TILED, int PW = 4>
struct FwdCfg {
    static constexpr int A_BYTES = BM * 128;      // 16 KB
    static constexpr int B_BYTES = BN * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int BUDGET = (CPS == 2 ? 113 : 226) * 1024 - 1280;
    static constexpr int NBR = TILED ? 2 * kNbrBytes : 0;
    static constexpr int STAGES = (BUDGET - NBR) / STAGE_BYTES;
    static constexpr int LAG = STAGES - 1;        // cp.async groups kept in flight per producer
    static constexpr int PRODUCERS = PW * 32;     // producer warps 0..PW-1
    static constexpr int THREADS = PW * 32 + 160;  // + epilogue warps PW..PW+3, MMA warp PW+4
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + NBR + 256;
};

// Y[m][0:BN] = sum_k A[m][k] * Wp[0:BN][k],  A[m][k] = X[nbr(m, k / C)][k % C] (0 if -1)
template <int BN, int CPS, bool TILED, typename OutT, int PW = 4>
__global__ void __launch_bounds__(FwdCfg<BN, CPS, TILED, PW>::THREADS, CPS)
    k_gather_gemm(FMap fm, long long rows, const bf16* __restrict__ X, int C, int K, const bf16* __restrict__ Wp,
                  int Kp, OutT* __restrict__ Y, int tiles, int async_arrive) {
    using Cfg = FwdCfg<BN, CPS, TILED, PW>;
    constexpr int NP = Cfg::PRODUCERS;
    static_assert(TILED || PW == 4, "the register-prefetch producer is written for 4 warps");
    static_assert(PW % 4 == 0, "epilogue warps must start on a TMEM lane-quadrant boundary");
    constexpr int RS = NP / 8;  // row stride between a producer thread's rows
    constexpr int S = Cfg::STAGES;
    constexpr int LAG = Cfg::LAG;
    static_assert(S >= 2, "ring too shallow");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    int* nbr_s = reinterpret_cast<int*>(smem + S * Cfg::STAGE_BYTES);  // [2][taps][128] when TILED
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES + Cfg::NBR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 6);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int nkb = Kp / BK;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
    const uint32_t tfull0 = smem_u32(bars + 2 * S), tempty0 = smem_u32(bars + 2 * S + 2);
    const uint32_t nfull0 = smem_u32(bars + 2 * S + 4);
    const int taps = fm.taps;
    const uint32_t nbr_bytes = (uint32_t)(taps * BM * 4);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, NP);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull0 + 8 * a, 1);
            mbar_init(tempty0 + 8 * a, 128);
            mbar_init(nfull0 + 8 * a, 1);
        }
        mbar_init_fence();
    }
    if (warp == PW + 4) tmem_alloc(smem_u32(tmem_slot), tmem_cols(2 * BN));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (TILED && warp < PW) {
        // ---------------- producers (tile-major map, staged by bulk copies)
        const int c = tid & 7;    // 16-byte chunk within a 128-byte row
        const int r0 = tid >> 3;  // rows r0 + RS*j
        auto request = [&](int tile, int buf) {
            mbar_arrive_expect_tx(nfull0 + 8 * buf, nbr_bytes);
            bulk_g2s(smem_u32(nbr_s + buf * kMaxTaps * BM), fm.p + (long long)tile * taps * BM, nbr_bytes,
                     nfull0 + 8 * buf);
        };
        if (tid == 0) {
            if (blockIdx.x < tiles) request(blockIdx.x, 0);
            if (blockIdx.x + gridDim.x < tiles) request(blockIdx.x + gridDim.x, 1);
        }
        long long it = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
            const int buf = i & 1;
            mbar_wait(nfull0 + 8 * buf, (uint32_t)((i >> 1) & 1));
            const int* nb = nbr_s + buf * kMaxTaps * BM;
            for (int kb = 0; kb < nkb; ++kb, ++it) {
                const int s = (int)(it % S);
                if (it >= S) mbar_wait(empty0 + 8 * s, (uint32_t)(((it / S) + 1) & 1));
                uint8_t* A = smem + s * Cfg::STAGE_BYTES;
                uint8_t* B = A + Cfg::A_BYTES;
                const int k = kb * BK + c * 8;
                const bool kin = k < K;
                const int t = kin ? k / C : 0;
                const int ci = kin ? k - t * C : 0;
                const int* nbt = nb + t * BM;
#pragma unroll
                for (int j = 0; j < BM / RS; ++j) {
                    const int r = r0 + RS * j;
                    const int g = kin ? nbt[r] : -1;
                    const bf16* src = g >= 0 ? X + (long long)g * C + ci : X;
                    cp_async16(smem_u32(A + sw128_offset(r, c)), src, g >= 0 ? 16u : 0u);
                }
#pragma unroll
                for (int j = 0; j < (BN + RS - 1) / RS; ++j) {
                    const int r = r0 + RS * j;
                    if (r < BN)
                        cp_async16(smem_u32(B + sw128_offset(r, c)), Wp + (long long)r * Kp + kb * BK + c * 8, 16u);
                }
                if (async_arrive) {
                    cp_async_arrive_noinc(full0 + 8 * s);  // non-blocking: barrier completes on landing
                } else {
                    cp_async_commit();
                    if (it >= LAG) {
                        cp_async_wait<LAG>();
                        fence_proxy_async();
                        mbar_arrive(full0 + 8 * (int)((it - LAG) % S));
                    }
                }
            }
            // every producer is past this tile's map: refill the slot with tile i+2
            named_sync(1, NP);
            if (tid == 0 && tile + 2 * (int)gridDim.x < tiles) request(tile + 2 * gridDim.x, buf);
        }
        if (!async_arrive) {
            cp_async_wait<0>();
            fence_proxy_async();
            for (long long q = std::max<long long>(0, it - LAG); q < it; ++q) mbar_arrive(full0 + 8 * (int)(q % S));
        }
    } else if (!TILED && warp < 4) {  // register-prefetch producers (PW == 4)
        // ---------------- producers
        const int c = tid & 7;    // 16-byte chunk within a 128-byte row
        const int r0 = tid >> 3;  // rows r0 + 16j
        // Field-map entries for stage it+2 are loaded while stage it is issued; the three
        // register buffers rotate by unrolling (no register copies, which would force
        // the in-flight loads to complete early).
        int fa[BM / 16], fb[BM / 16], fc[BM / 16];
        int lt = blockIdx.x, lk = 0;  // load cursor (two stages ahead)
        int ut = blockIdx.x, uk = 0;  // issue cursor
        auto fetch = [&](int (&dst)[BM / 16]) {
            const int k = lk * BK + c * 8;
            const bool ok = lt < tiles && k < K;
            const int t = ok ? k / C : 0;
#pragma unroll
            for (int j = 0; j < BM / 16; ++j) {
                const long long n = (long long)lt * BM + r0 + 16 * j;
                dst[j] = (ok && n < rows) ? fm_ld(fm, n, t) : -1;
            }
            if (++lk == nkb) {
                lk = 0;
                lt += gridDim.x;
            }
        };
        auto issue = [&](long long it, const int (&use)[BM / 16]) {
            const int s = (int)(it % S);
            if (it >= S) mbar_wait(empty0 + 8 * s, (uint32_t)(((it / S) + 1) & 1));
            uint8_t* A = smem + s * Cfg::STAGE_BYTES;
            uint8_t* B = A + Cfg::A_BYTES;
            const int k = uk * BK + c * 8;
            const int ci = k < K ? k - (k / C) * C : 0;
#pragma unroll
            for (int j = 0; j < BM / 16; ++j) {
                const int r = r0 + 16 * j;
                const int g = use[j];
                const bf16* src = g >= 0 ? X + (long long)g * C + ci : X;
                cp_async16(smem_u32(A + sw128_offset(r, c)), src, g >= 0 ? 16u : 0u);
            }
#pragma unroll
            for (int j = 0; j < BN / 16; ++j) {
                const int r = r0 + 16 * j;
                cp_async16(smem_u32(B + sw128_offset(r, c)), Wp + (long long)r * Kp + uk * BK + c * 8, 16u);
            }
            cp_async_commit();
            if (it >= LAG) {
                cp_async_wait<LAG>();
                fence_proxy_async();
                mbar_arrive(full0 + 8 * (int)((it - LAG) % S));
            }
            if (++uk == nkb) {
                uk = 0;
                ut += gridDim.x;
            }
        };
        const long long my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
        const long long total = my_tiles * nkb;
        fetch(fa);
        fetch(fb);
        long long it = 0;
        for (; it + 3 <= total; it += 3) {
            fetch(fc);
            issue(it, fa);
            fetch(fa);
            issue(it + 1, fb);
            fetch(fb);
            issue(it + 2, fc);
        }
        if (it < total) {
            fetch(fc);
            issue(it++, fa);
        }
        if (it < total) issue(it++, fb);
        cp_async_wait<0>();
        fence_proxy_async();
        for (long long i = std::max<long long>(0, it - LAG); i < it; ++i) mbar_arrive(full0 + 8 * (int)(i % S));
    } else if (warp < PW + 4) {
        // ---------------- epilogue warpgroup: TMEM -> registers -> Y rows
        const int q = warp & 3;  // TMEM lane quadrant of this warp
        const int row = q * 32 + (int)lane_id();
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
                if (m < rows) store_row(Y + m * BN + c0, f);
            }
            tc_fence_before();
            mbar_arrive(tempty0 + 8 * acc);
        }
    } else if (tid == (PW + 4) * 32) {
        // ---------------- MMA issuer (single thread)
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
                if (async_arrive) fence_proxy_async();
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
//   A[m][n] = X[nbr(n, m / C)][m % C]  (m = t*C + ci; MN-major: 128 B rows per voxel)
//   B[co][n] = dY[n][co]               (MN-major; C_out < 64 zero-padded to 64)
template <int NB>  // N tile = padded C_out (64, 128 or 256)
struct DwCfg {
    static constexpr int KB = 64;  // voxels per stage
    static constexpr int STAGES = NB <= 64 ? 4 : 3;
    static constexpr int LAG = STAGES - 1;
    static constexpr int A_BYTES = 2 * KB * 128;  // two 64-wide MN blocks (M = 128)
    static constexpr int B_BYTES = (NB / 64) * KB * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int PRODUCERS = 256;          // warps 0-7 (epilogue: warps 0-3)
    static constexpr int THREADS = PRODUCERS + 32;  // + warp 8: TMEM allocator and MMA issuer
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;
    static constexpr int AJ = 1024 / PRODUCERS;            // A chunks per producer per stage
    static constexpr int BJ = (NB / 64) * 512 / PRODUCERS;  // B chunks per producer per stage
};

template <int NB>
__global__ void __launch_bounds__(DwCfg<NB>::THREADS)
    k_gather_dw(FMap fm, long long rows, const bf16* __restrict__ X, int C, int K, const bf16* __restrict__ dY,
                int Cout, int kb_per_split, float* __restrict__ partial, int Mtot, int async_arrive) {
    using Cfg = DwCfg<NB>;
    constexpr int S = Cfg::STAGES;
    constexpr int LAG = Cfg::LAG;
    constexpr int KB = Cfg::KB;
    constexpr int AJ = Cfg::AJ, BJ = Cfg::BJ;
    constexpr int P = Cfg::PRODUCERS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 1);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int mt = blockIdx.x, split = blockIdx.y;
    const long long total_kb = (rows + KB - 1) / KB;
    const long long kb_begin = (long long)split * kb_per_split;
    const int nkb = (int)std::max<long long>(0, std::min<long long>(kb_per_split, total_kb - kb_begin));
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S), done = smem_u32(bars + 2 * S);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, P);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(done, 1);
        mbar_init_fence();
    }
    if (warp == 8) tmem_alloc(smem_u32(tmem_slot), tmem_cols(NB));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 8) {
        // ---------------- producers. Per-thread constants (hoisted out of the stage loop):
        // A chunk j: MN block / voxel row / 16-byte chunk -> its swizzled smem offset, the
        // field-map tap it reads, and its channel offset inside the gathered X row.
        const int c = tid & 7;
        const int q0 = tid >> 3;  // 0..31
        uint32_t a_off[AJ], b_off[BJ];
        int tap[AJ], cio[AJ], rj[AJ], b_r[BJ], b_co[BJ];
#pragma unroll
        for (int j = 0; j < AJ; ++j) {
            const int q = q0 + 32 * j;  // 0..127 = (block, voxel row)
            const int blk = q >> 6, r = q & 63;
            const int mm = mt * BM + blk * 64 + c * 8;
            tap[j] = mm < K ? mm / C : -1;
            cio[j] = mm < K ? mm - (mm / C) * C : 0;
            rj[j] = r;
            a_off[j] = blk * (KB * 128) + sw128_offset(r, c);
        }
#pragma unroll
        for (int j = 0; j < BJ; ++j) {
            const int q = q0 + 32 * j;
            const int blk = q >> 6, r = q & 63;
            b_r[j] = r;
            b_co[j] = blk * 64 + c * 8;
            b_off[j] = blk * (KB * 128) + sw128_offset(r, c);
        }
        int cur[AJ], nx1[AJ], nx2[AJ];
        auto fetch = [&](int kb, int (&dst)[AJ]) {
            const long long n0 = (kb_begin + kb) * KB;
#pragma unroll
            for (int j = 0; j < AJ; ++j) {
                const long long n = n0 + rj[j];
                dst[j] = (kb < nkb && tap[j] >= 0 && n < rows) ? fm_ld(fm, n, tap[j]) : -1;
            }
        };
        auto issue = [&](int kb, const int (&use)[AJ]) {
            const int s = kb % S;
            if (kb >= S) mbar_wait(empty0 + 8 * s, ((kb / S) + 1) & 1);
            const uint32_t A = smem_u32(smem + s * Cfg::STAGE_BYTES);
            const uint32_t B = A + Cfg::A_BYTES;
            const long long n0 = (kb_begin + kb) * KB;
#pragma unroll
            for (int j = 0; j < AJ; ++j) {
                const int g = use[j];
                const bf16* src = g >= 0 ? X + (long long)g * C + cio[j] : X;
                cp_async16(A + a_off[j], src, g >= 0 ? 16u : 0u);
            }
            const bf16* dyb = dY + n0 * Cout;
            const bool full_stage = n0 + KB <= rows;
#pragma unroll
            for (int j = 0; j < BJ; ++j) {
                const bool ok = b_co[j] < Cout && (full_stage || n0 + b_r[j] < rows);
                const bf16* src = ok ? dyb + (long long)b_r[j] * Cout + b_co[j] : dY;
                cp_async16(B + b_off[j], src, ok ? 16u : 0u);
            }
            if (async_arrive) {
                cp_async_arrive_noinc(full0 + 8 * s);
            } else {
                cp_async_commit();
                if (kb >= LAG) {
                    cp_async_wait<LAG>();
                    fence_proxy_async();
                    mbar_arrive(full0 + 8 * ((kb - LAG) % S));
                }
            }
        };
        // field-map entries two stages ahead; buffers rotate by unrolling (no copies)
        fetch(0, cur);
        fetch(1, nx1);
        int kb = 0;
        for (; kb + 3 <= nkb; kb += 3) {
            fetch(kb + 2, nx2);
            issue(kb, cur);
            fetch(kb + 3, cur);
            issue(kb + 1, nx1);
            fetch(kb + 4, nx1);
            issue(kb + 2, nx2);
        }
        if (kb < nkb) {
            fetch(kb + 2, nx2);
            issue(kb++, cur);
        }
        if (kb < nkb) issue(kb++, nx1);
        if (!async_arrive) {
            cp_async_wait<0>();
            fence_proxy_async();
            for (int q = std::max(0, nkb - LAG); q < nkb; ++q) mbar_arrive(full0 + 8 * (q % S));
        }

        // epilogue (warps 0-3 = TMEM lane quadrants): row m = (t,ci) index, columns co
        if (warp < 4) {
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
                    for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]);
                    store_row(dst + c0, f);
                }
            }
        }
    } else if (tid == 8 * 32 && nkb > 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(BM, NB, true, true);
        constexpr uint32_t LBO = KB * 128;  // next 64-wide MN block
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % S;
            mbar_wait(full0 + 8 * s, (kb / S) & 1);
            if (async_arrive) fence_proxy_async();
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
    if (warp == 8) {
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
template <int BN, int CPS, bool TILED, typename OutT, int PW = 4>
void launch_gg_cps(const FMap& fm, long long rows, const bf16* X, int C, int K, const bf16* Wp, int Kp, OutT* Y,
                   cudaStream_t s) {
    using Cfg = FwdCfg<BN, CPS, TILED, PW>;
    auto kern = k_gather_gemm<BN, CPS, TILED, OutT, PW>;
    static bool attr = false;  // per instantiation
    if (!attr) {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM), "smem attr");
        attr = true;
    }
    const int tiles = (int)((rows + BM - 1) / BM);
    const int grid = std::min(tiles, CPS * num_sms());
    kern<<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(fm, rows, X, C, K, Wp, Kp, Y, tiles, TILED ? async_arrive() : 0);
    launched("conv gather-GEMM (tcgen05)");
}

// Two resident CTAs per SM (twice the producer warps) whenever the ring still gets >= 3
// stages and the two CTAs' double-buffered TMEM accumulators fit (2 * 2 * BN <= 512);
// HCB_FWD_CPS=1 forces one.
int fwd_env_cps() {
    static int env = -1;
    if (env < 0) {
        const char* e = std::getenv("HCB_FWD_CPS");
        env = e ? std::atoi(e) : 0;
    }
    return env;
}

// Variant choice: the bulk-staged (TILED) producer when the map is tile-major and two
// CTAs per SM still get a >= 3-stage ring; otherwise the register-prefetch producer with
// two CTAs per SM; one CTA per SM only when nothing else fits (BN = 256).
// HCB_FWD_VARIANT=1 forces the register-prefetch producer (A/B experiments).
template <int BN, typename OutT>
void launch_gg(const FMap& fm, long long rows, const bf16* X, int C, int K, const bf16* Wp, int Kp, OutT* Y,
               cudaStream_t s) {
    constexpr bool tiled_two = BN <= 128 && FwdCfg<BN, 2, true>::STAGES >= 3;
    constexpr bool reg_two = BN <= 128 && FwdCfg<BN, 2, false>::STAGES >= 3;
    static int variant = -1;
    if (variant < 0) {
        const char* e = std::getenv("HCB_FWD_VARIANT");
        variant = e ? std::atoi(e) : 0;
    }
    const bool one = fwd_env_cps() == 1;
    if constexpr (tiled_two) {
        if (fm.tiled && variant != 1 && !one) {
            if (fwd_pw() == 8) return launch_gg_cps<BN, 2, true, OutT, 8>(fm, rows, X, C, K, Wp, Kp, Y, s);
            return launch_gg_cps<BN, 2, true, OutT, 4>(fm, rows, X, C, K, Wp, Kp, Y, s);
        }
    }
    if constexpr (reg_two) {
        if (!one) return launch_gg_cps<BN, 2, false>(fm, rows, X, C, K, Wp, Kp, Y, s);
    }
    if (fm.tiled && variant != 1) return launch_gg_cps<BN, 1, true>(fm, rows, X, C, K, Wp, Kp, Y, s);
    launch_gg_cps<BN, 1, false>(fm, rows, X, C, K, Wp, Kp, Y, s);
}

template <typename OutT>
void gather_gemm(const FMap& fm, long long rows, const bf16* X, int C, int K, const bf16* Wp, int Kp, int N, OutT* Y,
                 cudaStream_t s) {
    if (fm.tiled && gather_gemm_tma_supported(C, N)) {  // TMA gather4 producers (conv_tma.cu)
        gather_gemm_tma<OutT>(fm.p, fm.taps, rows, X, C, Wp, Kp, N, Y, s);
        return;
    }
    switch (N) {
        case 16: launch_gg<16>(fm, rows, X, C, K, Wp, Kp, Y, s); break;
        case 32: launch_gg<32>(fm, rows, X, C, K, Wp, Kp, Y, s); break;
        case 64: launch_gg<64>(fm, rows, X, C, K, Wp, Kp, Y, s); break;
        case 128: launch_gg<128>(fm, rows, X, C, K, Wp, Kp, Y, s); break;
        case 256: launch_gg<256>(fm, rows, X, C, K, Wp, Kp, Y, s); break;
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
    const int smem = p.nb <= 64 ? DwCfg<64>::SMEM : p.nb <= 128 ? DwCfg<128>::SMEM : DwCfg<256>::SMEM;
    const int per_sm = smem <= 113 * 1024 ? 2 : 1;  // resident CTAs per SM (shared-memory bound)
    const int slots = num_sms() * per_sm;
    // one wave: mt * splits <= resident slots
    int want = std::max(1, slots / p.mt);
    want = (int)std::min<long long>(want, std::max<long long>(1, total_kb));
    p.kbps = (int)((total_kb + want - 1) / want);
    p.splits = (int)((total_kb + p.kbps - 1) / p.kbps);
    p.partial_floats = (long long)p.splits * p.mt * BM * p.nb;
    return p;
}

template <int NB>
void launch_dw(const DwPlan& p, const FMap& fm, long long rows, const bf16* X, int C, int K, const bf16* dY, int Cout,
               float* partial, cudaStream_t s) {
    using Cfg = DwCfg<NB>;
    auto kern = k_gather_dw<NB>;
    static bool attr = false;
    if (!attr) {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM), "smem attr");
        attr = true;
    }
    dim3 g((unsigned)p.mt, (unsigned)p.splits);
    kern<<<g, Cfg::THREADS, Cfg::SMEM, s>>>(fm, rows, X, C, K, dY, Cout, p.kbps, partial, p.mt * BM, async_arrive());
    launched("conv dW gather-GEMM (tcgen05)");
}

void check_native(int cin, int cout, int taps) {
    if (cin <= 0 || cin % 8 != 0) throw std::invalid_argument("native conv: input channels must be a multiple of 8");
    if (cout <= 0 || cout % 8 != 0) throw std::invalid_argument("native conv: output channels must be a multiple of 8");
    if (taps < 1 || taps > 27) throw std::invalid_argument("native conv: 1..27 field taps supported");
}

FMap make_fmap(const int32_t* fmap, int32_t layout, long long n, int taps) {
    if (layout == 2) return FMap{fmap, 0, 0, 1, taps};
    if (layout == 1) return FMap{fmap, 1, n, 0, taps};
    if (layout != 0) throw std::invalid_argument("native conv: unknown field-map layout");
    return FMap{fmap, taps, 1, 0, taps};
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

hc_status hc_native_gather_gemm(const int32_t* fmap, int32_t fmap_layout, int64_t n_out, int32_t taps,
                                const void* x, int32_t c_in, const void* w_packed, int32_t c_out, void* y,
                                hc_dtype y_dtype, hc_stream stream) {
    return guard([&] {
        check_native(c_in, c_out, taps);
        if (n_out <= 0) return;
        const int Kp = (int)hc_native_packed_k(c_in, taps);
        const FMap fm = make_fmap(fmap, fmap_layout, n_out, taps);
        cudaStream_t s = as_stream(stream);
        const bf16* X = static_cast<const bf16*>(x);
        const bf16* W = static_cast<const bf16*>(w_packed);
        if (y_dtype == HC_DTYPE_F32)
            gather_gemm<float>(fm, n_out, X, c_in, taps * c_in, W, Kp, c_out, static_cast<float*>(y), s);
        else
            gather_gemm<bf16>(fm, n_out, X, c_in, taps * c_in, W, Kp, c_out, static_cast<bf16*>(y), s);
    });
}

size_t hc_native_dw_workspace(int64_t n_out, int32_t taps, int32_t c_in, int32_t c_out) {
    const DwPlan p = dw_plan(n_out, taps, c_in, c_out);
    return (size_t)p.partial_floats * sizeof(float);
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
        const FMap fm = make_fmap(fmap, fmap_layout, n_out, taps);
        const bf16* X = static_cast<const bf16*>(x);
        const bf16* DY = static_cast<const bf16*>(dy);
        switch (p.nb) {
            case 64: launch_dw<64>(p, fm, n_out, X, c_in, taps * c_in, DY, c_out, part, s); break;
            case 128: launch_dw<128>(p, fm, n_out, X, c_in, taps * c_in, DY, c_out, part, s); break;
            default: launch_dw<256>(p, fm, n_out, X, c_in, taps * c_in, DY, c_out, part, s); break;
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
