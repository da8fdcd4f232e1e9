// x2_layout.cuh — the split-precision row layout shared by the conv kernels (conv_tc.cu) and the
// net layers that write it directly (net_ops.cu).
//
// An fp32 value v is carried as two bf16 values: hi = rn(v), lo = rn(v - hi) (|v - hi - lo| <=
// 2^-17 |v|). A row of C channels becomes 2C bf16: the planes interleave in blocks of g channels,
// g = 64 when C is a multiple of 64 (else g = C, i.e. [hi | lo]): channel c of plane p sits at
// (c / g) * 2g + p * g + c % g, so a 64-wide K stage of the conv holds one plane of 64 channels.
#pragma once
#include <cuda_bf16.h>

namespace hcb {

__host__ __device__ __forceinline__ int x2_block(int C) { return C % 64 == 0 ? 64 : C; }
__host__ __device__ __forceinline__ int x2_pos(int c, int p, int g) { return (c / g) * 2 * g + p * g + c % g; }

__device__ __forceinline__ void split2(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(v);
    lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// 8 consecutive channels c0 .. c0+7 (c0 % 8 == 0, C % 8 == 0) of one row into its split row.
__device__ __forceinline__ void store8_split(__nv_bfloat16* row2c, int c0, int C, const float (&v)[8]) {
    const int g = x2_block(C);
    uint4 h, l;
    __nv_bfloat16* hp = reinterpret_cast<__nv_bfloat16*>(&h);
    __nv_bfloat16* lp = reinterpret_cast<__nv_bfloat16*>(&l);
#pragma unroll
    for (int e = 0; e < 8; ++e) split2(v[e], hp[e], lp[e]);
    *reinterpret_cast<uint4*>(row2c + x2_pos(c0, 0, g)) = h;
    *reinterpret_cast<uint4*>(row2c + x2_pos(c0, 1, g)) = l;
}

}  // namespace hcb
