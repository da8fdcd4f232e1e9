// dev_psh.cuh — device-resident super-PSH and the inlined probe (locate).
//
// Layout in HBM (built once by hc_psh_upload*, see device_psh.cu):
//   slots[M]   uint2 {idx (int32, -1 = redundant), key}: H* and T* fused into one
//              8-byte word per hash slot; key = x | y<<kb | z<<2kb (kb = bits of
//              resolution-1), 0xFFFFFFFF when a tag component cannot be a
//              coordinate (never matches). One load per probe instead of 4+6 bytes.
//   phi[R]     uint32 {x | y<<8 | z<<16}: Phi* with each component pre-reduced mod
//              m_bar of its model (exact: (a + phi) mod m == (a + phi mod m) mod m).
//   models[b]  per-model bases (M*, R*, N*), m_bar, r_bar and float reciprocals.
//   cols[N]    int4 {x, y, z, model}: column_info (cnn_ops.cpp:50-66), built on device.
// The raw H*/Phi*/T*/V* arrays are kept too (download, validation).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hcb {

struct ModelParam {
    long long hash_base;    // M*[v-1]
    long long offset_base;  // R*[v-1]
    long long data_base;    // N*[v-1]
    int m, r;               // m_bar, r_bar
    float inv_m, inv_r;     // 1/m, 1/r (fast exact mod for 0 <= p < 2^17)
};

struct DevPsh {
    int dim, resolution, batch, key_bits;
    long long M, R, N;
    const uint2* slots;
    const unsigned* phi;
    const ModelParam* models;
    const int4* cols;
};

// exact p mod d for 0 <= p < 2^17, d >= 1, using a float reciprocal + one fixup
__device__ __forceinline__ int fmod_small(int p, int d, float inv) {
    int q = __float2int_rz(__int2float_rn(p) * inv);
    int r = p - q * d;
    if (r < 0) r += d;
    if (r >= d) r -= d;
    return r;
}

__device__ __forceinline__ unsigned pack_key(int x, int y, int z, int kb) {
    return static_cast<unsigned>(x) | (static_cast<unsigned>(y) << kb) | (static_cast<unsigned>(z) << (2 * kb));
}

// psh_batch.cpp:56-78 locate for one in-domain coordinate, given its residues.
//   rm*, rr*: p mod m_bar / p mod r_bar per axis (z terms 0 for dim 2)
__device__ __forceinline__ int probe_res(const DevPsh& s, const ModelParam& mp, int dim, int x, int y,
                                         int z, int rmx, int rmy, int rmz, int rrx, int rry, int rrz) {
    const long long cell = dim == 3 ? ((long long)rrz * mp.r + rry) * mp.r + rrx : (long long)rry * mp.r + rrx;
    const unsigned ph = __ldg(s.phi + mp.offset_base + cell);
    int sx = rmx + (int)(ph & 0xFF);
    int sy = rmy + (int)((ph >> 8) & 0xFF);
    int sz = rmz + (int)((ph >> 16) & 0xFF);
    if (sx >= mp.m) sx -= mp.m;
    if (sy >= mp.m) sy -= mp.m;
    if (sz >= mp.m) sz -= mp.m;
    const long long slot = dim == 3 ? ((long long)sz * mp.m + sy) * mp.m + sx : (long long)sy * mp.m + sx;
    const uint2 e = __ldg(s.slots + mp.hash_base + slot);
    const int idx = (int)e.x;
    if (idx < 0 || e.y != pack_key(x, y, z, s.key_bits)) return -1;
    return (int)(mp.data_base + idx);
}

__device__ __forceinline__ int probe(const DevPsh& s, const ModelParam& mp, int x, int y, int z) {
    const int dim = s.dim;
    return probe_res(s, mp, dim, x, y, z, fmod_small(x, mp.m, mp.inv_m), fmod_small(y, mp.m, mp.inv_m),
                     dim == 3 ? fmod_small(z, mp.m, mp.inv_m) : 0, fmod_small(x, mp.r, mp.inv_r),
                     fmod_small(y, mp.r, mp.inv_r), dim == 3 ? fmod_small(z, mp.r, mp.inv_r) : 0);
}

// Field taps of one output voxel: base = field origin (cnn_ops.cpp:36-42), F per
// axis, taps in (dz,dy,dx) row order (cnn_ops.cpp:100-119). Residues are
// computed once per axis coordinate (3F fast mods instead of 6F^3); the cell row,
// the packed-key prefix and the per-model table bases are hoisted out of the tap
// loop, and all per-tap index math is 32-bit (tables < 2^31 entries, columns < 2^31),
// so a probe is ~25 instructions around its two dependent loads.
template <int F>
__device__ __forceinline__ void probe_field(const DevPsh& s, const ModelParam& mp, int bx, int by, int bz,
                                            int* out /* F^dim */) {
    const int dim = s.dim, res = s.resolution, kb = s.key_bits;
    const int m = mp.m, r = mp.r;
    const unsigned* phib = s.phi + mp.offset_base;
    const uint2* slotb = s.slots + mp.hash_base;
    const int dbase = (int)mp.data_base;
    int rmx[F], rmy[F], rmz[F], rrx[F], rry[F], rrz[F];
    bool vx[F], vy[F], vz[F];
#pragma unroll
    for (int d = 0; d < F; ++d) {
        const int x = bx + d, y = by + d, z = bz + d;
        vx[d] = x >= 0 && x < res;
        vy[d] = y >= 0 && y < res;
        vz[d] = dim == 3 ? (z >= 0 && z < res) : (d == 0);
        rmx[d] = vx[d] ? fmod_small(x, m, mp.inv_m) : 0;
        rmy[d] = vy[d] ? fmod_small(y, m, mp.inv_m) : 0;
        rmz[d] = (dim == 3 && vz[d]) ? fmod_small(z, m, mp.inv_m) : 0;
        rrx[d] = vx[d] ? fmod_small(x, r, mp.inv_r) : 0;
        rry[d] = vy[d] ? fmod_small(y, r, mp.inv_r) : 0;
        rrz[d] = (dim == 3 && vz[d]) ? fmod_small(z, r, mp.inv_r) : 0;
    }
    const int fz = dim == 3 ? F : 1;
#pragma unroll
    for (int dz = 0; dz < F; ++dz) {
        if (dz >= fz) break;
        const unsigned kz = dim == 3 ? (unsigned)(bz + dz) << (2 * kb) : 0u;
#pragma unroll
        for (int dy = 0; dy < F; ++dy) {
            const bool vzy = vz[dz] && vy[dy];
            const int cell_zy = (rrz[dz] * r + rry[dy]) * r;  // dim 2: rrz = 0 -> rry * r
            const unsigned key_zy = kz | ((unsigned)(by + dy) << kb);
#pragma unroll
            for (int dx = 0; dx < F; ++dx) {
                const int t = (dz * F + dy) * F + dx;
                int v = -1;
                if (vzy && vx[dx]) {
                    const unsigned ph = __ldg(phib + cell_zy + rrx[dx]);
                    int sx = rmx[dx] + (int)(ph & 0xFF);
                    int sy = rmy[dy] + (int)((ph >> 8) & 0xFF);
                    int sz = rmz[dz] + (int)((ph >> 16) & 0xFF);  // dim 2: both terms 0
                    if (sx >= m) sx -= m;
                    if (sy >= m) sy -= m;
                    if (sz >= m) sz -= m;
                    const uint2 e = __ldg(slotb + (sz * m + sy) * m + sx);
                    if ((int)e.x >= 0 && e.y == (key_zy | (unsigned)(bx + dx))) v = dbase + (int)e.x;
                }
                out[t] = v;
            }
        }
    }
}

// probe_field in three explicit phases — all F^dim offset-table loads, then all hash-slot
// loads, then the tag compares — so a thread keeps F^dim independent probe chains in
// flight (the fused form leaves ~1 chain in flight per thread; the K0 map kernels are
// bound by that latency, not by bytes). Same results as probe_field.
template <int F>
__device__ __forceinline__ void probe_field_batched(const DevPsh& s, const ModelParam& mp, int bx, int by, int bz,
                                                    int* out /* F^dim */) {
    constexpr int T = F * F * F;
    const int dim = s.dim, res = s.resolution, kb = s.key_bits;
    const int m = mp.m, r = mp.r;
    const unsigned* phib = s.phi + mp.offset_base;
    const uint2* slotb = s.slots + mp.hash_base;
    const int dbase = (int)mp.data_base;
    if (dim == 3 && bx >= 0 && by >= 0 && bz >= 0 && bx + F <= res && by + F <= res && bz + F <= res) {
        // interior field (every shell voxel away from the domain faces): no per-tap validity,
        // cell / slot-row / key prefixes per (dz, dy), 32-bit offsets from the model's bases
        int rmx[F], rmy[F], rmz[F], rrx[F], cyz[F * F];
        unsigned kyz[F * F];
#pragma unroll
        for (int d = 0; d < F; ++d) {
            rmx[d] = fmod_small(bx + d, m, mp.inv_m);
            rmy[d] = fmod_small(by + d, m, mp.inv_m);
            rmz[d] = fmod_small(bz + d, m, mp.inv_m);
            rrx[d] = fmod_small(bx + d, r, mp.inv_r);
        }
#pragma unroll
        for (int dz = 0; dz < F; ++dz)
#pragma unroll
            for (int dy = 0; dy < F; ++dy) {
                cyz[dz * F + dy] =
                    (fmod_small(bz + dz, r, mp.inv_r) * r + fmod_small(by + dy, r, mp.inv_r)) * r;
                kyz[dz * F + dy] = ((unsigned)(bz + dz) << (2 * kb)) | ((unsigned)(by + dy) << kb);
            }
        unsigned ph[T];
#pragma unroll
        for (int t = 0; t < T; ++t) ph[t] = __ldg(phib + cyz[t / F] + rrx[t % F]);
        uint2 e[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int dz = t / (F * F), dy = (t / F) % F, dx = t % F;
            int sx = rmx[dx] + (int)(ph[t] & 0xFF);
            int sy = rmy[dy] + (int)((ph[t] >> 8) & 0xFF);
            int sz = rmz[dz] + (int)((ph[t] >> 16) & 0xFF);
            if (sx >= m) sx -= m;
            if (sy >= m) sy -= m;
            if (sz >= m) sz -= m;
            e[t] = __ldg(slotb + (sz * m + sy) * m + sx);
        }
#pragma unroll
        for (int t = 0; t < T; ++t)
            out[t] = ((int)e[t].x >= 0 && e[t].y == (kyz[t / F] | (unsigned)(bx + t % F))) ? dbase + (int)e[t].x
                                                                                           : -1;
        return;
    }
    int rmx[F], rmy[F], rmz[F], rrx[F], rry[F], rrz[F];
    bool vx[F], vy[F], vz[F];
#pragma unroll
    for (int d = 0; d < F; ++d) {
        const int x = bx + d, y = by + d, z = bz + d;
        vx[d] = x >= 0 && x < res;
        vy[d] = y >= 0 && y < res;
        vz[d] = dim == 3 ? (z >= 0 && z < res) : (d == 0);
        rmx[d] = vx[d] ? fmod_small(x, m, mp.inv_m) : 0;
        rmy[d] = vy[d] ? fmod_small(y, m, mp.inv_m) : 0;
        rmz[d] = (dim == 3 && vz[d]) ? fmod_small(z, m, mp.inv_m) : 0;
        rrx[d] = vx[d] ? fmod_small(x, r, mp.inv_r) : 0;
        rry[d] = vy[d] ? fmod_small(y, r, mp.inv_r) : 0;
        rrz[d] = (dim == 3 && vz[d]) ? fmod_small(z, r, mp.inv_r) : 0;
    }
    unsigned ph[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int dz = t / (F * F), dy = (t / F) % F, dx = t % F;
        const bool ok = vz[dz] && vy[dy] && vx[dx];
        ph[t] = ok ? __ldg(phib + (rrz[dz] * r + rry[dy]) * r + rrx[dx]) : 0xFFFFFFFFu;
    }
    uint2 e[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int dz = t / (F * F), dy = (t / F) % F, dx = t % F;
        if (ph[t] != 0xFFFFFFFFu) {
            int sx = rmx[dx] + (int)(ph[t] & 0xFF);
            int sy = rmy[dy] + (int)((ph[t] >> 8) & 0xFF);
            int sz = rmz[dz] + (int)((ph[t] >> 16) & 0xFF);
            if (sx >= m) sx -= m;
            if (sy >= m) sy -= m;
            if (sz >= m) sz -= m;
            e[t] = __ldg(slotb + (sz * m + sy) * m + sx);
        } else {
            e[t] = make_uint2(0xFFFFFFFFu, 0u);
        }
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int dz = t / (F * F), dy = (t / F) % F, dx = t % F;
        const unsigned key = (dim == 3 ? (unsigned)(bz + dz) << (2 * kb) : 0u) | ((unsigned)(by + dy) << kb) |
                             (unsigned)(bx + dx);
        out[t] = ((int)e[t].x >= 0 && e[t].y == key) ? dbase + (int)e[t].x : -1;
    }
}

// Generic-F single tap (any kernel size): used by the fallback kernels.
__device__ __forceinline__ int probe_tap(const DevPsh& s, const ModelParam& mp, int bx, int by, int bz, int F,
                                         int t) {
    const int dim = s.dim;
    const int dx = t % F, dy = (t / F) % F, dz = dim == 3 ? t / (F * F) : 0;
    const int x = bx + dx, y = by + dy, z = dim == 3 ? bz + dz : 0;
    const int res = s.resolution;
    if (x < 0 || x >= res || y < 0 || y >= res || (dim == 3 && (z < 0 || z >= res))) return -1;
    return probe(s, mp, x, y, z);
}

// cnn_ops.cpp:15-18
__device__ __forceinline__ int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// cnn_ops.cpp:70-85 covering_range (per axis, clipped to the output domain)
__device__ __forceinline__ void cover_axis(int p, int F, int S, int pad, int out_res, int& lo, int& hi) {
    int l, h;
    if (S == 1) {
        l = p - (F - 1) / 2;
        h = p + (F - 1) / 2;
    } else {
        l = floordiv(p + pad - F + 1 + S - 1, S);
        h = floordiv(p + pad, S);
    }
    lo = l > 0 ? l : 0;
    hi = h < out_res - 1 ? h : out_res - 1;
}

__device__ __forceinline__ int origin_axis(int po, int F, int S, int pad) {
    return S == 1 ? po - (F - 1) / 2 : po * S - pad;
}

}  // namespace hcb

// Opaque handle behind hc_psh*.
struct hc_psh {
    hcb::DevPsh d;
    // raw device copies of the reference arrays
    int32_t* hash = nullptr;
    uint8_t* offsets = nullptr;
    uint16_t* tags = nullptr;
    int32_t* model_of_slot = nullptr;
    // host copies of the small per-model arrays (batch entries)
    int64_t* h_hash_acc = nullptr;
    int64_t* h_offset_acc = nullptr;
    int64_t* h_data_acc = nullptr;
    int32_t* h_hash_dims = nullptr;
    int32_t* h_offset_dims = nullptr;
    // owned derived device tables
    uint2* slots = nullptr;
    unsigned* phi = nullptr;
    hcb::ModelParam* models = nullptr;
    int4* cols = nullptr;
};
