// psh_build.cu — perfect spatial hash construction on the GPU (the
// paper's "future work").
//
// Same table sizing and lookup semantics as the reference builder (psh.cpp:170-227):
// m_bar = minimal_hash_dim(n), r_bar = initial_offset_dim(n) made coprime to m_bar, cells
// h1(p) = p mod r_bar, slot(p) = (p mod m_bar + Phi[h1(p)]) mod m_bar, hash[slot] = data
// index, tags = coordinates, redundant slots -1 / 0xFFFF; on failure r_bar grows by cbrt(2)
// per attempt. The search differs: instead of placing cells one at a time (greedy, in
// decreasing load), every cell of one load class searches for its offset concurrently —
// a seeded random candidate sequence, then an exhaustive scan from a seeded start — and
// claims its slots with atomicCAS (a partial claim that loses a race is rolled back and the
// search continues). Load classes still go largest first, so the greedy order's packing
// advantage is kept. The tables are therefore a DIFFERENT valid PSH of the same set: every
// lookup (locate, all operators) returns the same column as with the reference's tables,
// which is what tests/test_psh_device.py checks, together with perfection (each voxel in
// exactly one slot with its own tag).
#include <cuda_runtime.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "hashconv_b200.h"
#include "hc_internal.h"
#include "hc_launch.cuh"

namespace hcb {
namespace {

constexpr int kT = 256;

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {  // splitmix64 finaliser
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ long long slot_of(int3 p, int ox, int oy, int oz, int m, int dim) {
    const int sx = (p.x % m + ox) % m, sy = (p.y % m + oy) % m;
    if (dim == 2) return (long long)sy * m + sx;
    const int sz = (p.z % m + oz) % m;
    return ((long long)sz * m + sy) * m + sx;
}

__global__ void k_cells(const int3* __restrict__ pts, long long n, int r, int dim, long long* __restrict__ cell) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int3 p = pts[i];
    const long long c = dim == 2 ? (long long)(p.y % r) * r + p.x % r
                                 : ((long long)(p.z % r) * r + p.y % r) * r + p.x % r;
    cell[i] = c;
}

// Try to place `cell` (voxel ids ids[0..k)) with offset (ox,oy,oz): claim every slot by CAS,
// roll back on the first lost slot. Returns true when all k slots are ours.
__device__ bool try_claim(const int3* __restrict__ pts, const int* __restrict__ ids, int k, int ox, int oy, int oz,
                          int m, int dim, int* __restrict__ hash) {
    for (int j = 0; j < k; ++j) {
        const int id = ids[j];
        const long long s = slot_of(pts[id], ox, oy, oz, m, dim);
        if (hash[s] != -1 || atomicCAS(hash + s, -1, id) != -1) {
            for (int u = 0; u < j; ++u) atomicExch(hash + slot_of(pts[ids[u]], ox, oy, oz, m, dim), -1);
            return false;
        }
    }
    return true;
}

// One thread per cell of a load class: random candidates, then an exhaustive scan.
__global__ void k_place(const int3* __restrict__ pts, const int* __restrict__ sorted_ids,
                        const int* __restrict__ cell_begin, const long long* __restrict__ cell_id,
                        const int* __restrict__ cell_size, int first, int count, int m, int dim, int lim,
                        unsigned long long seed, int* __restrict__ hash, unsigned char* __restrict__ offsets,
                        int* __restrict__ failed) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int c = first + i;
    const int* ids = sorted_ids + cell_begin[c];
    const int k = cell_size[c];
    const long long cid = cell_id[c];
    const int oz_lim = dim == 3 ? lim : 1;
    bool ok = false;
    int ox = 0, oy = 0, oz = 0;
    for (int t = 0; t < 256 && !ok; ++t) {  // seeded random candidates
        const unsigned long long h = mix64(seed ^ mix64((unsigned long long)cid * 1315423911ull + t));
        ox = (int)(h % lim);
        oy = (int)((h >> 21) % lim);
        oz = dim == 3 ? (int)((h >> 42) % lim) : 0;
        ok = try_claim(pts, ids, k, ox, oy, oz, m, dim, hash);
    }
    if (!ok) {  // exhaustive scan from a seeded start (every distinct offset once)
        const long long total = (long long)lim * lim * oz_lim;
        const long long start = (long long)(mix64(seed + 0x51ED270Bull * (unsigned long long)(cid + 1)) % total);
        for (long long q = 0; q < total && !ok; ++q) {
            long long v = start + q;
            if (v >= total) v -= total;
            ox = (int)(v % lim);
            oy = (int)((v / lim) % lim);
            oz = (int)(v / ((long long)lim * lim));
            ok = try_claim(pts, ids, k, ox, oy, oz, m, dim, hash);
        }
    }
    if (!ok) {
        atomicAdd(failed, 1);
        return;
    }
    offsets[cid * dim + 0] = (unsigned char)ox;
    offsets[cid * dim + 1] = (unsigned char)oy;
    if (dim == 3) offsets[cid * dim + 2] = (unsigned char)oz;
}

__global__ void k_tags(const int3* __restrict__ pts, long long n, int m, int r, int dim,
                       const unsigned char* __restrict__ offsets, unsigned short* __restrict__ tags) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int3 p = pts[i];
    const long long c = dim == 2 ? (long long)(p.y % r) * r + p.x % r
                                 : ((long long)(p.z % r) * r + p.y % r) * r + p.x % r;
    const int oz = dim == 3 ? offsets[c * dim + 2] : 0;
    const long long s = slot_of(p, offsets[c * dim], offsets[c * dim + 1], oz, m, dim);
    tags[s * dim + 0] = (unsigned short)p.x;
    tags[s * dim + 1] = (unsigned short)p.y;
    if (dim == 3) tags[s * dim + 2] = (unsigned short)p.z;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(size_t n) { cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// One attempt at fixed (m, r); false when some cell found no offset.
bool device_attempt(const VoxelSet& s, const int3* pts, int m, int r, unsigned long long seed, PshLevel& L) {
    const int dim = s.dim;
    const long long n = s.count();
    const long long slots = ipow(m, dim), cells = ipow(r, dim);
    DevBuf<long long> cell(n);
    DevBuf<int> ids(n);
    k_cells<<<grid_for(n, kT), kT>>>(pts, n, r, dim, cell.p);
    launched("psh cells");
    thrust::sequence(thrust::device, ids.p, ids.p + n);
    thrust::sort_by_key(thrust::device, cell.p, cell.p + n, ids.p);  // bucket = run of equal cells
    // bucket boundaries on the host (n int64 cell keys: one copy; the class loop is host-driven)
    std::vector<long long> hc(static_cast<size_t>(n));
    cuda_check(cudaMemcpy(hc.data(), cell.p, sizeof(long long) * n, cudaMemcpyDeviceToHost), "cells D2H");
    std::vector<int> begin, size;
    std::vector<long long> cid;
    for (long long i = 0; i < n;) {
        long long j = i;
        while (j < n && hc[static_cast<size_t>(j)] == hc[static_cast<size_t>(i)]) ++j;
        begin.push_back((int)i);
        size.push_back((int)(j - i));
        cid.push_back(hc[static_cast<size_t>(i)]);
        i = j;
    }
    // load classes, largest first (psh.cpp:51-57 orders cells by decreasing load)
    std::vector<int> order(begin.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return size[a] > size[b]; });
    std::vector<int> ob(order.size()), os(order.size());
    std::vector<long long> oc(order.size());
    for (size_t i = 0; i < order.size(); ++i) {
        ob[i] = begin[static_cast<size_t>(order[i])];
        os[i] = size[static_cast<size_t>(order[i])];
        oc[i] = cid[static_cast<size_t>(order[i])];
    }
    const int nc = (int)ob.size();
    DevBuf<int> d_begin(nc), d_size(nc), failed(1);
    DevBuf<long long> d_cid(nc);
    DevBuf<int> hash(slots);
    DevBuf<unsigned char> offs(cells * dim);
    DevBuf<unsigned short> tags(slots * dim);
    cuda_check(cudaMemcpy(d_begin.p, ob.data(), sizeof(int) * nc, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d_size.p, os.data(), sizeof(int) * nc, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d_cid.p, oc.data(), sizeof(long long) * nc, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemset(hash.p, 0xFF, sizeof(int) * slots), "memset");
    cuda_check(cudaMemset(offs.p, 0, cells * dim), "memset");
    cuda_check(cudaMemset(tags.p, 0xFF, sizeof(unsigned short) * slots * dim), "memset");
    cuda_check(cudaMemset(failed.p, 0, sizeof(int)), "memset");
    const int lim = std::min(m, 256);
    for (int a = 0; a < nc;) {
        int b = a;
        while (b < nc && os[static_cast<size_t>(b)] == os[static_cast<size_t>(a)]) ++b;
        k_place<<<grid_for(b - a, 128), 128>>>(pts, ids.p, d_begin.p, d_cid.p, d_size.p, a, b - a, m, dim, lim,
                                             seed + (unsigned long long)os[static_cast<size_t>(a)], hash.p, offs.p,
                                             failed.p);
        launched("psh place");
        a = b;
    }
    int bad = 0;
    cuda_check(cudaMemcpy(&bad, failed.p, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    if (bad) return false;
    k_tags<<<grid_for(n, kT), kT>>>(pts, n, m, r, dim, offs.p, tags.p);
    launched("psh tags");
    L.hash.resize(static_cast<size_t>(slots));
    L.offsets.resize(static_cast<size_t>(cells * dim));
    L.tags.resize(static_cast<size_t>(slots * dim));
    cuda_check(cudaMemcpy(L.hash.data(), hash.p, sizeof(int) * slots, cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(L.offsets.data(), offs.p, cells * dim, cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(L.tags.data(), tags.p, sizeof(unsigned short) * slots * dim, cudaMemcpyDeviceToHost),
               "D2H");
    return true;
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" hc_status hc_build_psh_device(const hc_voxel_set* s, uint64_t seed, hc_psh_level** out) {
    return guard([&] {
        const VoxelSet& v = *s;
        if (v.voxels.empty()) throw std::invalid_argument("empty input");
        if (v.resolution >= 65536)
            throw std::invalid_argument(
                "resolution 65536 conflicts with the redundant-slot tag; pass allow_tag_ambiguity");
        const long long n = v.count();
        std::vector<int3> hp(static_cast<size_t>(n));
        for (long long i = 0; i < n; ++i) {
            const Coord& p = v.voxels[static_cast<size_t>(i)];
            hp[static_cast<size_t>(i)] = make_int3(p[0], p[1], v.dim == 3 ? p[2] : 0);
        }
        DevBuf<int3> pts(n);
        cuda_check(cudaMemcpy(pts.p, hp.data(), sizeof(int3) * n, cudaMemcpyHostToDevice), "coords H2D");
        auto* L = new hc_psh_level;
        L->dim = v.dim;
        L->resolution = v.resolution;
        L->n = n;
        L->hash_dim = psh_hash_dim(n, v.dim);
        L->channels = v.channels;
        L->data = v.features;
        std::int32_t r = psh_first_offset_dim(n, v.dim);
        for (int attempt = 0;; ++attempt) {  // psh.cpp:204-226 growth schedule
            if (r < v.resolution)
                while (std::gcd(L->hash_dim, r) != 1 && r < v.resolution) ++r;
            r = std::min(r, v.resolution);
            if (ipow(r, v.dim) * v.dim > (std::int64_t{1} << 31)) {
                delete L;
                throw std::runtime_error("hash construction diverged");
            }
            if (device_attempt(v, pts.p, L->hash_dim, r, seed * 0x9E3779B97F4A7C15ull + attempt, *L)) {
                L->offset_dim = r;
                *out = L;
                return;
            }
            if (r >= v.resolution) {
                delete L;
                throw std::runtime_error("hash construction diverged");
            }
            r = std::max(static_cast<std::int32_t>(std::ceil(static_cast<double>(r) * std::cbrt(2.0))), r + 1);
        }
    });
}
