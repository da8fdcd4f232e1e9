// device_psh.cu — device-resident super-PSH: upload, device-side build_super,
// derived probe tables, column table, batched locate, plus ABI plumbing.
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "dev_psh.cuh"
#include "hc_internal.h"
#include "hc_launch.cuh"

namespace hcb {

namespace {
thread_local std::string g_last_error;
thread_local hc_math g_math = HC_MATH_EXACT;
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw cuda_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

void* dev_alloc(size_t bytes) {
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    return p;
}

hc_math current_math() { return g_math; }
void scratch_pool_init() {
    static thread_local int done_dev = -1;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (done_dev == dev) return;
    const char* e = std::getenv("HCB_POOL_KEEP_GB");
    const double gb = e ? std::atof(e) : 48.0;
    cudaMemPool_t pool;
    cuda_check(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool");
    uint64_t keep = static_cast<uint64_t>(gb * (1ull << 30));
    cuda_check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "pool release threshold");
    done_dev = dev;
}


namespace {
std::atomic<long long> g_launches{0};
}
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

long long fused_route_count(long long add) {
    static std::atomic<long long> n{0};
    return n.fetch_add(add, std::memory_order_relaxed) + add;
}

// One sticky status word in mapped pinned host memory (kernels write it through the device
// alias; the host reads it after a synchronisation): deferred argument checks.
static volatile int* g_deferred = nullptr;
static int* g_deferred_dev = nullptr;
static std::mutex g_deferred_mu;
int* deferred_flag_device() {
    std::lock_guard<std::mutex> lock(g_deferred_mu);
    if (!g_deferred) {
        void* h = nullptr;
        cuda_check(cudaHostAlloc(&h, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc");
        *static_cast<volatile int*>(h) = 0;
        void* d = nullptr;
        cuda_check(cudaHostGetDevicePointer(&d, h, 0), "cudaHostGetDevicePointer");
        g_deferred = static_cast<volatile int*>(h);
        g_deferred_dev = static_cast<int*>(d);
    }
    return g_deferred_dev;
}

bool smem_optin_needed(const void* kern, int dev) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lock(mu);
    return done.insert({kern, dev}).second;
}

namespace {

// ------------------------------------------------------------------ derived tables
// One slot word per hash slot: {idx, packed tag key}.
__global__ void k_build_slots(const int32_t* hash, const uint16_t* tags, long long M, int dim, int kb,
                              uint2* slots) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int idx = hash[i];
    unsigned key = 0xFFFFFFFFu;
    const unsigned lim = 1u << kb;
    const unsigned x = tags[i * dim], y = tags[i * dim + 1], z = dim == 3 ? tags[i * dim + 2] : 0u;
    if (x < lim && y < lim && z < lim) key = x | (y << kb) | (z << (2 * kb));
    slots[i] = make_uint2(static_cast<unsigned>(idx), key);
}

__device__ int find_segment(const long long* acc, int batch, long long i) {
    int lo = 0, hi = batch - 1;  // largest v with acc[v] <= i
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (acc[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Phi pre-reduced mod m_bar of the owning model.
__global__ void k_build_phi(const uint8_t* offsets, long long R, int dim, const long long* offset_acc,
                            const int* hash_dims, int batch, unsigned* phi) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= R) return;
    const int v = find_segment(offset_acc, batch, i);
    const unsigned m = static_cast<unsigned>(hash_dims[v]);
    const unsigned x = offsets[i * dim] % m, y = offsets[i * dim + 1] % m, z = dim == 3 ? offsets[i * dim + 2] % m : 0u;
    phi[i] = x | (y << 8) | (z << 16);
}

// column_info (cnn_ops.cpp:50-66), plus V* when absent.
__global__ void k_build_cols(const int32_t* hash, const uint16_t* tags, const int32_t* model_of_slot,
                             const long long* hash_acc, const long long* data_acc, int batch, long long M,
                             int dim, int4* cols) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int idx = hash[i];
    if (idx < 0) return;
    const int v = model_of_slot[i];
    const long long g = data_acc[v - 1] + idx;
    cols[g] = make_int4(tags[i * dim], tags[i * dim + 1], dim == 3 ? tags[i * dim + 2] : 0, v);
}

__global__ void k_fill_model_of_slot(const long long* hash_acc, int batch, long long M, int32_t* mos) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= M) return;
    mos[i] = find_segment(hash_acc, batch, i) + 1;
}

__global__ void k_locate(hcb::DevPsh s, const int4* q, long long n, long long* out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 e = q[i];  // {model, x, y, z}
    const int res = s.resolution;
    long long r = -1;
    if (e.x >= 1 && e.x <= s.batch && e.y >= 0 && e.y < res && e.z >= 0 && e.z < res &&
        (s.dim == 2 ? e.w == 0 : (e.w >= 0 && e.w < res))) {
        const ModelParam mp = s.models[e.x - 1];
        const int g = probe(s, mp, e.y, e.z, e.w);
        r = g;
    }
    out[i] = r;
}

int bits_for(int res) {
    int kb = 0;
    while ((1 << kb) < res) ++kb;
    return std::max(kb, 1);
}

// Shared tail of both upload paths: raw arrays already on the device.
void finish_upload(hc_psh* p, const std::vector<int64_t>& hacc, const std::vector<int64_t>& oacc,
                   const std::vector<int64_t>& dacc, const std::vector<int32_t>& hdims,
                   const std::vector<int32_t>& odims, bool have_mos, cudaStream_t st) {
    DevPsh& d = p->d;
    const int b = d.batch;
    if (d.dim != 2 && d.dim != 3) throw std::invalid_argument("dim must be 2 or 3");
    d.key_bits = bits_for(d.resolution);
    if (d.dim * d.key_bits > 30)
        throw std::invalid_argument("device super-PSH supports resolution <= 1024 (3D) / 32768 (2D)");
    if (d.N >= (1LL << 31)) throw std::invalid_argument("device super-PSH supports < 2^31 data columns");
    for (int v = 0; v < b; ++v) {
        if (hdims[static_cast<size_t>(v)] < 1 || odims[static_cast<size_t>(v)] < 1)
            throw std::invalid_argument("corrupt super-PSH: bad table dims");
    }
    // host copies
    p->h_hash_acc = new int64_t[b + 1];
    p->h_offset_acc = new int64_t[b + 1];
    p->h_data_acc = new int64_t[b + 1];
    p->h_hash_dims = new int32_t[b];
    p->h_offset_dims = new int32_t[b];
    std::memcpy(p->h_hash_acc, hacc.data(), 8 * (b + 1));
    std::memcpy(p->h_offset_acc, oacc.data(), 8 * (b + 1));
    std::memcpy(p->h_data_acc, dacc.data(), 8 * (b + 1));
    std::memcpy(p->h_hash_dims, hdims.data(), 4 * b);
    std::memcpy(p->h_offset_dims, odims.data(), 4 * b);

    std::vector<ModelParam> mp(static_cast<size_t>(b));
    for (int v = 0; v < b; ++v) {
        ModelParam& q = mp[static_cast<size_t>(v)];
        q.hash_base = hacc[static_cast<size_t>(v)];
        q.offset_base = oacc[static_cast<size_t>(v)];
        q.data_base = dacc[static_cast<size_t>(v)];
        q.m = hdims[static_cast<size_t>(v)];
        q.r = odims[static_cast<size_t>(v)];
        q.inv_m = 1.0f / static_cast<float>(q.m);
        q.inv_r = 1.0f / static_cast<float>(q.r);
    }
    p->models = static_cast<ModelParam*>(dev_alloc(sizeof(ModelParam) * b));
    cuda_check(cudaMemcpyAsync(p->models, mp.data(), sizeof(ModelParam) * b, cudaMemcpyHostToDevice, st), "upload");

    long long* d_hacc = static_cast<long long*>(dev_alloc(8 * (b + 1)));
    long long* d_oacc = static_cast<long long*>(dev_alloc(8 * (b + 1)));
    long long* d_dacc = static_cast<long long*>(dev_alloc(8 * (b + 1)));
    int* d_hd = static_cast<int*>(dev_alloc(4 * b));
    cuda_check(cudaMemcpyAsync(d_hacc, hacc.data(), 8 * (b + 1), cudaMemcpyHostToDevice, st), "upload");
    cuda_check(cudaMemcpyAsync(d_oacc, oacc.data(), 8 * (b + 1), cudaMemcpyHostToDevice, st), "upload");
    cuda_check(cudaMemcpyAsync(d_dacc, dacc.data(), 8 * (b + 1), cudaMemcpyHostToDevice, st), "upload");
    cuda_check(cudaMemcpyAsync(d_hd, hdims.data(), 4 * b, cudaMemcpyHostToDevice, st), "upload");

    const int T = 256;
    auto blocks = [&](long long n) { return static_cast<unsigned>((n + T - 1) / T); };
    if (!have_mos && d.M > 0) k_fill_model_of_slot<<<blocks(d.M), T, 0, st>>>(d_hacc, b, d.M, p->model_of_slot);
    p->slots = static_cast<uint2*>(dev_alloc(8 * d.M));
    p->phi = static_cast<unsigned*>(dev_alloc(4 * d.R));
    p->cols = static_cast<int4*>(dev_alloc(16 * d.N));
    if (d.M > 0) k_build_slots<<<blocks(d.M), T, 0, st>>>(p->hash, p->tags, d.M, d.dim, d.key_bits, p->slots);
    if (d.R > 0) k_build_phi<<<blocks(d.R), T, 0, st>>>(p->offsets, d.R, d.dim, d_oacc, d_hd, b, p->phi);
    if (d.M > 0)
        k_build_cols<<<blocks(d.M), T, 0, st>>>(p->hash, p->tags, p->model_of_slot, d_hacc, d_dacc, b, d.M, d.dim,
                                                p->cols);
    launched("super-PSH table kernels", (have_mos ? 0 : 1) + 3);
    cuda_check(cudaStreamSynchronize(st), "super-PSH upload");
    cudaFree(d_hacc);
    cudaFree(d_oacc);
    cudaFree(d_dacc);
    cudaFree(d_hd);
    d.slots = p->slots;
    d.phi = p->phi;
    d.models = p->models;
    d.cols = p->cols;
}

void release(hc_psh* p) {
    if (!p) return;
    cudaFree(p->hash);
    cudaFree(p->offsets);
    cudaFree(p->tags);
    cudaFree(p->model_of_slot);
    cudaFree(p->slots);
    cudaFree(p->phi);
    cudaFree(p->models);
    cudaFree(p->cols);
    delete[] p->h_hash_acc;
    delete[] p->h_offset_acc;
    delete[] p->h_data_acc;
    delete[] p->h_hash_dims;
    delete[] p->h_offset_dims;
    delete p;
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

const char* hc_last_error(void) { return g_last_error.c_str(); }
const char* hc_version(void) { return "hashconv_b200 0.1 (sm_100a)"; }
int64_t hc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
int64_t hc_fused_route_count(void) { return hcb::fused_route_count(0); }

hc_status hc_deferred_status(void) {
    if (g_deferred && *g_deferred) {
        *g_deferred = 0;
        set_last_error("unpool: switch index out of range");  // cnn_ops.cpp:331
        return HC_ERR_INVALID_ARGUMENT;
    }
    return HC_OK;
}

hc_status hc_malloc(void** ptr, size_t bytes) {
    return guard([&] { *ptr = dev_alloc(bytes); });
}
hc_status hc_free(void* ptr) {
    return guard([&] { cuda_check(cudaFree(ptr), "cudaFree"); });
}
hc_status hc_memcpy_h2d(void* dst, const void* src, size_t bytes, hc_stream stream) {
    return guard([&] {
        cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, reinterpret_cast<cudaStream_t>(stream)),
                   "H2D copy");
    });
}
hc_status hc_memcpy_d2h(void* dst, const void* src, size_t bytes, hc_stream stream) {
    return guard([&] {
        cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(stream)),
                   "D2H copy");
    });
}
hc_status hc_stream_synchronize(hc_stream stream) {
    return guard([&] { cuda_check(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)), "sync"); });
}
hc_status hc_set_math(hc_math mode) {
    if (mode != HC_MATH_EXACT && mode != HC_MATH_FAST && mode != HC_MATH_TF32) {
        set_last_error("unknown math mode");
        return HC_ERR_INVALID_ARGUMENT;
    }
    g_math = mode;
    return HC_OK;
}
hc_math hc_get_math(void) { return g_math; }

hc_status hc_psh_upload(const hc_super_psh_host* h, hc_psh** out, hc_stream stream) {
    hc_psh* p = nullptr;
    const hc_status st = guard([&] {
        if (!h || !out) throw std::invalid_argument("null argument");
        if (h->batch < 1) throw std::invalid_argument("batch must contain at least one model");
        const int b = h->batch, dim = h->dim;
        p = new hc_psh;
        DevPsh& d = p->d;
        d.dim = dim;
        d.resolution = h->resolution;
        d.batch = b;
        d.M = h->hash_acc[b];
        d.R = h->offset_acc[b];
        d.N = h->data_acc[b];
        cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
        p->hash = static_cast<int32_t*>(dev_alloc(4 * d.M));
        p->offsets = static_cast<uint8_t*>(dev_alloc(d.R * dim));
        p->tags = static_cast<uint16_t*>(dev_alloc(2 * d.M * dim));
        p->model_of_slot = static_cast<int32_t*>(dev_alloc(4 * d.M));
        cuda_check(cudaMemcpyAsync(p->hash, h->hash, 4 * d.M, cudaMemcpyHostToDevice, s), "upload H*");
        cuda_check(cudaMemcpyAsync(p->offsets, h->offsets, d.R * dim, cudaMemcpyHostToDevice, s), "upload Phi*");
        cuda_check(cudaMemcpyAsync(p->tags, h->tags, 2 * d.M * dim, cudaMemcpyHostToDevice, s), "upload T*");
        if (h->model_of_slot)
            cuda_check(cudaMemcpyAsync(p->model_of_slot, h->model_of_slot, 4 * d.M, cudaMemcpyHostToDevice, s),
                       "upload V*");
        std::vector<int64_t> hacc(h->hash_acc, h->hash_acc + b + 1), oacc(h->offset_acc, h->offset_acc + b + 1),
            dacc(h->data_acc, h->data_acc + b + 1);
        std::vector<int32_t> hd(h->hash_dims, h->hash_dims + b), od(h->offset_dims, h->offset_dims + b);
        finish_upload(p, hacc, oacc, dacc, hd, od, h->model_of_slot != nullptr, s);
        *out = p;
    });
    if (st != HC_OK) release(p);
    return st;
}

hc_status hc_psh_upload_levels(const hc_psh_level* const* levels, int32_t count, hc_psh** out, hc_stream stream) {
    hc_psh* p = nullptr;
    const hc_status st = guard([&] {
        // psh_batch.cpp:8-54 build_super checks
        if (count < 1) throw std::invalid_argument("batch must contain at least one model");
        const PshLevel& first = *levels[0];
        for (int32_t k = 0; k < count; ++k) {
            if (levels[k]->dim != first.dim || levels[k]->resolution != first.resolution)
                throw std::invalid_argument("mixed resolutions in one batch");
            if (levels[k]->channels != first.channels)
                throw std::invalid_argument("mixed channel counts in one batch");
        }
        const int dim = first.dim;
        std::vector<int64_t> hacc(count + 1, 0), oacc(count + 1, 0), dacc(count + 1, 0);
        std::vector<int32_t> hd, od;
        for (int32_t k = 0; k < count; ++k) {
            hacc[k + 1] = hacc[k] + levels[k]->slots();
            oacc[k + 1] = oacc[k] + levels[k]->cells();
            dacc[k + 1] = dacc[k] + levels[k]->n;
            hd.push_back(levels[k]->hash_dim);
            od.push_back(levels[k]->offset_dim);
        }
        p = new hc_psh;
        DevPsh& d = p->d;
        d.dim = dim;
        d.resolution = first.resolution;
        d.batch = count;
        d.M = hacc[count];
        d.R = oacc[count];
        d.N = dacc[count];
        cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
        p->hash = static_cast<int32_t*>(dev_alloc(4 * d.M));
        p->offsets = static_cast<uint8_t*>(dev_alloc(d.R * dim));
        p->tags = static_cast<uint16_t*>(dev_alloc(2 * d.M * dim));
        p->model_of_slot = static_cast<int32_t*>(dev_alloc(4 * d.M));
        // identical levels (replicated pyramids) are uploaded once per distinct pointer
        for (int32_t k = 0; k < count; ++k) {
            const PshLevel& l = *levels[k];
            cuda_check(cudaMemcpyAsync(p->hash + hacc[k], l.hash.data(), 4 * l.slots(), cudaMemcpyHostToDevice, s),
                       "upload H*");
            cuda_check(cudaMemcpyAsync(p->offsets + oacc[k] * dim, l.offsets.data(), l.cells() * dim,
                                       cudaMemcpyHostToDevice, s),
                       "upload Phi*");
            cuda_check(cudaMemcpyAsync(p->tags + hacc[k] * dim, l.tags.data(), 2 * l.slots() * dim,
                                       cudaMemcpyHostToDevice, s),
                       "upload T*");
        }
        finish_upload(p, hacc, oacc, dacc, hd, od, false, s);
        *out = p;
    });
    if (st != HC_OK) release(p);
    return st;
}

hc_status hc_psh_info(const hc_psh* p, int64_t info[6]) {
    if (!p) {
        set_last_error("null super-PSH handle");
        return HC_ERR_INVALID_ARGUMENT;
    }
    info[0] = p->d.dim;
    info[1] = p->d.resolution;
    info[2] = p->d.batch;
    info[3] = p->d.M;
    info[4] = p->d.R;
    info[5] = p->d.N;
    return HC_OK;
}

hc_status hc_psh_download(const hc_psh* p, int32_t* hash, uint8_t* offsets, uint16_t* tags, int32_t* model_of_slot,
                          int64_t* hash_acc, int64_t* offset_acc, int64_t* data_acc, int32_t* hash_dims,
                          int32_t* offset_dims) {
    return guard([&] {
        const DevPsh& d = p->d;
        const int b = d.batch;
        if (hash) cuda_check(cudaMemcpy(hash, p->hash, 4 * d.M, cudaMemcpyDeviceToHost), "download");
        if (offsets) cuda_check(cudaMemcpy(offsets, p->offsets, d.R * d.dim, cudaMemcpyDeviceToHost), "download");
        if (tags) cuda_check(cudaMemcpy(tags, p->tags, 2 * d.M * d.dim, cudaMemcpyDeviceToHost), "download");
        if (model_of_slot)
            cuda_check(cudaMemcpy(model_of_slot, p->model_of_slot, 4 * d.M, cudaMemcpyDeviceToHost), "download");
        if (hash_acc) std::memcpy(hash_acc, p->h_hash_acc, 8 * (b + 1));
        if (offset_acc) std::memcpy(offset_acc, p->h_offset_acc, 8 * (b + 1));
        if (data_acc) std::memcpy(data_acc, p->h_data_acc, 8 * (b + 1));
        if (hash_dims) std::memcpy(hash_dims, p->h_hash_dims, 4 * b);
        if (offset_dims) std::memcpy(offset_dims, p->h_offset_dims, 4 * b);
    });
}

// psh_batch.cpp:80-102 split_super: one host PshLevel per model, tables sliced by the
// prefix arrays; `data` (device, channels x N, optional) supplies each level's data rows.
hc_status hc_split_super(const hc_psh* p, const float* data, int64_t channels, hc_psh_level** out,
                         int32_t max_levels, int32_t* count) {
    return guard([&] {
        if (!p || !out || !count) throw std::invalid_argument("null argument");
        const DevPsh& d = p->d;
        const int b = d.batch, dim = d.dim;
        if (b > max_levels) throw std::invalid_argument("split_super: output array too small");
        std::vector<std::int32_t> hash(d.M);
        std::vector<std::uint8_t> offsets(d.R * dim);
        std::vector<std::uint16_t> tags(d.M * dim);
        if (d.M) cuda_check(cudaMemcpy(hash.data(), p->hash, 4 * d.M, cudaMemcpyDeviceToHost), "download");
        if (d.R) cuda_check(cudaMemcpy(offsets.data(), p->offsets, d.R * dim, cudaMemcpyDeviceToHost), "download");
        if (d.M) cuda_check(cudaMemcpy(tags.data(), p->tags, 2 * d.M * dim, cudaMemcpyDeviceToHost), "download");
        std::vector<float> hdata;
        if (data && channels > 0 && d.N > 0) {
            hdata.resize((size_t)(channels * d.N));
            cuda_check(cudaMemcpy(hdata.data(), data, 4 * channels * d.N, cudaMemcpyDeviceToHost), "download");
        }
        for (int k = 0; k < b; ++k) {
            auto* l = new hc_psh_level();
            l->dim = dim;
            l->resolution = d.resolution;
            const long long h0 = p->h_hash_acc[k], h1 = p->h_hash_acc[k + 1];
            const long long o0 = p->h_offset_acc[k], o1 = p->h_offset_acc[k + 1];
            const long long n0 = p->h_data_acc[k], n1 = p->h_data_acc[k + 1];
            l->n = n1 - n0;
            l->hash_dim = p->h_hash_dims[k];
            l->offset_dim = p->h_offset_dims[k];
            l->hash.assign(hash.begin() + h0, hash.begin() + h1);
            l->tags.assign(tags.begin() + h0 * dim, tags.begin() + h1 * dim);
            l->offsets.assign(offsets.begin() + o0 * dim, offsets.begin() + o1 * dim);
            if (!hdata.empty()) {
                l->channels = channels;
                l->data.resize((size_t)(channels * l->n));
                for (long long r = 0; r < channels; ++r)
                    std::copy(hdata.begin() + r * d.N + n0, hdata.begin() + r * d.N + n1,
                              l->data.begin() + r * l->n);
            }
            out[k] = l;
        }
        *count = b;
    });
}

hc_status hc_psh_columns(const hc_psh* p, const void** xyzm) {
    if (!p || !xyzm) {
        set_last_error("null argument");
        return HC_ERR_INVALID_ARGUMENT;
    }
    *xyzm = p->cols;
    return HC_OK;
}

hc_status hc_psh_free(hc_psh* p) {
    release(p);
    return HC_OK;
}

hc_status hc_locate(const hc_psh* p, const int32_t* queries, int64_t n, int64_t* result, hc_stream stream) {
    return guard([&] {
        if (!p) throw std::invalid_argument("null super-PSH handle");
        if (n <= 0) return;
        const int T = 256;
        k_locate<<<static_cast<unsigned>((n + T - 1) / T), T, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
            p->d, reinterpret_cast<const int4*>(queries), n, reinterpret_cast<long long*>(result));
        launched("hc_locate");
    });
}

}  // extern "C"
