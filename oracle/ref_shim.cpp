// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle). A flat extern "C" surface
// over the *unmodified* reference library (/root/reference/proj, compiled by
// oracle/Makefile into oracle/_ref/), so pytest / golden-fixture scripts /
// bench.py's cpu_baseline leg can drive the reference through ctypes.
//
// Nothing in the product (paper_1803_11385_b200/) links or loads this file.
// Every entry point forwards to exactly one reference API call; the mapping is
// given in the comment above each function (reference file:line).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "hashconv/bench.hpp"
#include "hashconv/cnn_ops.hpp"
#include "hashconv/gemm.hpp"
#include "hashconv/net.hpp"
#include "hashconv/psh.hpp"
#include "hashconv/psh_batch.hpp"
#include "hashconv/psh_io.hpp"
#include "hashconv/serial_ref.hpp"
#include "hashconv/threading.hpp"
#include "hashconv/voxel.hpp"
#include "test_utils.hpp"  // reference tests/test_utils.hpp: random_sparse_set, random_matrix

using namespace hashconv;

namespace {

thread_local std::string g_err;

// 0 ok, 1 std::invalid_argument, 2 std::runtime_error / other
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

template <class T>
FeatureMatrixT<T> wrap(const T* p, std::int64_t rows, std::int64_t cols) {
    FeatureMatrixT<T> m(rows, cols);
    if (rows * cols) std::memcpy(m.values.data(), p, sizeof(T) * static_cast<size_t>(rows * cols));
    return m;
}

template <class T>
void out(const FeatureMatrixT<T>& m, T* dst) {
    if (!m.values.empty()) std::memcpy(dst, m.values.data(), sizeof(T) * m.values.size());
}

ConvSpec spec_of(const int* s) { return ConvSpec{s[0], s[1], s[2], s[3], s[4]}; }

const SuperPsh& S(const void* h) { return *static_cast<const SuperPsh*>(h); }

}  // namespace

extern "C" {

// ---------------------------------------------------------------- plumbing
int hcref_last_error(char* buf, int n) {
    if (n > 0) {
        std::strncpy(buf, g_err.c_str(), static_cast<size_t>(n - 1));
        buf[n - 1] = 0;
    }
    return static_cast<int>(g_err.size());
}
// threading.cpp:33 set_thread_override / threading.cpp:24 max_threads
void hcref_set_threads(int n) { set_thread_override(n); }
int hcref_max_threads() { return max_threads(); }

// ---------------------------------------------------------------- voxel sets
// bench.cpp:33 sphere_voxels
void* hcref_set_sphere(int res, int shell) {
    void* r = nullptr;
    guarded([&] { r = new SparseVoxelSet(sphere_voxels(res, shell != 0)); });
    return r;
}
// tests/test_utils.hpp:14 random_sparse_set
void* hcref_set_random(int res, std::int64_t n, std::uint64_t seed, int channels, int unit_normals) {
    void* r = nullptr;
    guarded([&] {
        r = new SparseVoxelSet(testing::random_sparse_set(res, n, seed, channels, unit_normals != 0));
    });
    return r;
}
// voxel.cpp:76 make_sparse_set
void* hcref_set_make(int dim, int res, std::int64_t n, const std::int32_t* coords, int channels,
                     const float* features) {
    void* r = nullptr;
    guarded([&] {
        std::vector<Coord> c(static_cast<size_t>(n));
        for (std::int64_t i = 0; i < n; ++i)
            c[static_cast<size_t>(i)] = {coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
        r = new SparseVoxelSet(make_sparse_set(dim, res, std::move(c), wrap(features, channels, n)));
    });
    return r;
}
// voxel.cpp:218 coarsen
void* hcref_set_coarsen(const void* set) {
    void* r = nullptr;
    guarded([&] { r = new SparseVoxelSet(coarsen(*static_cast<const SparseVoxelSet*>(set))); });
    return r;
}
void hcref_set_info(const void* set, std::int64_t* info /*dim,res,n,channels*/) {
    const auto& s = *static_cast<const SparseVoxelSet*>(set);
    info[0] = s.dim;
    info[1] = s.resolution;
    info[2] = s.count();
    info[3] = s.features.rows;
}
void hcref_set_copy(const void* set, std::int32_t* coords, float* features) {
    const auto& s = *static_cast<const SparseVoxelSet*>(set);
    for (size_t i = 0; i < s.voxels.size(); ++i)
        for (int a = 0; a < 3; ++a) coords[3 * i + a] = s.voxels[i][static_cast<size_t>(a)];
    out(s.features, features);
}
void hcref_set_free(void* set) { delete static_cast<SparseVoxelSet*>(set); }

// ---------------------------------------------------------------- PSH levels
// psh.cpp:179 build_psh (optionally with injected offsets, psh.hpp:55-58)
void* hcref_psh_build(const void* set, std::uint64_t seed, const std::uint8_t* injected,
                      std::int64_t injected_len, int injected_dim) {
    void* r = nullptr;
    guarded([&] {
        PshBuildOptions o;
        o.seed = seed;
        std::vector<std::uint8_t> inj;
        if (injected) {
            inj.assign(injected, injected + injected_len);
            o.injected_offsets = &inj;
            o.injected_offset_dim = injected_dim;
        }
        r = new PshLevel(build_psh(*static_cast<const SparseVoxelSet*>(set), o));
    });
    return r;
}
// psh.hpp:21-35 PshLevel fields
void hcref_psh_info(const void* h, std::int64_t* info /*dim,res,n,m,r,channels*/) {
    const auto& l = *static_cast<const PshLevel*>(h);
    info[0] = l.dim;
    info[1] = l.resolution;
    info[2] = l.n;
    info[3] = l.hash_dim;
    info[4] = l.offset_dim;
    info[5] = l.data.rows;
}
void hcref_psh_copy(const void* h, std::int32_t* hash, std::uint8_t* offsets, std::uint16_t* tags,
                    float* data) {
    const auto& l = *static_cast<const PshLevel*>(h);
    std::memcpy(hash, l.hash.data(), l.hash.size() * 4);
    std::memcpy(offsets, l.offsets.data(), l.offsets.size());
    std::memcpy(tags, l.tags.data(), l.tags.size() * 2);
    out(l.data, data);
}
// psh.cpp:250 validate -> number of violations
int hcref_psh_validate(const void* h, const void* set) {
    return static_cast<int>(
        validate(*static_cast<const PshLevel*>(h), *static_cast<const SparseVoxelSet*>(set)).size());
}
// psh.cpp:239 query (-1 when empty)
std::int64_t hcref_psh_query(const void* h, int x, int y, int z) {
    const auto r = query(*static_cast<const PshLevel*>(h), Coord{x, y, z});
    return r ? *r : -1;
}
// psh.cpp:229 hash_slot
std::int64_t hcref_psh_hash_slot(const void* h, int x, int y, int z) {
    return hash_slot(*static_cast<const PshLevel*>(h), Coord{x, y, z});
}
void hcref_psh_free(void* h) { delete static_cast<PshLevel*>(h); }
// psh_io.cpp:92 write_psh_file
int hcref_psh_write_file(const char* path, const void* const* levels, int count) {
    return guarded([&] {
        std::vector<PshLevel> v;
        for (int i = 0; i < count; ++i) v.push_back(*static_cast<const PshLevel*>(levels[i]));
        write_psh_file(path, v);
    });
}
// psh_io.cpp:98 read_psh_file -> number of levels, handles written to out[]
int hcref_psh_read_file(const char* path, void** out_levels, int max_levels) {
    int n = -1;
    guarded([&] {
        auto v = read_psh_file(path);
        n = static_cast<int>(v.size());
        for (int i = 0; i < n && i < max_levels; ++i) out_levels[i] = new PshLevel(std::move(v[static_cast<size_t>(i)]));
    });
    return n;
}

// ---------------------------------------------------------------- super-PSH
// psh_batch.cpp:8 build_super
void* hcref_super_build(const void* const* levels, int count) {
    void* r = nullptr;
    guarded([&] {
        std::vector<PshLevel> v;
        for (int i = 0; i < count; ++i) v.push_back(*static_cast<const PshLevel*>(levels[i]));
        r = new SuperPsh(build_super(v));
    });
    return r;
}
// Rebuild a SuperPsh from flat arrays (any producer) so reference ops can run on
// tables made by the product's own builder. Field meaning: psh_batch.hpp:15-38.
void* hcref_super_from_arrays(int dim, int res, int batch, const std::int32_t* hash,
                              const std::uint8_t* offsets, const std::uint16_t* tags,
                              const std::int32_t* model_of_slot, const std::int64_t* hash_acc,
                              const std::int64_t* offset_acc, const std::int64_t* data_acc,
                              const std::int32_t* hash_dims, const std::int32_t* offset_dims,
                              int channels, const float* data) {
    auto* s = new SuperPsh;
    s->dim = dim;
    s->resolution = res;
    s->batch = batch;
    const std::int64_t M = hash_acc[batch], R = offset_acc[batch], N = data_acc[batch];
    s->hash.assign(hash, hash + M);
    s->offsets.assign(offsets, offsets + R * dim);
    s->tags.assign(tags, tags + M * dim);
    s->model_of_slot.assign(model_of_slot, model_of_slot + M);
    s->hash_acc.assign(hash_acc, hash_acc + batch + 1);
    s->offset_acc.assign(offset_acc, offset_acc + batch + 1);
    s->data_acc.assign(data_acc, data_acc + batch + 1);
    s->hash_dims.assign(hash_dims, hash_dims + batch);
    s->offset_dims.assign(offset_dims, offset_dims + batch);
    s->data = data ? wrap(data, channels, N) : FeatureMatrix(channels, N);
    return s;
}
void hcref_super_info(const void* h, std::int64_t* info /*dim,res,batch,M,R,N,channels*/) {
    const auto& s = S(h);
    info[0] = s.dim;
    info[1] = s.resolution;
    info[2] = s.batch;
    info[3] = s.total_slots();
    info[4] = s.offset_acc.back();
    info[5] = s.total_columns();
    info[6] = s.data.rows;
}
void hcref_super_copy(const void* h, std::int32_t* hash, std::uint8_t* offsets, std::uint16_t* tags,
                      std::int32_t* model_of_slot, std::int64_t* hash_acc, std::int64_t* offset_acc,
                      std::int64_t* data_acc, std::int32_t* hash_dims, std::int32_t* offset_dims,
                      float* data) {
    const auto& s = S(h);
    std::memcpy(hash, s.hash.data(), s.hash.size() * 4);
    std::memcpy(offsets, s.offsets.data(), s.offsets.size());
    std::memcpy(tags, s.tags.data(), s.tags.size() * 2);
    std::memcpy(model_of_slot, s.model_of_slot.data(), s.model_of_slot.size() * 4);
    std::memcpy(hash_acc, s.hash_acc.data(), s.hash_acc.size() * 8);
    std::memcpy(offset_acc, s.offset_acc.data(), s.offset_acc.size() * 8);
    std::memcpy(data_acc, s.data_acc.data(), s.data_acc.size() * 8);
    std::memcpy(hash_dims, s.hash_dims.data(), s.hash_dims.size() * 4);
    std::memcpy(offset_dims, s.offset_dims.data(), s.offset_dims.size() * 4);
    if (data) out(s.data, data);
}
void hcref_super_free(void* h) { delete static_cast<SuperPsh*>(h); }
// psh_batch.cpp:56 locate (-1 when absent)
std::int64_t hcref_locate(const void* h, int model, int x, int y, int z) {
    const auto r = locate(S(h), model, Coord{x, y, z});
    return r ? *r : -1;
}

// ---------------------------------------------------------------- fixtures
// rng.hpp:28-37 Rng::uniform_int drawn in sequence from one stream (e.g. the
// parameter draws of tests/acceptance.cpp:174-203 make_instance).
void hcref_rng_draws(std::uint64_t seed, int count, const std::int64_t* lo, const std::int64_t* hi,
                     std::int64_t* out) {
    Rng rng(seed);
    for (int i = 0; i < count; ++i) out[i] = rng.uniform_int(lo[i], hi[i]);
}
// tests/test_utils.hpp:41 random_matrix
void hcref_random_matrix_f32(std::int64_t rows, std::int64_t cols, std::uint64_t seed, float lo,
                             float hi, float* dst) {
    out(testing::random_matrix<float>(rows, cols, seed, lo, hi), dst);
}
void hcref_random_matrix_f64(std::int64_t rows, std::int64_t cols, std::uint64_t seed, double lo,
                             double hi, double* dst) {
    out(testing::random_matrix<double>(rows, cols, seed, lo, hi), dst);
}

// ---------------------------------------------------------------- operators
#define HCREF_OPS(T, SUF)                                                                         \
    /* cnn_ops.cpp:123 hash2col */                                                                \
    int hcref_hash2col_##SUF(const void* in, const T* data, std::int64_t dr, std::int64_t dc,     \
                             const void* outs, const int* spec, T* cols) {                        \
        return guarded([&] { out(hash2col(S(in), wrap(data, dr, dc), S(outs), spec_of(spec)), cols); }); \
    }                                                                                             \
    /* cnn_ops.cpp:160 col2hash */                                                                \
    int hcref_col2hash_##SUF(const T* g, std::int64_t gr, std::int64_t gc, const void* in,        \
                             const void* outs, const int* spec, T* res) {                         \
        return guarded([&] { out(col2hash(wrap(g, gr, gc), S(in), S(outs), spec_of(spec)), res); }); \
    }                                                                                             \
    /* cnn_ops.cpp:206 conv_forward */                                                            \
    int hcref_conv_forward_##SUF(const void* in, const T* data, std::int64_t dr, std::int64_t dc, \
                                 const void* outs, const T* w, std::int64_t wr, std::int64_t wc,  \
                                 const int* spec, T* res) {                                       \
        return guarded([&] {                                                                      \
            KernelWeightsT<T> kw{wrap(w, wr, wc)};                                                \
            out(conv_forward(S(in), wrap(data, dr, dc), S(outs), kw, spec_of(spec)), res);        \
        });                                                                                       \
    }                                                                                             \
    /* cnn_ops.cpp:217 conv_backward */                                                           \
    int hcref_conv_backward_##SUF(const T* dout, std::int64_t gr, std::int64_t gc, const T* w,    \
                                  std::int64_t wr, std::int64_t wc, const T* cols,                \
                                  std::int64_t cr, std::int64_t cc, const void* in,               \
                                  const void* outs, const int* spec, T* dw, T* dx) {              \
        return guarded([&] {                                                                      \
            KernelWeightsT<T> kw{wrap(w, wr, wc)};                                                \
            auto g = conv_backward(wrap(dout, gr, gc), kw, wrap(cols, cr, cc), S(in), S(outs),    \
                                   spec_of(spec));                                                \
            out(g.weights, dw);                                                                   \
            out(g.input, dx);                                                                     \
        });                                                                                       \
    }                                                                                             \
    /* cnn_ops.cpp:234 max_pool */                                                                \
    int hcref_max_pool_##SUF(const void* in, const T* data, std::int64_t dr, std::int64_t dc,     \
                             const void* outs, const int* spec, T* res, std::int32_t* sw) {       \
        return guarded([&] {                                                                      \
            auto r = max_pool(S(in), wrap(data, dr, dc), S(outs), spec_of(spec));                 \
            out(r.output, res);                                                                   \
            std::memcpy(sw, r.switches.values.data(), r.switches.values.size() * 4);              \
        });                                                                                       \
    }                                                                                             \
    /* cnn_ops.cpp:286 avg_pool */                                                                \
    int hcref_avg_pool_##SUF(const void* in, const T* data, std::int64_t dr, std::int64_t dc,     \
                             const void* outs, const int* spec, T* res) {                         \
        return guarded([&] { out(avg_pool(S(in), wrap(data, dr, dc), S(outs), spec_of(spec)), res); }); \
    }                                                                                             \
    /* cnn_ops.cpp:336 max_unpool */                                                              \
    int hcref_max_unpool_##SUF(const T* coarse, std::int64_t cr, std::int64_t cc,                 \
                               const std::int32_t* sw, std::int64_t sr, std::int64_t sc,          \
                               const void* fine, const void* coarse_s, const int* spec, T* res) { \
        return guarded([&] {                                                                      \
            PoolSwitches p;                                                                       \
            p.rows = sr;                                                                          \
            p.cols = sc;                                                                          \
            p.values.assign(sw, sw + sr * sc);                                                    \
            out(max_unpool(wrap(coarse, cr, cc), p, S(fine), S(coarse_s), spec_of(spec)), res);   \
        });                                                                                       \
    }                                                                                             \
    /* cnn_ops.cpp:374 avg_unpool */                                                              \
    int hcref_avg_unpool_##SUF(const T* coarse, std::int64_t cr, std::int64_t cc,                 \
                               const void* fine, const void* coarse_s, const int* spec, T* res) { \
        return guarded([&] {                                                                      \
            out(avg_unpool(wrap(coarse, cr, cc), S(fine), S(coarse_s), spec_of(spec)), res);      \
        });                                                                                       \
    }                                                                                             \
    /* cnn_ops.cpp:408 deconv_forward */                                                          \
    int hcref_deconv_forward_##SUF(const void* coarse, const T* data, std::int64_t dr,            \
                                   std::int64_t dc, const void* fine, const T* w,                 \
                                   std::int64_t wr, std::int64_t wc, const int* spec, T* res) {   \
        return guarded([&] {                                                                      \
            KernelWeightsT<T> kw{wrap(w, wr, wc)};                                                \
            out(deconv_forward(S(coarse), wrap(data, dr, dc), S(fine), kw, spec_of(spec)), res);  \
        });                                                                                       \
    }                                                                                             \
    /* cnn_ops.cpp:421 deconv_backward */                                                         \
    int hcref_deconv_backward_##SUF(const T* fg, std::int64_t gr, std::int64_t gc, const T* w,    \
                                    std::int64_t wr, std::int64_t wc, const T* cd,                \
                                    std::int64_t cr, std::int64_t cc, const void* coarse,         \
                                    const void* fine, const int* spec, T* dw, T* dx) {            \
        return guarded([&] {                                                                      \
            KernelWeightsT<T> kw{wrap(w, wr, wc)};                                                \
            auto g = deconv_backward(wrap(fg, gr, gc), kw, wrap(cd, cr, cc), S(coarse), S(fine),  \
                                     spec_of(spec));                                              \
            out(g.weights, dw);                                                                   \
            out(g.input, dx);                                                                     \
        });                                                                                       \
    }                                                                                             \
    /* gemm.cpp:71-93 matmul / matmul_trans_a / matmul_trans_b */                                 \
    int hcref_matmul_##SUF(const T* a, std::int64_t ar, std::int64_t ac, const T* b,              \
                           std::int64_t br, std::int64_t bc, T* c) {                              \
        return guarded([&] { out(matmul(wrap(a, ar, ac), wrap(b, br, bc)), c); });               \
    }                                                                                             \
    int hcref_matmul_trans_a_##SUF(const T* a, std::int64_t ar, std::int64_t ac, const T* b,      \
                                   std::int64_t br, std::int64_t bc, T* c) {                      \
        return guarded([&] { out(matmul_trans_a(wrap(a, ar, ac), wrap(b, br, bc)), c); });       \
    }                                                                                             \
    int hcref_matmul_trans_b_##SUF(const T* a, std::int64_t ar, std::int64_t ac, const T* b,      \
                                   std::int64_t br, std::int64_t bc, T* c) {                      \
        return guarded([&] { out(matmul_trans_b(wrap(a, ar, ac), wrap(b, br, bc)), c); });       \
    }

HCREF_OPS(float, f32)
HCREF_OPS(double, f64)

// cnn_ops.cpp:437-608: batch norm, scale, relu, dropout (test oracle for ops_layer.cu)
#define HCREF_LAYER(T, SUF)                                                                        \
    int hcref_bn_forward_##SUF(const T* x, std::int64_t c, std::int64_t n, T* rm, T* rv, T eps, T mom, \
                               int training, T* y, T* inv_std) {                                   \
        return guarded([&] {                                                                       \
            BatchNormStats<T> st(c);                                                               \
            std::memcpy(st.running_mean.data(), rm, sizeof(T) * c);                                \
            std::memcpy(st.running_var.data(), rv, sizeof(T) * c);                                 \
            st.eps = eps;                                                                          \
            st.momentum = mom;                                                                     \
            BatchNormCache<T> cache;                                                               \
            out(batch_norm_forward(wrap(x, c, n), st, training != 0, &cache), y);                  \
            std::memcpy(rm, st.running_mean.data(), sizeof(T) * c);                                \
            std::memcpy(rv, st.running_var.data(), sizeof(T) * c);                                 \
            std::memcpy(inv_std, cache.inv_std.data(), sizeof(T) * cache.inv_std.size());          \
        });                                                                                        \
    }                                                                                              \
    int hcref_bn_backward_##SUF(const T* dy, std::int64_t c, std::int64_t n, const T* xh,          \
                                const T* inv_std, T* dx) {                                         \
        return guarded([&] {                                                                       \
            BatchNormCache<T> cache;                                                               \
            cache.normalized = wrap(xh, c, n);                                                     \
            cache.inv_std.assign(inv_std, inv_std + c);                                            \
            out(batch_norm_backward(wrap(dy, c, n), cache), dx);                                   \
        });                                                                                        \
    }                                                                                              \
    int hcref_scale_backward_##SUF(const T* dy, const T* x, std::int64_t r, std::int64_t c,        \
                                   const T* gamma, T* dg, T* db, T* dx) {                          \
        return guarded([&] {                                                                       \
            auto g = scale_backward(wrap(dy, r, c), wrap(x, r, c), std::vector<T>(gamma, gamma + r)); \
            std::memcpy(dg, g.gamma.data(), sizeof(T) * r);                                        \
            std::memcpy(db, g.beta.data(), sizeof(T) * r);                                         \
            out(g.input, dx);                                                                      \
        });                                                                                        \
    }                                                                                              \
    int hcref_scale_forward_##SUF(const T* x, std::int64_t r, std::int64_t c, const T* g, const T* b, T* y) { \
        return guarded([&] {                                                                       \
            out(scale_forward(wrap(x, r, c), std::vector<T>(g, g + r), std::vector<T>(b, b + r)), y); \
        });                                                                                        \
    }                                                                                              \
    int hcref_relu_##SUF(const T* x, std::int64_t r, std::int64_t c, const T* dy, T* y, T* dx) {   \
        return guarded([&] {                                                                       \
            const auto fo = relu_forward(wrap(x, r, c));                                           \
            out(fo, y);                                                                            \
            out(relu_backward(wrap(dy, r, c), fo), dx);                                            \
        });                                                                                        \
    }                                                                                              \
    int hcref_dropout_##SUF(const T* x, std::int64_t r, std::int64_t c, T ratio, std::uint64_t seed, \
                            int training, const T* dy, T* y, std::uint8_t* keep, T* dx) {          \
        return guarded([&] {                                                                       \
            DropoutMask m;                                                                         \
            out(dropout_forward(wrap(x, r, c), ratio, seed, training != 0, &m), y);                \
            std::memcpy(keep, m.keep.data(), m.keep.size());                                       \
            out(dropout_backward(wrap(dy, r, c), m, ratio), dx);                                   \
        });                                                                                        \
    }

HCREF_LAYER(float, f32)
HCREF_LAYER(double, f64)

// serial_ref.cpp:33-171 (paper-literal task loops; float only)
int hcref_serial_hash2col(const void* in, const float* data, std::int64_t dr, std::int64_t dc,
                          const void* outs, const int* spec, float* cols) {
    return guarded([&] { out(serial::hash2col_ref(S(in), wrap(data, dr, dc), S(outs), spec_of(spec)), cols); });
}
int hcref_serial_col2hash(const float* g, std::int64_t gr, std::int64_t gc, const void* in,
                          const void* outs, const int* spec, float* res) {
    return guarded([&] { out(serial::col2hash_ref(wrap(g, gr, gc), S(in), S(outs), spec_of(spec)), res); });
}
int hcref_serial_max_pool(const void* in, const float* data, std::int64_t dr, std::int64_t dc,
                          const void* outs, const int* spec, float* res, std::int32_t* sw) {
    return guarded([&] {
        auto r = serial::max_pool_ref(S(in), wrap(data, dr, dc), S(outs), spec_of(spec));
        out(r.output, res);
        std::memcpy(sw, r.switches.values.data(), r.switches.values.size() * 4);
    });
}

// ---------------------------------------------------------------- net (net.cpp)
// net.cpp:135-180 make_graph<float>
void* hcref_net_make(int level_max, int classes, std::uint64_t seed, int input_channels) {
    void* r = nullptr;
    guarded([&] { r = new LayerGraph(make_graph<float>(level_max, classes, seed, input_channels)); });
    return r;
}
void hcref_net_free(void* g) { delete static_cast<LayerGraph*>(g); }
int hcref_net_blocks(const void* g) { return (int)static_cast<const LayerGraph*>(g)->blocks.size(); }
// block i conv weights (rows x cols = C_out x C_in*27, KernelWeightsT layout cnn_ops.hpp:21-27)
void hcref_net_conv_shape(const void* g, int i, std::int64_t* rc) {
    const auto& w = static_cast<const LayerGraph*>(g)->blocks[i].conv.w;
    rc[0] = w.rows;
    rc[1] = w.cols;
}
void hcref_net_get_conv(const void* g, int i, float* w) { out(static_cast<const LayerGraph*>(g)->blocks[i].conv.w, w); }
void hcref_net_get_bn(const void* g, int i, float* mean, float* var) {
    const auto& bn = static_cast<const LayerGraph*>(g)->blocks[i].bn;
    std::memcpy(mean, bn.running_mean.data(), bn.running_mean.size() * 4);
    std::memcpy(var, bn.running_var.data(), bn.running_var.size() * 4);
}
void hcref_net_get_fc(const void* g, float* w1, float* b1, float* w2, float* b2) {
    const auto* G = static_cast<const LayerGraph*>(g);
    out(G->fc1.weights, w1);
    std::memcpy(b1, G->fc1.bias.data(), G->fc1.bias.size() * 4);
    out(G->fc2.weights, w2);
    std::memcpy(b2, G->fc2.bias.data(), G->fc2.bias.size() * 4);
}
void hcref_net_set_dropout(void* g, float ratio) { static_cast<LayerGraph*>(g)->dropout_ratio = ratio; }
// net.cpp:260-323 net_loss_and_gradients, training mode (running stats updated); the batch
// is the given super-PSH levels (finest first, finest carrying the input data array).
// conv_grads: the blocks' C_out x C_in*27 gradients concatenated.
int hcref_net_loss_grads(void* g, const void* const* levels, int nlevels, const int* labels, int b, float* loss,
                         float* conv_grads, float* fc1w, float* fc1b, float* fc2w, float* fc2b) {
    return guarded([&] {
        auto* G = static_cast<LayerGraph*>(g);
        MultiLevelBatch batch;
        for (int i = 0; i < nlevels; ++i) batch.levels.push_back(S(levels[i]));
        NetRunOptions opt;
        opt.training = true;
        opt.update_running_stats = true;
        NetGradientsT<float> grads;
        *loss = net_loss_and_gradients(*G, batch, std::vector<int>(labels, labels + b), opt, &grads);
        float* dst = conv_grads;
        for (const auto& m : grads.conv) {
            out(m, dst);
            dst += m.values.size();
        }
        out(grads.fc1_w, fc1w);
        std::memcpy(fc1b, grads.fc1_b.data(), grads.fc1_b.size() * 4);
        out(grads.fc2_w, fc2w);
        std::memcpy(fc2b, grads.fc2_b.data(), grads.fc2_b.size() * 4);
    });
}

// net.cpp:181-258 net_forward<float>; training = 0: running statistics, dropout off.
// scores: classes x b.
int hcref_net_forward(void* g, const void* const* levels, int nlevels, int training, float* scores) {
    return guarded([&] {
        auto* G = static_cast<LayerGraph*>(g);
        MultiLevelBatch batch;
        for (int i = 0; i < nlevels; ++i) batch.levels.push_back(S(levels[i]));
        NetRunOptions opt;
        opt.training = training != 0;
        opt.update_running_stats = training != 0;
        out(net_forward(*G, batch, opt), scores);
    });
}

}  // extern "C"
