// hashconv_b200.hpp — header-only C++ drop-in for the reference operator surface.
//
// Same names, argument order, return-by-value and exception types as
// proj/include/hashconv/cnn_ops.hpp and gemm.hpp, executed on the B200 through the
// C ABI (hashconv_b200.h). The functions are templates over the caller's own types,
// so existing code built on the reference's SuperPsh / FeatureMatrixT<float> /
// KernelWeightsT<float> / ConvSpec keeps compiling:
//
//     #include "hashconv/cnn_ops.hpp"      // reference types
//     #include "hashconv_b200.hpp"         // B200 operators
//     auto cols = hashconv_b200::hash2col(in, data, out, spec);   // == hashconv::hash2col
//
// Requirements on the types (exactly the reference's members):
//   Super: dim, resolution, batch, hash, offsets, tags, model_of_slot, hash_acc,
//          offset_acc, data_acc, hash_dims, offset_dims (std::vector-like .data()/.size())
//   Mat:   rows, cols, values (contiguous float or double), constructor Mat(rows, cols)
//   Spec:  kernel, stride, pad, in_channels, out_channels
//   W:     member `w` of type Mat
// Every call uploads its inputs, runs the kernels and downloads the result (the
// reference's host-memory contract); callers that keep data on the device use the C
// ABI directly (device super-PSH handles, device pointers, streams).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <memory>
#include <vector>

#include "hashconv_b200.h"

namespace hashconv_b200 {

namespace detail {

inline void check(hc_status s) {
    if (s == HC_OK) return;
    const std::string msg = hc_last_error();
    if (s == HC_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// element type of a Mat (its `values` container)
template <class Mat>
using value_t = typename std::decay<decltype(std::declval<Mat>().values[0])>::type;

// RAII device buffer
class Buf {
   public:
    explicit Buf(size_t bytes) { check(hc_malloc(&p_, bytes ? bytes : 16)); }
    ~Buf() {
        if (p_) hc_free(p_);
    }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    Buf(Buf&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
    template <class T>
    T* as() const {
        return static_cast<T*>(p_);
    }

   private:
    void* p_ = nullptr;
};

template <class T>
inline Buf upload(const T* host, size_t count) {
    Buf b(sizeof(T) * count);
    check(hc_memcpy_h2d(b.as<void>(), host, sizeof(T) * count, nullptr));
    return b;
}

template <class Mat>
inline Buf upload(const Mat& m) {
    return upload(m.values.data(), static_cast<size_t>(m.rows * m.cols));
}

template <class Mat>
inline Mat download(const Buf& b, std::int64_t rows, std::int64_t cols) {
    Mat m(rows, cols);
    check(hc_memcpy_d2h(m.values.data(), b.as<void>(), sizeof(value_t<Mat>) * static_cast<size_t>(rows * cols),
                        nullptr));
    check(hc_stream_synchronize(nullptr));
    return m;
}

// A super-PSH uploaded for the duration of one call.
class Structure {
   public:
    template <class Super>
    explicit Structure(const Super& s) {
        hc_super_psh_host h{};
        h.dim = s.dim;
        h.resolution = s.resolution;
        h.batch = s.batch;
        h.hash = s.hash.data();
        h.offsets = s.offsets.data();
        h.tags = s.tags.data();
        h.model_of_slot = s.model_of_slot.empty() ? nullptr : s.model_of_slot.data();
        h.hash_acc = reinterpret_cast<const int64_t*>(s.hash_acc.data());
        h.offset_acc = reinterpret_cast<const int64_t*>(s.offset_acc.data());
        h.data_acc = reinterpret_cast<const int64_t*>(s.data_acc.data());
        h.hash_dims = s.hash_dims.data();
        h.offset_dims = s.offset_dims.data();
        check(hc_psh_upload(&h, &p_, nullptr));
    }
    ~Structure() {
        if (p_) hc_psh_free(p_);
    }
    Structure(const Structure&) = delete;
    Structure& operator=(const Structure&) = delete;
    const hc_psh* get() const { return p_; }
    std::int64_t columns() const {
        int64_t info[6];
        check(hc_psh_info(p_, info));
        return info[5];
    }
    int dim() const {
        int64_t info[6];
        check(hc_psh_info(p_, info));
        return static_cast<int>(info[0]);
    }

   private:
    hc_psh* p_ = nullptr;
};

// The reference instantiates every operator for float and double (cnn_ops.cpp:652-653,
// gemm.cpp:117-118); the C ABI has one entry point per precision.
template <class T>
struct abi;
template <>
struct abi<float> {
    static constexpr auto batch_norm_forward = hc_batch_norm_forward_f32;
    static constexpr auto batch_norm_backward = hc_batch_norm_backward_f32;
    static constexpr auto scale_forward = hc_scale_forward_f32;
    static constexpr auto scale_backward = hc_scale_backward_f32;
    static constexpr auto relu_forward = hc_relu_forward_f32;
    static constexpr auto relu_backward = hc_relu_backward_f32;
    static constexpr auto dropout_forward = hc_dropout_forward_f32;
    static constexpr auto dropout_backward = hc_dropout_backward_f32;
    static constexpr auto hash2col = hc_hash2col_f32;
    static constexpr auto col2hash = hc_col2hash_f32;
    static constexpr auto conv_forward = hc_conv_forward_f32;
    static constexpr auto conv_backward = hc_conv_backward_f32;
    static constexpr auto max_pool = hc_max_pool_f32;
    static constexpr auto avg_pool = hc_avg_pool_f32;
    static constexpr auto max_unpool = hc_max_unpool_f32;
    static constexpr auto avg_unpool = hc_avg_unpool_f32;
    static constexpr auto deconv_forward = hc_deconv_forward_f32;
    static constexpr auto deconv_backward = hc_deconv_backward_f32;
    static constexpr auto matmul = hc_matmul_f32;
    static constexpr auto matmul_trans_a = hc_matmul_trans_a_f32;
    static constexpr auto matmul_trans_b = hc_matmul_trans_b_f32;
};
template <>
struct abi<double> {
    static constexpr auto batch_norm_forward = hc_batch_norm_forward_f64;
    static constexpr auto batch_norm_backward = hc_batch_norm_backward_f64;
    static constexpr auto scale_forward = hc_scale_forward_f64;
    static constexpr auto scale_backward = hc_scale_backward_f64;
    static constexpr auto relu_forward = hc_relu_forward_f64;
    static constexpr auto relu_backward = hc_relu_backward_f64;
    static constexpr auto dropout_forward = hc_dropout_forward_f64;
    static constexpr auto dropout_backward = hc_dropout_backward_f64;
    static constexpr auto hash2col = hc_hash2col_f64;
    static constexpr auto col2hash = hc_col2hash_f64;
    static constexpr auto conv_forward = hc_conv_forward_f64;
    static constexpr auto conv_backward = hc_conv_backward_f64;
    static constexpr auto max_pool = hc_max_pool_f64;
    static constexpr auto avg_pool = hc_avg_pool_f64;
    static constexpr auto max_unpool = hc_max_unpool_f64;
    static constexpr auto avg_unpool = hc_avg_unpool_f64;
    static constexpr auto deconv_forward = hc_deconv_forward_f64;
    static constexpr auto deconv_backward = hc_deconv_backward_f64;
    static constexpr auto matmul = hc_matmul_f64;
    static constexpr auto matmul_trans_a = hc_matmul_trans_a_f64;
    static constexpr auto matmul_trans_b = hc_matmul_trans_b_f64;
};

template <class Spec>
inline hc_conv_spec spec_of(const Spec& s) {
    return hc_conv_spec{s.kernel, s.stride, s.pad, s.in_channels, s.out_channels};
}

inline std::int64_t field_size(const hc_conv_spec& s, int dim) {
    std::int64_t v = 1;
    for (int a = 0; a < dim; ++a) v *= s.kernel;
    return v;
}

}  // namespace detail

// cnn_ops.hpp:48-52 / 62-79 result types (same member names as the reference's)
template <class Mat>
struct ConvGradients {
    Mat weights;
    Mat input;
};

struct PoolSwitches {
    std::int64_t rows = 0;
    std::int64_t cols = 0;
    std::vector<std::int32_t> values;
    std::int32_t& at(std::int64_t r, std::int64_t c) { return values[static_cast<size_t>(r * cols + c)]; }
    const std::int32_t& at(std::int64_t r, std::int64_t c) const { return values[static_cast<size_t>(r * cols + c)]; }
};

template <class Mat>
struct MaxPoolResult {
    Mat output;
    PoolSwitches switches;
};

// Math mode of the contraction: exact (reference order, bit-identical) or fast.
inline void set_fast_math(bool fast) { detail::check(hc_set_math(fast ? HC_MATH_FAST : HC_MATH_EXACT)); }
// Any hc_math mode (EXACT / FAST = 3xTF32 / TF32), thread-local like the C ABI.
inline void set_math(hc_math mode) { detail::check(hc_set_math(mode)); }

// cnn_ops.cpp:123-158
template <class Super, class Mat, class Spec>
Mat hash2col(const Super& input, const Mat& input_data, const Super& output, const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure in(input), out(output);
    const hc_conv_spec sp = detail::spec_of(spec);
    const std::int64_t rows = sp.in_channels * detail::field_size(sp, in.dim()), cols = out.columns();
    auto d = detail::upload(input_data);
    detail::Buf r(sizeof(T) * static_cast<size_t>(rows * cols));
    detail::check(detail::abi<T>::hash2col(in.get(), d.template as<T>(), input_data.rows, input_data.cols, out.get(), sp,
                                  r.as<T>(), nullptr));
    return detail::download<Mat>(r, rows, cols);
}

// cnn_ops.cpp:160-204
template <class Super, class Mat, class Spec>
Mat col2hash(const Mat& col_grads, const Super& input, const Super& output, const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure in(input), out(output);
    const hc_conv_spec sp = detail::spec_of(spec);
    auto g = detail::upload(col_grads);
    detail::Buf r(sizeof(T) * static_cast<size_t>(sp.in_channels * in.columns()));
    detail::check(detail::abi<T>::col2hash(g.template as<T>(), col_grads.rows, col_grads.cols, in.get(), out.get(), sp,
                                  r.as<T>(), nullptr));
    return detail::download<Mat>(r, sp.in_channels, in.columns());
}

// cnn_ops.cpp:206-215
// A stride-1 layer over ONE structure (&input == &output, as net.cpp:196-197 calls it) uploads
// it once: the library sees one handle, which is what routes HC_MATH_FAST float calls to the
// fused split-precision tensor-core conv (no column matrix).
template <class Super, class Mat, class W, class Spec>
Mat conv_forward(const Super& input, const Mat& input_data, const Super& output, const W& weights, const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure in(input);
    const bool same = static_cast<const void*>(&input) == static_cast<const void*>(&output);
    std::unique_ptr<detail::Structure> out_own(same ? nullptr : new detail::Structure(output));
    const detail::Structure& out = same ? in : *out_own;
    const hc_conv_spec sp = detail::spec_of(spec);
    auto d = detail::upload(input_data);
    auto w = detail::upload(weights.w);
    detail::Buf r(sizeof(T) * static_cast<size_t>(sp.out_channels * out.columns()));
    detail::check(detail::abi<T>::conv_forward(in.get(), d.template as<T>(), input_data.rows, input_data.cols, out.get(),
                                      w.template as<T>(), weights.w.rows, weights.w.cols, sp, r.as<T>(),
                                      nullptr));
    return detail::download<Mat>(r, sp.out_channels, out.columns());
}

// cnn_ops.cpp:217-232
template <class Mat, class W, class Super, class Spec>
ConvGradients<Mat> conv_backward(const Mat& output_grad, const W& weights, const Mat& cached_cols, const Super& input,
                                 const Super& output, const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure in(input);
    const bool same = static_cast<const void*>(&input) == static_cast<const void*>(&output);
    std::unique_ptr<detail::Structure> out_own(same ? nullptr : new detail::Structure(output));
    const detail::Structure& out = same ? in : *out_own;
    const hc_conv_spec sp = detail::spec_of(spec);
    auto g = detail::upload(output_grad);
    auto w = detail::upload(weights.w);
    auto c = detail::upload(cached_cols);
    detail::Buf dw(sizeof(T) * static_cast<size_t>(output_grad.rows * cached_cols.rows));
    detail::Buf dx(sizeof(T) * static_cast<size_t>(sp.in_channels * in.columns()));
    detail::check(detail::abi<T>::conv_backward(g.template as<T>(), output_grad.rows, output_grad.cols,
                                       w.template as<T>(), weights.w.rows, weights.w.cols, c.template as<T>(),
                                       cached_cols.rows, cached_cols.cols, in.get(), out.get(), sp, dw.as<T>(),
                                       dx.as<T>(), nullptr));
    return ConvGradients<Mat>{detail::download<Mat>(dw, output_grad.rows, cached_cols.rows),
                              detail::download<Mat>(dx, sp.in_channels, in.columns())};
}

// cnn_ops.cpp:234-284
template <class Super, class Mat, class Spec>
MaxPoolResult<Mat> max_pool(const Super& input, const Mat& input_data, const Super& output, const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure in(input), out(output);
    const hc_conv_spec sp = detail::spec_of(spec);
    const std::int64_t n = out.columns();
    auto d = detail::upload(input_data);
    detail::Buf r(sizeof(T) * static_cast<size_t>(sp.in_channels * n));
    detail::Buf s(sizeof(std::int32_t) * static_cast<size_t>(sp.in_channels * n));
    detail::check(detail::abi<T>::max_pool(in.get(), d.template as<T>(), input_data.rows, input_data.cols, out.get(), sp,
                                  r.as<T>(), s.as<std::int32_t>(), nullptr));
    MaxPoolResult<Mat> res;
    res.switches.rows = sp.in_channels;
    res.switches.cols = n;
    res.switches.values.resize(static_cast<size_t>(sp.in_channels * n));
    detail::check(hc_memcpy_d2h(res.switches.values.data(), s.as<void>(), res.switches.values.size() * 4, nullptr));
    res.output = detail::download<Mat>(r, sp.in_channels, n);
    return res;
}

// cnn_ops.cpp:286-322
template <class Super, class Mat, class Spec>
Mat avg_pool(const Super& input, const Mat& input_data, const Super& output, const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure in(input), out(output);
    const hc_conv_spec sp = detail::spec_of(spec);
    auto d = detail::upload(input_data);
    detail::Buf r(sizeof(T) * static_cast<size_t>(sp.in_channels * out.columns()));
    detail::check(detail::abi<T>::avg_pool(in.get(), d.template as<T>(), input_data.rows, input_data.cols, out.get(), sp,
                                  r.as<T>(), nullptr));
    return detail::download<Mat>(r, sp.in_channels, out.columns());
}

// cnn_ops.cpp:336-372
template <class Mat, class Switches, class Super, class Spec>
Mat max_unpool(const Mat& coarse_data, const Switches& switches, const Super& fine, const Super& coarse,
               const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure f(fine), c(coarse);
    const hc_conv_spec sp = detail::spec_of(spec);
    auto d = detail::upload(coarse_data);
    auto s = detail::upload(switches.values.data(), switches.values.size());
    detail::Buf r(sizeof(T) * static_cast<size_t>(sp.in_channels * f.columns()));
    detail::check(detail::abi<T>::max_unpool(d.template as<T>(), coarse_data.rows, coarse_data.cols,
                                    s.template as<std::int32_t>(), switches.rows, switches.cols, f.get(), c.get(), sp,
                                    r.as<T>(), nullptr));
    Mat out = detail::download<Mat>(r, sp.in_channels, f.columns());  // synchronises
    detail::check(hc_deferred_status());  // an out-of-range switch throws invalid_argument here
    return out;
}

// cnn_ops.cpp:374-406
template <class Mat, class Super, class Spec>
Mat avg_unpool(const Mat& coarse_data, const Super& fine, const Super& coarse, const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure f(fine), c(coarse);
    const hc_conv_spec sp = detail::spec_of(spec);
    auto d = detail::upload(coarse_data);
    detail::Buf r(sizeof(T) * static_cast<size_t>(sp.in_channels * f.columns()));
    detail::check(detail::abi<T>::avg_unpool(d.template as<T>(), coarse_data.rows, coarse_data.cols, f.get(), c.get(), sp,
                                    r.as<T>(), nullptr));
    return detail::download<Mat>(r, sp.in_channels, f.columns());
}

// cnn_ops.cpp:408-419
template <class Super, class Mat, class W, class Spec>
Mat deconv_forward(const Super& coarse, const Mat& coarse_data, const Super& fine, const W& weights,
                   const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure c(coarse), f(fine);
    const hc_conv_spec sp = detail::spec_of(spec);
    auto d = detail::upload(coarse_data);
    auto w = detail::upload(weights.w);
    detail::Buf r(sizeof(T) * static_cast<size_t>(sp.in_channels * f.columns()));
    detail::check(detail::abi<T>::deconv_forward(c.get(), d.template as<T>(), coarse_data.rows, coarse_data.cols, f.get(),
                                        w.template as<T>(), weights.w.rows, weights.w.cols, sp, r.as<T>(),
                                        nullptr));
    return detail::download<Mat>(r, sp.in_channels, f.columns());
}

// cnn_ops.cpp:421-435
template <class Mat, class W, class Super, class Spec>
ConvGradients<Mat> deconv_backward(const Mat& fine_grad, const W& weights, const Mat& cached_coarse_data,
                                   const Super& coarse, const Super& fine, const Spec& spec) {
    using T = detail::value_t<Mat>;
    detail::Structure c(coarse), f(fine);
    const hc_conv_spec sp = detail::spec_of(spec);
    auto g = detail::upload(fine_grad);
    auto w = detail::upload(weights.w);
    auto cd = detail::upload(cached_coarse_data);
    const std::int64_t k = sp.in_channels * detail::field_size(sp, f.dim());
    detail::Buf dw(sizeof(T) * static_cast<size_t>(cached_coarse_data.rows * k));
    detail::Buf dx(sizeof(T) * static_cast<size_t>(weights.w.rows * c.columns()));
    detail::check(detail::abi<T>::deconv_backward(g.template as<T>(), fine_grad.rows, fine_grad.cols,
                                         w.template as<T>(), weights.w.rows, weights.w.cols,
                                         cd.template as<T>(), cached_coarse_data.rows, cached_coarse_data.cols,
                                         c.get(), f.get(), sp, dw.as<T>(), dx.as<T>(), nullptr));
    return ConvGradients<Mat>{detail::download<Mat>(dw, cached_coarse_data.rows, k),
                              detail::download<Mat>(dx, weights.w.rows, c.columns())};
}

// gemm.cpp:71-93
template <class Mat>
Mat matmul(const Mat& a, const Mat& b) {
    using T = detail::value_t<Mat>;
    if (a.cols != b.rows) throw std::invalid_argument("matmul: shape mismatch");
    auto da = detail::upload(a), db = detail::upload(b);
    detail::Buf c(sizeof(T) * static_cast<size_t>(a.rows * b.cols));
    detail::check(detail::abi<T>::matmul(da.template as<T>(), db.template as<T>(), c.as<T>(), a.rows, a.cols,
                                b.cols, nullptr));
    return detail::download<Mat>(c, a.rows, b.cols);
}

template <class Mat>
Mat matmul_trans_a(const Mat& a, const Mat& b) {
    using T = detail::value_t<Mat>;
    if (a.rows != b.rows) throw std::invalid_argument("matmul_trans_a: shape mismatch");
    auto da = detail::upload(a), db = detail::upload(b);
    detail::Buf c(sizeof(T) * static_cast<size_t>(a.cols * b.cols));
    detail::check(detail::abi<T>::matmul_trans_a(da.template as<T>(), db.template as<T>(), c.as<T>(), a.rows,
                                        a.cols, b.cols, nullptr));
    return detail::download<Mat>(c, a.cols, b.cols);
}

template <class Mat>
Mat matmul_trans_b(const Mat& a, const Mat& b) {
    using T = detail::value_t<Mat>;
    if (a.cols != b.cols) throw std::invalid_argument("matmul_trans_b: shape mismatch");
    auto da = detail::upload(a), db = detail::upload(b);
    detail::Buf c(sizeof(T) * static_cast<size_t>(a.rows * b.rows));
    detail::check(detail::abi<T>::matmul_trans_b(da.template as<T>(), db.template as<T>(), c.as<T>(), a.rows,
                                        a.cols, b.rows, nullptr));
    return detail::download<Mat>(c, a.rows, b.rows);
}

// cnn_ops.hpp:118-170 — batch norm, scale, ReLU, inverted dropout (cnn_ops.cpp:437-608).
// Stats / Cache / Mask are the caller's types with the reference's members
// (running_mean, running_var, eps, momentum / normalized, inv_std / keep).
template <class Mat>
struct ScaleGradients {
    std::vector<detail::value_t<Mat>> gamma;
    std::vector<detail::value_t<Mat>> beta;
    Mat input;
};

namespace detail {
template <class V>
inline Buf upload_vec(const V& v) {
    return upload(v.data(), v.size());
}
template <class T>
inline std::vector<T> download_vec(const Buf& b, size_t n) {
    std::vector<T> v(n);
    if (n) check(hc_memcpy_d2h(v.data(), b.as<void>(), sizeof(T) * n, nullptr));
    check(hc_stream_synchronize(nullptr));
    return v;
}
}  // namespace detail

template <class Mat, class Stats, class Cache = std::nullptr_t>
Mat batch_norm_forward(const Mat& x, Stats& stats, bool training, Cache* cache = nullptr) {
    using T = detail::value_t<Mat>;
    auto d = detail::upload(x);
    auto rm = detail::upload_vec(stats.running_mean), rv = detail::upload_vec(stats.running_var);
    detail::Buf y(sizeof(T) * static_cast<size_t>(x.rows * x.cols)), inv(sizeof(T) * static_cast<size_t>(x.rows));
    detail::check(detail::abi<T>::batch_norm_forward(d.template as<T>(), x.rows, x.cols, rm.template as<T>(),
                                                     rv.template as<T>(),
                                                     static_cast<std::int64_t>(stats.running_mean.size()),
                                                     stats.eps, stats.momentum, training ? 1 : 0, y.as<T>(),
                                                     inv.as<T>(), nullptr));
    if (training) {
        stats.running_mean = detail::download_vec<T>(rm, stats.running_mean.size());
        stats.running_var = detail::download_vec<T>(rv, stats.running_var.size());
    }
    Mat out = detail::download<Mat>(y, x.rows, x.cols);
    if constexpr (!std::is_same<Cache, std::nullptr_t>::value) {
        if (cache) {
            cache->normalized = out;
            cache->inv_std = detail::download_vec<T>(inv, static_cast<size_t>(x.rows));
        }
    }
    return out;
}

template <class Mat, class Cache>
Mat batch_norm_backward(const Mat& dy, const Cache& cache) {
    using T = detail::value_t<Mat>;
    auto d = detail::upload(dy), xh = detail::upload(cache.normalized), inv = detail::upload_vec(cache.inv_std);
    detail::Buf dx(sizeof(T) * static_cast<size_t>(dy.rows * dy.cols));
    detail::check(detail::abi<T>::batch_norm_backward(d.template as<T>(), dy.rows, dy.cols, xh.template as<T>(),
                                                      cache.normalized.rows, cache.normalized.cols,
                                                      inv.template as<T>(), dx.as<T>(), nullptr));
    return detail::download<Mat>(dx, dy.rows, dy.cols);
}

template <class Mat, class V>
Mat scale_forward(const Mat& x, const V& gamma, const V& beta) {
    using T = detail::value_t<Mat>;
    auto d = detail::upload(x), g = detail::upload_vec(gamma), b = detail::upload_vec(beta);
    detail::Buf y(sizeof(T) * static_cast<size_t>(x.rows * x.cols));
    detail::check(detail::abi<T>::scale_forward(d.template as<T>(), x.rows, x.cols, g.template as<T>(),
                                                static_cast<std::int64_t>(gamma.size()), b.template as<T>(),
                                                static_cast<std::int64_t>(beta.size()), y.as<T>(), nullptr));
    return detail::download<Mat>(y, x.rows, x.cols);
}

template <class Mat, class V>
ScaleGradients<Mat> scale_backward(const Mat& dy, const Mat& x, const V& gamma) {
    using T = detail::value_t<Mat>;
    auto d = detail::upload(dy), xx = detail::upload(x), g = detail::upload_vec(gamma);
    detail::Buf dg(sizeof(T) * static_cast<size_t>(dy.rows)), db(sizeof(T) * static_cast<size_t>(dy.rows));
    detail::Buf dx(sizeof(T) * static_cast<size_t>(dy.rows * dy.cols));
    detail::check(detail::abi<T>::scale_backward(d.template as<T>(), xx.template as<T>(), dy.rows, dy.cols,
                                                 g.template as<T>(), dg.as<T>(), db.as<T>(), dx.as<T>(), nullptr));
    ScaleGradients<Mat> r;
    r.gamma = detail::download_vec<T>(dg, static_cast<size_t>(dy.rows));
    r.beta = detail::download_vec<T>(db, static_cast<size_t>(dy.rows));
    r.input = detail::download<Mat>(dx, dy.rows, dy.cols);
    return r;
}

template <class Mat>
Mat relu_forward(const Mat& x) {
    using T = detail::value_t<Mat>;
    auto d = detail::upload(x);
    detail::Buf y(sizeof(T) * static_cast<size_t>(x.rows * x.cols));
    detail::check(detail::abi<T>::relu_forward(d.template as<T>(), x.rows * x.cols, y.as<T>(), nullptr));
    return detail::download<Mat>(y, x.rows, x.cols);
}

template <class Mat>
Mat relu_backward(const Mat& dy, const Mat& forward_out) {
    using T = detail::value_t<Mat>;
    auto d = detail::upload(dy), f = detail::upload(forward_out);
    detail::Buf dx(sizeof(T) * static_cast<size_t>(dy.rows * dy.cols));
    detail::check(detail::abi<T>::relu_backward(d.template as<T>(), dy.rows, dy.cols, f.template as<T>(),
                                                forward_out.rows, forward_out.cols, dx.as<T>(), nullptr));
    return detail::download<Mat>(dx, dy.rows, dy.cols);
}

template <class Mat, class T, class Mask = std::nullptr_t>
Mat dropout_forward(const Mat& x, T ratio, std::uint64_t seed, bool training, Mask* mask = nullptr) {
    using V = detail::value_t<Mat>;
    const std::int64_t total = x.rows * x.cols;
    auto d = detail::upload(x);
    detail::Buf y(sizeof(V) * static_cast<size_t>(total)), keep(static_cast<size_t>(total));
    detail::check(detail::abi<V>::dropout_forward(d.template as<V>(), total, static_cast<V>(ratio), seed,
                                                  training ? 1 : 0, y.as<V>(), keep.as<std::uint8_t>(), nullptr));
    if constexpr (!std::is_same<Mask, std::nullptr_t>::value) {
        if (mask) mask->keep = detail::download_vec<std::uint8_t>(keep, static_cast<size_t>(total));
    }
    return detail::download<Mat>(y, x.rows, x.cols);
}

template <class Mat, class Mask, class T>
Mat dropout_backward(const Mat& dy, const Mask& mask, T ratio) {
    using V = detail::value_t<Mat>;
    const std::int64_t total = dy.rows * dy.cols;
    auto d = detail::upload(dy), k = detail::upload_vec(mask.keep);
    detail::Buf dx(sizeof(V) * static_cast<size_t>(total));
    detail::check(detail::abi<V>::dropout_backward(d.template as<V>(), total, k.template as<std::uint8_t>(),
                                                   static_cast<std::int64_t>(mask.keep.size()), static_cast<V>(ratio),
                                                   dx.as<V>(), nullptr));
    return detail::download<Mat>(dx, dy.rows, dy.cols);
}

}  // namespace hashconv_b200
