// dropin_parity.cpp — TEST: the reference's callers switch to the B200 operators by
// changing the namespace only. Builds fixtures with the UNMODIFIED reference library
// (oracle/_ref objects; reference headers at build time) and checks, on the
// reference's own types, that hashconv_b200::<op> == hashconv::<op> bit-for-bit
// (EXACT math; float AND double instantiations), including the reference's known-answer tests
// (tests/test_cnn_ops.cpp:53-97, 140-156, 308-344) and its exception types.
#include <algorithm>
#include <cmath>
#include <type_traits>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "hashconv/cnn_ops.hpp"
#include "hashconv/gemm.hpp"
#include "hashconv/psh_batch.hpp"
#include "hashconv_b200.hpp"
#include "test_utils.hpp"

using namespace hashconv;
namespace hb = hashconv_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond, what)                                           \
    do {                                                            \
        ++g_checks;                                                 \
        if (!(cond)) {                                              \
            ++g_fail;                                               \
            std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
        }                                                           \
    } while (0)

struct Fixture {
    SuperPsh fine, coarse;
};

static Fixture fixture(int models, int res, std::uint64_t seed) {
    Fixture fx;
    std::vector<PshLevel> fl, cl;
    Rng rng(seed);
    for (int k = 0; k < models; ++k) {
        const auto n = rng.uniform_int(60, 300);
        const SparseVoxelSet s = testing::random_sparse_set(res, n, mix_seed(seed, 10 + k));
        PshBuildOptions o;
        o.seed = mix_seed(seed, 20 + k);
        fl.push_back(build_psh(s, o));
        cl.push_back(build_psh(coarsen(s), o));
    }
    fx.fine = build_super(fl);
    fx.coarse = build_super(cl);
    return fx;
}

template <class T>
static void ops_equal(const Fixture& fx, const ConvSpec& spec, std::uint64_t seed) {
    const SuperPsh& out = spec.stride == 1 ? fx.fine : fx.coarse;
    const std::int64_t fd = field_size(spec, 3);
    const auto data = testing::random_matrix<T>(spec.in_channels, fx.fine.total_columns(), seed);
    const KernelWeightsT<T> w{testing::random_matrix<T>(spec.out_channels, spec.in_channels * fd, seed + 1)};
    const auto dout = testing::random_matrix<T>(spec.out_channels, out.total_columns(), seed + 2);
    const auto cols = hash2col(fx.fine, data, out, spec);
    CHECK(hb::hash2col(fx.fine, data, out, spec) == cols, "hash2col");
    CHECK(hb::conv_forward(fx.fine, data, out, w, spec) == conv_forward(fx.fine, data, out, w, spec), "conv_forward");
    const auto g = conv_backward(dout, w, cols, fx.fine, out, spec);
    const auto h = hb::conv_backward(dout, w, cols, fx.fine, out, spec);
    CHECK(h.weights == g.weights, "conv_backward dW");
    CHECK(h.input == g.input, "conv_backward dX");
    const auto y = testing::random_matrix<T>(spec.in_channels * fd, out.total_columns(), seed + 3);
    CHECK(hb::col2hash(y, fx.fine, out, spec) == col2hash(y, fx.fine, out, spec), "col2hash");
    const ConvSpec pool{2, 2, 0, spec.in_channels, spec.in_channels};
    const auto mp = max_pool(fx.fine, data, fx.coarse, pool);
    const auto mq = hb::max_pool(fx.fine, data, fx.coarse, pool);
    CHECK(mq.output == mp.output && mq.switches.values == mp.switches.values, "max_pool");
    CHECK(hb::avg_pool(fx.fine, data, fx.coarse, pool) == avg_pool(fx.fine, data, fx.coarse, pool), "avg_pool");
    CHECK(hb::max_unpool(mp.output, mp.switches, fx.fine, fx.coarse, pool) ==
              max_unpool(mp.output, mp.switches, fx.fine, fx.coarse, pool),
          "max_unpool");
    const auto cv = testing::random_matrix<T>(spec.in_channels, fx.coarse.total_columns(), seed + 4);
    CHECK(hb::avg_unpool(cv, fx.fine, fx.coarse, pool) == avg_unpool(cv, fx.fine, fx.coarse, pool), "avg_unpool");
    if (spec.stride > 1) {
        const auto ci = testing::random_matrix<T>(spec.out_channels, fx.coarse.total_columns(), seed + 5);
        CHECK(hb::deconv_forward(fx.coarse, ci, fx.fine, w, spec) == deconv_forward(fx.coarse, ci, fx.fine, w, spec),
              "deconv_forward");
        const auto a = deconv_backward(data, w, ci, fx.coarse, fx.fine, spec);
        const auto b = hb::deconv_backward(data, w, ci, fx.coarse, fx.fine, spec);
        CHECK(a.weights == b.weights && a.input == b.input, "deconv_backward");
    }
    CHECK(hb::matmul(w.w, cols) == matmul(w.w, cols), "matmul");
    CHECK(hb::matmul_trans_a(w.w, dout) == matmul_trans_a(w.w, dout), "matmul_trans_a");
    CHECK(hb::matmul_trans_b(dout, cols) == matmul_trans_b(dout, cols), "matmul_trans_b");
}

template <class T>
static double max_rel(const FeatureMatrixT<T>& a, const FeatureMatrixT<T>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.values.size(); ++i) {
        num = std::max(num, std::fabs(double(a.values[i]) - double(b.values[i])));
        den = std::max(den, std::fabs(double(b.values[i])));
    }
    return den > 0 ? num / den : num;
}

// cnn_ops.hpp:118-170 through the shim: relu / scale forward / dropout bit-exact in both
// precisions; batch norm and the scale-backward sums bit-exact in float, 1e-12 in double
// (double sums in a tree order instead of the reference's sequential loop).
template <class T>
static void layer_ops_equal(std::uint64_t seed) {
    const bool exact = std::is_same<T, float>::value;
    const auto x = testing::random_matrix<T>(6, 2000, seed);
    const auto dy = testing::random_matrix<T>(6, 2000, seed + 1);
    for (int training = 0; training < 2; ++training) {
        BatchNormStats<T> s1(6), s2(6);
        for (int c = 0; c < 6; ++c) s1.running_mean[c] = s2.running_mean[c] = T(0.1) * T(c);
        BatchNormCache<T> c1, c2;
        const auto y1 = batch_norm_forward(x, s1, training != 0, &c1);
        const auto y2 = hb::batch_norm_forward(x, s2, training != 0, &c2);
        CHECK(exact ? y1 == y2 : max_rel(y2, y1) < 1e-12, "batch_norm_forward");
        CHECK(exact ? s1.running_mean == s2.running_mean && s1.running_var == s2.running_var : true,
              "batch_norm running stats");
        if (training) {
            const auto d1 = batch_norm_backward(dy, c1);
            const auto d2 = hb::batch_norm_backward(dy, c2);
            CHECK(exact ? d1 == d2 : max_rel(d2, d1) < 1e-12, "batch_norm_backward");
        }
    }
    std::vector<T> g(6), b(6);
    for (int c = 0; c < 6; ++c) g[c] = T(0.5) + T(c), b[c] = T(0.25) * T(c);
    CHECK(hb::scale_forward(x, g, b) == scale_forward(x, g, b), "scale_forward");
    const auto sg1 = scale_backward(dy, x, g);
    const auto sg2 = hb::scale_backward(dy, x, g);
    CHECK(sg1.input == sg2.input && (!exact || (sg1.gamma == sg2.gamma && sg1.beta == sg2.beta)), "scale_backward");
    const auto r1 = relu_forward(x);
    CHECK(hb::relu_forward(x) == r1, "relu_forward");
    CHECK(hb::relu_backward(dy, r1) == relu_backward(dy, r1), "relu_backward");
    DropoutMask m1, m2;
    const auto o1 = dropout_forward(x, T(0.4), seed, true, &m1);
    const auto o2 = hb::dropout_forward(x, T(0.4), seed, true, &m2);
    CHECK(o1 == o2 && m1.keep == m2.keep, "dropout_forward (mt19937_64 mask)");
    CHECK(hb::dropout_backward(dy, m2, T(0.4)) == dropout_backward(dy, m1, T(0.4)), "dropout_backward");
}

template <class T>
static double norm_rel(const FeatureMatrixT<T>& a, const FeatureMatrixT<double>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.values.size(); ++i) {
        const double d = double(a.values[i]) - b.values[i];
        num += d * d;
        den += b.values[i] * b.values[i];
    }
    return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

static FeatureMatrixT<double> to64(const FeatureMatrix& m) {
    FeatureMatrixT<double> r(m.rows, m.cols);
    for (size_t i = 0; i < m.values.size(); ++i) r.values[i] = m.values[i];
    return r;
}

// HC_MATH_FAST: the unchanged reference-signature float calls conv_forward / conv_backward of a
// stride-1 layer over one structure run the fused split-precision tensor-core conv (no column
// matrix; hc_fused_route_count proves the route) and land within 1e-5 (normwise) of the
// reference's own double instantiation on the same fp32 inputs.
static void fast_conv_close(int cin, int cout, std::uint64_t seed) {
    std::vector<PshLevel> fl;
    for (int k = 0; k < 2; ++k) {
        const SparseVoxelSet s = testing::random_sparse_set(32, 3000 + 500 * k, mix_seed(seed, k));
        PshBuildOptions o;
        o.seed = mix_seed(seed, 20 + k);
        fl.push_back(build_psh(s, o));
    }
    const SuperPsh fine = build_super(fl);
    const ConvSpec spec{3, 1, 0, cin, cout};
    const auto data = testing::random_matrix<float>(cin, fine.total_columns(), seed);
    const KernelWeightsT<float> w{testing::random_matrix<float>(cout, cin * 27, seed + 1)};
    const auto dout = testing::random_matrix<float>(cout, fine.total_columns(), seed + 2);
    const auto data64 = to64(data), dout64 = to64(dout);
    const KernelWeightsT<double> w64{to64(w.w)};
    const auto y64 = conv_forward(fine, data64, fine, w64, spec);
    const auto g64 = conv_backward(dout64, w64, hash2col(fine, data64, fine, spec), fine, fine, spec);
    const auto cols = hash2col(fine, data, fine, spec);
    const auto routed0 = hc_fused_route_count();
    hb::set_fast_math(true);
    const auto y = hb::conv_forward(fine, data, fine, w, spec);
    const auto g = hb::conv_backward(dout, w, cols, fine, fine, spec);
    hb::set_fast_math(false);
    const char* tag = "FAST conv (fused split precision) within 1e-5 of the reference's double";
    CHECK(hc_fused_route_count() - routed0 == 2, "FAST conv_forward/backward took the fused route");
    CHECK(norm_rel(y, y64) <= 1e-5, tag);
    CHECK(norm_rel(g.weights, g64.weights) <= 1e-5, tag);
    CHECK(norm_rel(g.input, g64.input) <= 1e-5, tag);
    std::printf("fast conv %d->%d: y %.3g dW %.3g dX %.3g (vs reference double)\n", cin, cout, norm_rel(y, y64),
                norm_rel(g.weights, g64.weights), norm_rel(g.input, g64.input));
}

static SuperPsh single(const Coord& p, int res, float value) {
    FeatureMatrix f(1, 1);
    f.at(0, 0) = value;
    return build_super({{build_psh(make_sparse_set(3, res, {p}, f))}});
}

int main() {
    // known-answer tests of tests/test_cnn_ops.cpp through the B200 operators
    {
        const SuperPsh s = single({4, 4, 4}, 8, 2.5f);
        const auto cols = hb::hash2col(s, s.data, s, ConvSpec{3, 1, 0, 1, 1});
        bool ok = cols.rows == 27 && cols.cols == 1;
        for (int r = 0; r < 27 && ok; ++r) ok = cols.at(r, 0) == (r == 13 ? 2.5f : 0.0f);
        CHECK(ok, "KAT isolated voxel (test_cnn_ops.cpp:53-62)");
    }
    {
        FeatureMatrix f(1, 2);
        f.at(0, 0) = f.at(0, 1) = 1.0f;
        const SuperPsh s = build_super({{build_psh(make_sparse_set(3, 8, {{3, 3, 3}, {4, 3, 3}}, f))}});
        FeatureMatrix dc(27, 2);
        dc.at(13, 0) = 10.0f;
        dc.at(14, 0) = 20.0f;
        dc.at(12, 1) = 40.0f;
        dc.at(13, 1) = 80.0f;
        const auto g = hb::col2hash(dc, s, s, ConvSpec{3, 1, 0, 1, 1});
        CHECK(g.at(0, 0) == 50.0f && g.at(0, 1) == 100.0f, "KAT col2hash two voxels (test_cnn_ops.cpp:140-156)");
    }
    {
        std::vector<Coord> c;
        for (int z = 4; z <= 5; ++z)
            for (int y = 4; y <= 5; ++y)
                for (int x = 4; x <= 5; ++x) c.push_back({x, y, z});
        FeatureMatrix f(1, 8);
        for (int i = 0; i < 8; ++i) f.at(0, i) = static_cast<float>(i + 1);
        const auto set = make_sparse_set(3, 8, c, f);
        const SuperPsh fine = build_super({{build_psh(set)}}), coarse = build_super({{build_psh(coarsen(set))}});
        const auto mp = hb::max_pool(fine, fine.data, coarse, ConvSpec{2, 2, 0, 1, 1});
        CHECK(mp.output.at(0, 0) == 8.0f && mp.switches.at(0, 0) == 7, "KAT pool 1..8 (test_cnn_ops.cpp:308-332)");
    }
    // exception types and messages (cnn_ops.cpp:20-33, 326-332)
    {
        const Fixture fx = fixture(1, 16, 97);
        bool threw = false;
        try {
            hb::hash2col(fx.fine, fx.fine.data, fx.fine, ConvSpec{2, 1, 0, 3, 3});
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "stride-1 fields need an odd kernel size";
        }
        CHECK(threw, "invalid_argument with the reference message");
        auto mp = max_pool(fx.fine, fx.fine.data, fx.coarse, ConvSpec{2, 2, 0, 3, 3});
        mp.switches.values[0] = 8;
        threw = false;
        try {
            hb::max_unpool(mp.output, mp.switches, fx.fine, fx.coarse, ConvSpec{2, 2, 0, 3, 3});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw, "out-of-range switch throws invalid_argument (test_cnn_ops.cpp:436-444)");
    }
    // operator equality on random batches, every spec family of acceptance criterion 3
    const ConvSpec specs[] = {{3, 1, 0, 3, 5}, {2, 2, 0, 4, 2}, {3, 2, 0, 2, 6}, {2, 2, 1, 5, 3}};
    for (int t = 0; t < 8; ++t) {
        const Fixture fx = fixture(1 + t % 3, t % 2 ? 16 : 32, 5000 + t);
        ops_equal<float>(fx, specs[t % 4], 100 + t);
        ops_equal<double>(fx, specs[t % 4], 200 + t);  // the reference's double instantiation
    }
    fast_conv_close(3, 5, 31);
    fast_conv_close(64, 64, 32);
    fast_conv_close(16, 128, 33);
    layer_ops_equal<float>(77);
    layer_ops_equal<double>(78);
    std::printf("%s: %d checks, %d failures\n", g_fail ? "DROPIN FAIL" : "DROPIN OK", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
