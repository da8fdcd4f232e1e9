// host_psh.cpp — host-side input producers of the framework (not the GPU hot path).
//
// These restate the reference producers so the framework can make its own
// perfect-spatial-hash tables and synthetic shells without the reference
// library: sphere_voxels (bench.cpp:33-77), make_sparse_set (voxel.cpp:76-110),
// coarsen (voxel.cpp:218-268), the greedy PSH construction (psh.cpp:31-227) and
// the ".psh" container (psh_io.cpp:45-90). The construction follows the same
// deterministic decisions (cell order, seeded reuse probes, exhaustive scan
// order), so the tables are byte-identical to the reference's for the same
// (set, seed) — tests/test_host_psh.py checks that against oracle/_ref.
// The candidate test is re-engineered for speed: per-voxel p mod m_bar is
// precomputed once instead of per probe.
//
// Compiled with -ffp-contract=off and no -march so float feature arithmetic
// rounds exactly like the reference build.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <random>

#include "hc_internal.h"

namespace hcb {

std::int64_t ipow(std::int64_t b, int e) {
    std::int64_t r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}
std::int64_t PshLevel::slots() const { return ipow(hash_dim, dim); }
std::int64_t PshLevel::cells() const { return ipow(offset_dim, dim); }

namespace {

// types.hpp:57-61, x fastest
inline std::int64_t flat(const Coord& p, std::int64_t e, int dim) {
    std::int64_t f = 0;
    for (int a = dim - 1; a >= 0; --a) f = f * e + p[static_cast<size_t>(a)];
    return f;
}
inline Coord unflat(std::int64_t f, std::int64_t e, int dim) {
    Coord p{0, 0, 0};
    for (int a = 0; a < dim; ++a) {
        p[static_cast<size_t>(a)] = static_cast<std::int32_t>(f % e);
        f /= e;
    }
    return p;
}
inline bool zyx_less(const Coord& a, const Coord& b) {
    if (a[2] != b[2]) return a[2] < b[2];
    if (a[1] != b[1]) return a[1] < b[1];
    return a[0] < b[0];
}

// rng.hpp:12-58 — mt19937_64 stream + the reference's distribution helpers.
struct Stream {
    std::mt19937_64 eng;
    explicit Stream(std::uint64_t s) : eng(s) {}
    std::int64_t uniform_int(std::int64_t lo, std::int64_t hi) {
        const std::uint64_t span = static_cast<std::uint64_t>(hi - lo) + 1;
        if (span == 0) return static_cast<std::int64_t>(eng());
        const std::uint64_t limit = UINT64_MAX - UINT64_MAX % span;
        std::uint64_t v;
        do v = eng();
        while (v >= limit);
        return lo + static_cast<std::int64_t>(v % span);
    }
};

std::uint64_t splitmix(std::uint64_t seed, std::uint64_t item) {
    std::uint64_t z = seed + 0x9E3779B97F4A7C15ull * (item + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void check_resolution(std::int32_t res) {
    // voxel.cpp (check_resolution): power of two in [4, 65536]
    if (res < 4 || res > 65536 || (res & (res - 1)) != 0)
        throw std::invalid_argument("resolution must be a power of two in [4, 65536]");
}

// ------------------------------------------------------------------ greedy build
struct Off {
    std::uint8_t v[3] = {0, 0, 0};
    bool operator==(const Off& o) const { return v[0] == o.v[0] && v[1] == o.v[1] && v[2] == o.v[2]; }
};

// psh.cpp:31-138 try_build: fixed (m_bar, r_bar) greedy attempt.
bool greedy_attempt(const VoxelSet& s, std::int32_t m, std::int32_t r, std::uint64_t seed,
                    std::vector<std::int32_t>& hash, std::vector<std::uint8_t>& offsets,
                    std::vector<std::uint16_t>& tags) {
    const int dim = s.dim;
    const std::int64_t slots = ipow(m, dim), cells = ipow(r, dim);
    const std::int64_t n = s.count();

    // per-voxel residues mod m_bar, computed once
    std::vector<std::array<std::int32_t, 3>> res_m(static_cast<size_t>(n));
    std::vector<std::int64_t> cell_of(static_cast<size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) {
        const Coord& p = s.voxels[static_cast<size_t>(i)];
        Coord h1{0, 0, 0};
        for (int a = 0; a < dim; ++a) {
            res_m[static_cast<size_t>(i)][static_cast<size_t>(a)] = p[static_cast<size_t>(a)] % m;
            h1[static_cast<size_t>(a)] = p[static_cast<size_t>(a)] % r;
        }
        for (int a = dim; a < 3; ++a) res_m[static_cast<size_t>(i)][static_cast<size_t>(a)] = 0;
        cell_of[static_cast<size_t>(i)] = flat(h1, r, dim);
    }
    // bucket voxels per offset cell (CSR), voxel ids ascending inside a bucket
    std::vector<std::int64_t> start(static_cast<size_t>(cells + 1), 0);
    for (std::int64_t i = 0; i < n; ++i) ++start[static_cast<size_t>(cell_of[static_cast<size_t>(i)] + 1)];
    for (std::int64_t c = 0; c < cells; ++c) start[static_cast<size_t>(c + 1)] += start[static_cast<size_t>(c)];
    std::vector<std::int32_t> members(static_cast<size_t>(n));
    {
        std::vector<std::int64_t> fill(start.begin(), start.end() - 1);
        for (std::int64_t i = 0; i < n; ++i)
            members[static_cast<size_t>(fill[static_cast<size_t>(cell_of[static_cast<size_t>(i)])]++)] =
                static_cast<std::int32_t>(i);
    }
    // cells by decreasing load, ties by ascending cell index (stable)
    std::vector<std::int64_t> order;
    for (std::int64_t c = 0; c < cells; ++c)
        if (start[static_cast<size_t>(c + 1)] > start[static_cast<size_t>(c)]) order.push_back(c);
    std::stable_sort(order.begin(), order.end(), [&](std::int64_t a, std::int64_t b) {
        return start[static_cast<size_t>(a + 1)] - start[static_cast<size_t>(a)] >
               start[static_cast<size_t>(b + 1)] - start[static_cast<size_t>(b)];
    });

    hash.assign(static_cast<size_t>(slots), -1);
    tags.assign(static_cast<size_t>(slots * dim), 0xFFFF);
    offsets.assign(static_cast<size_t>(cells * dim), 0);

    Stream rng(seed);
    std::vector<Off> used;
    std::vector<std::int32_t> perm;
    constexpr int kReuseProbes = 64;  // psh.cpp:87
    const std::int32_t lim = std::min<std::int32_t>(m, 256);

    std::vector<std::int64_t> slot_buf;
    auto slot_of = [&](std::int32_t id, const Off& o) {
        const auto& a = res_m[static_cast<size_t>(id)];
        std::int64_t f = 0;
        for (int ax = dim - 1; ax >= 0; --ax) {
            std::int32_t v = a[static_cast<size_t>(ax)] + o.v[ax];
            if (v >= m) v -= m;  // residue < m and offset < m (all accepted offsets are < lim <= m)
            f = f * m + v;
        }
        return f;
    };
    auto fits = [&](std::int64_t b, std::int64_t e, const Off& o) {
        slot_buf.clear();
        for (std::int64_t k = b; k < e; ++k) {
            const std::int64_t sl = slot_of(members[static_cast<size_t>(k)], o);
            if (hash[static_cast<size_t>(sl)] != -1) return false;
            slot_buf.push_back(sl);
        }
        for (size_t i = 0; i < slot_buf.size(); ++i)
            for (size_t j = i + 1; j < slot_buf.size(); ++j)
                if (slot_buf[i] == slot_buf[j]) return false;
        return true;
    };

    for (const std::int64_t cell : order) {
        const std::int64_t b = start[static_cast<size_t>(cell)], e = start[static_cast<size_t>(cell + 1)];
        bool ok = false;
        Off pick;
        const int probes = static_cast<int>(std::min<size_t>(used.size(), kReuseProbes));
        for (int t = 0; t < probes && !ok; ++t) {
            const auto j = static_cast<size_t>(rng.uniform_int(t, static_cast<std::int64_t>(used.size()) - 1));
            std::swap(perm[static_cast<size_t>(t)], perm[j]);
            const Off& cand = used[static_cast<size_t>(perm[static_cast<size_t>(t)])];
            if (fits(b, e, cand)) {
                pick = cand;
                ok = true;
            }
        }
        if (!ok) {
            Off o;
            for (std::int32_t z = 0; z < (dim == 3 ? lim : 1) && !ok; ++z) {
                o.v[2] = static_cast<std::uint8_t>(z);
                for (std::int32_t y = 0; y < lim && !ok; ++y) {
                    o.v[1] = static_cast<std::uint8_t>(y);
                    for (std::int32_t x = 0; x < lim && !ok; ++x) {
                        o.v[0] = static_cast<std::uint8_t>(x);
                        if (fits(b, e, o)) {
                            pick = o;
                            ok = true;
                        }
                    }
                }
            }
        }
        if (!ok) return false;
        for (int a = 0; a < dim; ++a) offsets[static_cast<size_t>(cell * dim + a)] = pick.v[a];
        for (std::int64_t k = b; k < e; ++k) {
            const std::int32_t id = members[static_cast<size_t>(k)];
            const std::int64_t sl = slot_of(id, pick);
            hash[static_cast<size_t>(sl)] = id;
            for (int a = 0; a < dim; ++a)
                tags[static_cast<size_t>(sl * dim + a)] =
                    static_cast<std::uint16_t>(s.voxels[static_cast<size_t>(id)][static_cast<size_t>(a)]);
        }
        if (std::find(used.begin(), used.end(), pick) == used.end()) {
            used.push_back(pick);
            perm.push_back(static_cast<std::int32_t>(perm.size()));
        }
    }
    return true;
}

// psh.cpp:164-177
std::int32_t min_hash_dim(std::int64_t n, int dim) {
    auto m = static_cast<std::int32_t>(std::floor(std::pow(static_cast<double>(n), 1.0 / dim)));
    m = std::max(m - 2, 1);
    while (ipow(m, dim) <= n) ++m;
    return m;
}
std::int32_t first_offset_dim(std::int64_t n, int dim) {
    const double target = static_cast<double>(n) / (2.0 * dim);
    auto r = static_cast<std::int32_t>(std::floor(std::pow(target, 1.0 / dim)));
    r = std::max(r - 2, 1);
    while (ipow(r, dim) < static_cast<std::int64_t>(std::ceil(target))) ++r;
    return std::max(r, 1);
}

PshLevel build_level(const VoxelSet& s, std::uint64_t seed, const std::uint8_t* inj,
                     std::int64_t inj_len, std::int32_t inj_dim) {
    if (s.voxels.empty()) throw std::invalid_argument("empty input");
    if (s.resolution >= 65536)
        throw std::invalid_argument(
            "resolution 65536 conflicts with the redundant-slot tag; pass allow_tag_ambiguity");
    PshLevel L;
    L.dim = s.dim;
    L.resolution = s.resolution;
    L.n = s.count();
    L.hash_dim = min_hash_dim(L.n, s.dim);
    L.channels = s.channels;
    L.data = s.features;
    if (inj) {
        // psh.cpp:193-202 + fill_from_offsets (psh.cpp:140-160)
        L.offset_dim = inj_dim;
        if (inj_dim <= 0) throw std::invalid_argument("injected offsets need offset_dim");
        if (inj_len != ipow(inj_dim, s.dim) * s.dim)
            throw std::invalid_argument("injected offset table has the wrong size");
        L.offsets.assign(inj, inj + inj_len);
        const std::int32_t m = L.hash_dim;
        L.hash.assign(static_cast<size_t>(L.slots()), -1);
        L.tags.assign(static_cast<size_t>(L.slots() * s.dim), 0xFFFF);
        for (std::int64_t i = 0; i < L.n; ++i) {
            const Coord& p = s.voxels[static_cast<size_t>(i)];
            Coord h1{0, 0, 0}, sl{0, 0, 0};
            for (int a = 0; a < s.dim; ++a) h1[static_cast<size_t>(a)] = p[static_cast<size_t>(a)] % inj_dim;
            const std::int64_t cell = flat(h1, inj_dim, s.dim);
            for (int a = 0; a < s.dim; ++a)
                sl[static_cast<size_t>(a)] =
                    (p[static_cast<size_t>(a)] % m + L.offsets[static_cast<size_t>(cell * s.dim + a)]) % m;
            const std::int64_t slot = flat(sl, m, s.dim);
            if (L.hash[static_cast<size_t>(slot)] != -1)
                throw std::runtime_error("injected offset table is not perfect for this set");
            L.hash[static_cast<size_t>(slot)] = static_cast<std::int32_t>(i);
            for (int a = 0; a < s.dim; ++a)
                L.tags[static_cast<size_t>(slot * s.dim + a)] = static_cast<std::uint16_t>(p[static_cast<size_t>(a)]);
        }
        return L;
    }
    std::int32_t r = first_offset_dim(L.n, s.dim);
    for (int attempt = 0;; ++attempt) {
        if (r < s.resolution)
            while (std::gcd(L.hash_dim, r) != 1 && r < s.resolution) ++r;
        r = std::min(r, s.resolution);
        if (ipow(r, s.dim) * s.dim > (std::int64_t{1} << 31))
            throw std::runtime_error("hash construction diverged");
        if (greedy_attempt(s, L.hash_dim, r, splitmix(seed, static_cast<std::uint64_t>(attempt)), L.hash,
                           L.offsets, L.tags)) {
            L.offset_dim = r;
            return L;
        }
        if (r >= s.resolution) throw std::runtime_error("hash construction diverged");
        const auto grown = static_cast<std::int32_t>(std::ceil(static_cast<double>(r) * std::cbrt(2.0)));
        r = std::max(grown, r + 1);
    }
}

// voxel.cpp:76-110 make_sparse_set
VoxelSet make_set(int dim, std::int32_t res, std::vector<Coord> coords, std::int64_t channels,
                  const float* feats) {
    if (dim != 2 && dim != 3) throw std::invalid_argument("dim must be 2 or 3");
    check_resolution(res);
    if (coords.empty()) throw std::invalid_argument("sparse voxel set must be non-empty");
    const std::int64_t n = static_cast<std::int64_t>(coords.size());
    std::vector<std::int64_t> idx(static_cast<size_t>(n));
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](std::int64_t a, std::int64_t b) {
        return zyx_less(coords[static_cast<size_t>(a)], coords[static_cast<size_t>(b)]);
    });
    VoxelSet s;
    s.dim = dim;
    s.resolution = res;
    s.channels = channels;
    s.features.assign(static_cast<size_t>(channels * n), 0.0f);
    s.voxels.reserve(static_cast<size_t>(n));
    for (std::int64_t k = 0; k < n; ++k) {
        const Coord& p = coords[static_cast<size_t>(idx[static_cast<size_t>(k)])];
        for (int a = 0; a < 3; ++a) {
            const bool ok = a < dim ? (p[static_cast<size_t>(a)] >= 0 && p[static_cast<size_t>(a)] < res)
                                    : p[static_cast<size_t>(a)] == 0;
            if (!ok) throw std::invalid_argument("voxel coordinate out of range");
        }
        if (!s.voxels.empty() && s.voxels.back() == p) throw std::invalid_argument("duplicate voxel coordinate");
        s.voxels.push_back(p);
        for (std::int64_t c = 0; c < channels; ++c)
            s.features[static_cast<size_t>(c * n + k)] = feats ? feats[c * n + idx[static_cast<size_t>(k)]] : 0.0f;
    }
    return s;
}

// bench.cpp:33-77 sphere_voxels (radius 0.4*res; shell band sqrt(3)/2)
VoxelSet sphere(std::int32_t res, bool shell) {
    const double center = res / 2.0, radius = 0.4 * res, band = std::sqrt(3.0) / 2.0;
    std::vector<Coord> pts;
    for (std::int32_t z = 0; z < res; ++z)
        for (std::int32_t y = 0; y < res; ++y)
            for (std::int32_t x = 0; x < res; ++x) {
                const Coord p{x, y, z};
                bool occ;
                if (shell) {
                    double d = 0;
                    for (int a = 0; a < 3; ++a) {
                        const double c = p[static_cast<size_t>(a)] + 0.5 - center;
                        d += c * c;
                    }
                    occ = std::abs(std::sqrt(d) - radius) <= band;
                } else {
                    double lo = 0, hi = 0;
                    for (int a = 0; a < 3; ++a) {
                        const double pa = p[static_cast<size_t>(a)];
                        const double dlo = std::max(std::max(pa - center, center - (pa + 1.0)), 0.0);
                        const double dhi = std::max(std::abs(pa - center), std::abs(pa + 1.0 - center));
                        lo += dlo * dlo;
                        hi += dhi * dhi;
                    }
                    occ = std::sqrt(lo) <= radius && radius <= std::sqrt(hi);
                }
                if (occ) pts.push_back(p);
            }
    const std::int64_t n = static_cast<std::int64_t>(pts.size());
    std::vector<float> f(static_cast<size_t>(3 * n));
    for (std::int64_t i = 0; i < n; ++i) {
        const Coord& p = pts[static_cast<size_t>(i)];
        float v[3];
        for (int a = 0; a < 3; ++a) v[a] = static_cast<float>(p[static_cast<size_t>(a)] + 0.5 - center);
        // types.hpp:28-39: dot (a.x*b.x + a.y*b.y + a.z*b.z), sqrt, scale by 1/n
        const float dd = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
        const float nn = std::sqrt(dd);
        if (nn > 0.0f) {
            const float inv = 1.0f / nn;
            for (int a = 0; a < 3; ++a) v[a] = v[a] * inv;
        } else {
            v[0] = v[1] = v[2] = 0.0f;
        }
        for (int a = 0; a < 3; ++a) f[static_cast<size_t>(a * n + i)] = v[a];
    }
    return make_set(3, res, std::move(pts), 3, f.data());
}

// voxel.cpp:218-268 coarsen: parent occupied iff any child; renormalised mean feature.
VoxelSet coarsen_set(const VoxelSet& s) {
    if (s.resolution < 8) throw std::invalid_argument("coarsen requires resolution >= 8");
    const std::int32_t res = s.resolution / 2;
    const std::int64_t n = s.count();
    std::vector<std::pair<std::int64_t, std::int64_t>> par(static_cast<size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) {
        const Coord& p = s.voxels[static_cast<size_t>(i)];
        par[static_cast<size_t>(i)] = {flat(Coord{p[0] / 2, p[1] / 2, p[2] / 2}, res, s.dim), i};
    }
    std::stable_sort(par.begin(), par.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    VoxelSet out;
    out.dim = s.dim;
    out.resolution = res;
    out.channels = s.channels;
    std::vector<std::vector<double>> acc;
    for (size_t i = 0; i < par.size();) {
        size_t j = i;
        std::vector<double> sum(static_cast<size_t>(s.channels), 0.0);
        while (j < par.size() && par[j].first == par[i].first) {
            for (std::int64_t c = 0; c < s.channels; ++c)
                sum[static_cast<size_t>(c)] += s.features[static_cast<size_t>(c * n + par[j].second)];
            ++j;
        }
        double len = 0;
        for (const double v : sum) len += v * v;
        len = std::sqrt(len);
        if (len < 1e-8)
            std::fill(sum.begin(), sum.end(), 0.0);
        else
            for (double& v : sum) v /= len;
        out.voxels.push_back(unflat(par[i].first, res, s.dim));
        acc.push_back(std::move(sum));
        i = j;
    }
    const std::int64_t m = out.count();
    out.features.assign(static_cast<size_t>(s.channels * m), 0.0f);
    for (std::int64_t k = 0; k < m; ++k)
        for (std::int64_t c = 0; c < s.channels; ++c)
            out.features[static_cast<size_t>(c * m + k)] = static_cast<float>(acc[static_cast<size_t>(k)][static_cast<size_t>(c)]);
    return out;
}

// psh_io.hpp:11-17 container
constexpr char kMagic[4] = {'P', 'S', 'H', '1'};

void put32(std::ostream& o, std::uint32_t v) { o.write(reinterpret_cast<const char*>(&v), 4); }
std::uint32_t get32(std::istream& i) {
    std::uint32_t v = 0;
    if (!i.read(reinterpret_cast<char*>(&v), 4)) throw std::runtime_error("truncated .psh container");
    return v;
}
template <class T>
void get_array(std::istream& in, std::vector<T>& v, std::size_t count) {
    v.resize(count);
    if (!in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(count * sizeof(T))))
        throw std::runtime_error("truncated .psh container");
}

}  // namespace

// psh.cpp:170-185 sizing, shared with the device builder (psh_build.cu)
std::int32_t psh_hash_dim(std::int64_t n, int dim) { return min_hash_dim(n, dim); }
std::int32_t psh_first_offset_dim(std::int64_t n, int dim) { return first_offset_dim(n, dim); }
}  // namespace hcb

using namespace hcb;

extern "C" {

uint64_t hc_mix_seed(uint64_t seed, uint64_t item) { return splitmix(seed, item); }

hc_status hc_sphere_voxels(int32_t resolution, int shell, hc_voxel_set** out) {
    return guard([&] {
        check_resolution(resolution);
        auto* s = new hc_voxel_set;
        static_cast<VoxelSet&>(*s) = sphere(resolution, shell != 0);
        *out = s;
    });
}

hc_status hc_voxel_set_make(int32_t dim, int32_t resolution, int64_t n, const int32_t* coords,
                            int64_t channels, const float* features, hc_voxel_set** out) {
    return guard([&] {
        std::vector<Coord> c(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) c[static_cast<size_t>(i)] = {coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
        auto* s = new hc_voxel_set;
        static_cast<VoxelSet&>(*s) = make_set(dim, resolution, std::move(c), channels, features);
        *out = s;
    });
}

hc_status hc_coarsen(const hc_voxel_set* s, hc_voxel_set** out) {
    return guard([&] {
        auto* o = new hc_voxel_set;
        static_cast<VoxelSet&>(*o) = coarsen_set(*s);
        *out = o;
    });
}

hc_status hc_voxel_set_info(const hc_voxel_set* s, int64_t info[4]) {
    info[0] = s->dim;
    info[1] = s->resolution;
    info[2] = s->count();
    info[3] = s->channels;
    return HC_OK;
}

hc_status hc_voxel_set_copy(const hc_voxel_set* s, int32_t* coords, float* features) {
    for (size_t i = 0; i < s->voxels.size(); ++i)
        for (int a = 0; a < 3; ++a) coords[3 * i + static_cast<size_t>(a)] = s->voxels[i][static_cast<size_t>(a)];
    if (features && !s->features.empty()) std::memcpy(features, s->features.data(), s->features.size() * 4);
    return HC_OK;
}

void hc_voxel_set_free(hc_voxel_set* s) { delete s; }

hc_status hc_build_psh(const hc_voxel_set* s, uint64_t seed, const uint8_t* injected, int64_t injected_len,
                       int32_t injected_dim, hc_psh_level** out) {
    return guard([&] {
        auto* l = new hc_psh_level;
        static_cast<PshLevel&>(*l) = build_level(*s, seed, injected, injected_len, injected_dim);
        *out = l;
    });
}

hc_status hc_psh_level_info(const hc_psh_level* l, int64_t info[6]) {
    info[0] = l->dim;
    info[1] = l->resolution;
    info[2] = l->n;
    info[3] = l->hash_dim;
    info[4] = l->offset_dim;
    info[5] = l->channels;
    return HC_OK;
}

hc_status hc_psh_level_copy(const hc_psh_level* l, int32_t* hash, uint8_t* offsets, uint16_t* tags, float* data) {
    if (hash) std::memcpy(hash, l->hash.data(), l->hash.size() * 4);
    if (offsets) std::memcpy(offsets, l->offsets.data(), l->offsets.size());
    if (tags) std::memcpy(tags, l->tags.data(), l->tags.size() * 2);
    if (data && !l->data.empty()) std::memcpy(data, l->data.data(), l->data.size() * 4);
    return HC_OK;
}

void hc_psh_level_free(hc_psh_level* l) { delete l; }

hc_status hc_write_psh_file(const char* path, const hc_psh_level* const* levels, int32_t count) {
    return guard([&] {
        if (count <= 0) throw std::invalid_argument("no levels to write");
        std::ofstream o(path, std::ios::binary);
        if (!o) throw std::runtime_error(std::string("cannot open for writing: ") + path);
        o.write(kMagic, 4);
        put32(o, static_cast<std::uint32_t>(count));
        for (int32_t i = 0; i < count; ++i) {
            const PshLevel& l = *levels[i];
            for (std::uint32_t v : {1u, static_cast<std::uint32_t>(l.dim), static_cast<std::uint32_t>(l.resolution),
                                    static_cast<std::uint32_t>(l.n), static_cast<std::uint32_t>(l.hash_dim),
                                    static_cast<std::uint32_t>(l.offset_dim), static_cast<std::uint32_t>(l.channels)})
                put32(o, v);
            o.write(reinterpret_cast<const char*>(l.hash.data()), static_cast<std::streamsize>(l.hash.size() * 4));
            o.write(reinterpret_cast<const char*>(l.offsets.data()), static_cast<std::streamsize>(l.offsets.size()));
            o.write(reinterpret_cast<const char*>(l.tags.data()), static_cast<std::streamsize>(l.tags.size() * 2));
            o.write(reinterpret_cast<const char*>(l.data.data()), static_cast<std::streamsize>(l.data.size() * 4));
        }
        if (!o) throw std::runtime_error("failed writing .psh stream");
    });
}

hc_status hc_read_psh_file(const char* path, hc_psh_level** levels, int32_t max_levels, int32_t* count) {
    return guard([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("cannot open file: ") + path);
        char magic[4] = {};
        if (!in.read(magic, 4) || std::memcmp(magic, kMagic, 4) != 0)
            throw std::runtime_error("not a .psh container (bad magic)");
        const std::uint32_t n = get32(in);
        if (n == 0 || n > 32) throw std::runtime_error("unreasonable .psh level count");
        std::vector<hc_psh_level*> got;
        try {
            for (std::uint32_t k = 0; k < n; ++k) {
                auto* l = new hc_psh_level;
                got.push_back(l);
                if (get32(in) != 1) throw std::runtime_error("unsupported .psh version");
                l->dim = static_cast<int>(get32(in));
                l->resolution = static_cast<std::int32_t>(get32(in));
                l->n = get32(in);
                l->hash_dim = static_cast<std::int32_t>(get32(in));
                l->offset_dim = static_cast<std::int32_t>(get32(in));
                l->channels = get32(in);
                if (l->dim != 2 && l->dim != 3) throw std::runtime_error("corrupt .psh: bad dim");
                if (l->hash_dim <= 0 || l->offset_dim <= 0 || l->n <= 0)
                    throw std::runtime_error("corrupt .psh: bad table dims");
                get_array(in, l->hash, static_cast<size_t>(l->slots()));
                get_array(in, l->offsets, static_cast<size_t>(l->cells() * l->dim));
                get_array(in, l->tags, static_cast<size_t>(l->slots() * l->dim));
                get_array(in, l->data, static_cast<size_t>(l->channels * l->n));
            }
        } catch (...) {
            for (auto* l : got) delete l;
            throw;
        }
        if (static_cast<std::int32_t>(n) > max_levels) {
            for (auto* l : got) delete l;
            throw std::invalid_argument("too many levels for the output array");
        }
        for (std::uint32_t k = 0; k < n; ++k) levels[k] = got[k];
        *count = static_cast<std::int32_t>(n);
    });
}

}  // extern "C"
