/* hc_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference
 * hot path, used as the checker (see hc_oracle.h). Each function cites the
 * reference lines it restates (paths relative to /root/reference/proj).
 *
 * Arithmetic contract: compiled with -ffp-contract=off and no -march, so each
 * fp multiply and add rounds on its own, matching the reference's default
 * non-FMA build. Reduction orders are the reference's:
 *   - col2hash / unpool sum covering outputs in ascending (z,y,x) order
 *     (src/cnn_ops.cpp:184-196, 357-367, 394-401);
 *   - matmul accumulates k ascending and skips zero a-entries
 *     (src/gemm.cpp:14-26, 37-52); matmul_trans_b is a plain dot (54-69).
 */
#include "hc_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ helpers */

/* types.hpp:57-61 — x fastest */
static int64_t flat3(const int32_t p[3], int64_t extent, int dim) {
    int64_t f = 0;
    for (int a = dim - 1; a >= 0; --a) f = f * extent + p[a];
    return f;
}

/* cnn_ops.cpp:15-18 */
static int64_t fdiv(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
static int64_t cdiv(int64_t a, int64_t b) { return fdiv(a + b - 1, b); }

static int64_t field_volume(hco_spec sp, int dim) {
    int64_t v = 1;
    for (int a = 0; a < dim; ++a) v *= sp.kernel;
    return v;
}

/* cnn_ops.cpp:20-33 check_pair (returns 0 when valid) */
static int pair_ok(const hco_super* in, const hco_super* out, hco_spec sp) {
    if (in->dim != out->dim || in->batch != out->batch) return 0;
    if (sp.kernel < 1 || sp.stride < 1 || sp.pad < 0) return 0;
    if (sp.stride == 1) return (sp.kernel % 2 == 1) && in->resolution == out->resolution;
    return in->resolution == out->resolution * sp.stride;
}

/* psh_batch.cpp:56-78 — Eq. 4 (offset cell), Eq. 5 (hash slot), tag check. */
int64_t hco_locate(const hco_super* s, int32_t model, int32_t x, int32_t y, int32_t z) {
    const int v = model - 1, dim = s->dim;
    const int32_t m = s->hash_dims[v], r = s->offset_dims[v];
    const int32_t p[3] = {x, y, z};
    int32_t h1[3] = {0, 0, 0}, slot[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) h1[a] = p[a] % r;
    const int64_t cell = s->offset_acc[v] + flat3(h1, r, dim);
    for (int a = 0; a < dim; ++a) slot[a] = (p[a] % m + (int32_t)s->offsets[cell * dim + a]) % m;
    const int64_t sl = s->hash_acc[v] + flat3(slot, m, dim);
    const int32_t idx = s->hash[sl];
    if (idx < 0) return -1;
    for (int a = 0; a < dim; ++a)
        if (s->tags[sl * dim + a] != (uint16_t)p[a]) return -1;
    return s->data_acc[v] + idx;
}

/* cnn_ops.cpp:50-66 column_info: coordinate + model ordinal per data column */
typedef struct {
    int32_t* xyz;   /* 3 per column */
    int32_t* model; /* 1-based      */
} col_table;

static col_table columns_of(const hco_super* s) {
    const int64_t n = s->data_acc[s->batch], slots = s->hash_acc[s->batch];
    col_table t;
    t.xyz = (int32_t*)calloc((size_t)(3 * n + 3), sizeof(int32_t));
    t.model = (int32_t*)calloc((size_t)(n + 1), sizeof(int32_t));
    for (int64_t sl = 0; sl < slots; ++sl) {
        const int32_t idx = s->hash[sl];
        if (idx < 0) continue;
        const int32_t v = s->model_of_slot[sl];
        const int64_t g = s->data_acc[v - 1] + idx;
        for (int a = 0; a < s->dim; ++a) t.xyz[3 * g + a] = s->tags[sl * s->dim + a];
        t.model[g] = v;
    }
    return t;
}
static void drop(col_table t) {
    free(t.xyz);
    free(t.model);
}

/* cnn_ops.cpp:36-42 field_base */
static void field_origin(const int32_t po[3], hco_spec sp, int dim, int32_t base[3]) {
    base[0] = base[1] = base[2] = 0;
    for (int a = 0; a < dim; ++a)
        base[a] = sp.stride == 1 ? po[a] - (sp.kernel - 1) / 2 : po[a] * sp.stride - sp.pad;
}

/* cnn_ops.cpp:100-119 collect_field_hits: taps in (dz,dy,dx) order; the row
 * counter advances for every tap, out-of-domain taps are skipped before the
 * probe. Writes hit rows/columns, returns the hit count. */
static int field_hits(const hco_super* in, int32_t model, const int32_t base[3], hco_spec sp,
                      int64_t* rows, int64_t* cols) {
    const int dim = in->dim, F = sp.kernel, nz = dim == 3 ? F : 1;
    int n = 0;
    int64_t row = 0;
    for (int dz = 0; dz < nz; ++dz)
        for (int dy = 0; dy < F; ++dy)
            for (int dx = 0; dx < F; ++dx, ++row) {
                const int32_t q[3] = {base[0] + dx, base[1] + dy, dim == 3 ? base[2] + dz : 0};
                int inside = 1;
                for (int a = 0; a < dim; ++a) inside &= q[a] >= 0 && q[a] < in->resolution;
                if (!inside) continue;
                const int64_t g = hco_locate(in, model, q[0], q[1], q[2]);
                if (g >= 0) {
                    rows[n] = row;
                    cols[n] = g;
                    ++n;
                }
            }
    return n;
}

/* cnn_ops.cpp:70-85 covering_range */
static void cover_range(const int32_t pi[3], hco_spec sp, int dim, int32_t out_res, int32_t lo[3],
                        int32_t hi[3]) {
    for (int a = 0; a < 3; ++a) lo[a] = hi[a] = 0;
    for (int a = 0; a < dim; ++a) {
        int64_t l, h;
        if (sp.stride == 1) {
            l = pi[a] - (sp.kernel - 1) / 2;
            h = pi[a] + (sp.kernel - 1) / 2;
        } else {
            l = cdiv((int64_t)pi[a] + sp.pad - sp.kernel + 1, sp.stride);
            h = fdiv((int64_t)pi[a] + sp.pad, sp.stride);
        }
        lo[a] = (int32_t)(l > 0 ? l : 0);
        hi[a] = (int32_t)(h < out_res - 1 ? h : out_res - 1);
    }
}

/* cnn_ops.cpp:88-92 field_row */
static int64_t row_in_field(const int32_t pi[3], const int32_t base[3], int F, int dim) {
    int64_t r = 0;
    for (int a = dim - 1; a >= 0; --a) r = r * F + (pi[a] - base[a]);
    return r;
}

/* ------------------------------------------------------------------ field map */
int hco_field_map(const hco_super* in, const hco_super* out, hco_spec sp, int64_t* map) {
    if (!pair_ok(in, out, sp)) return -1;
    const int dim = in->dim;
    const int64_t fd = field_volume(sp, dim), n = out->data_acc[out->batch];
    col_table ct = columns_of(out);
    int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)fd);
    int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)fd);
    for (int64_t i = 0; i < n * fd; ++i) map[i] = -1;
    for (int64_t col = 0; col < n; ++col) {
        int32_t base[3];
        field_origin(ct.xyz + 3 * col, sp, dim, base);
        const int k = field_hits(in, ct.model[col], base, sp, rows, cols);
        for (int h = 0; h < k; ++h) map[col * fd + rows[h]] = cols[h];
    }
    free(rows);
    free(cols);
    drop(ct);
    return 0;
}

/* ------------------------------------------------------------------ ops (typed) */
#define HCO_TYPED(T, SUF)                                                                        \
    /* cnn_ops.cpp:123-158 hash2col (Alg. 1) */                                \
    int hco_hash2col_##SUF(const hco_super* in, const T* data, const hco_super* out, hco_spec sp, \
                           T* dst) {                                                             \
        if (!pair_ok(in, out, sp)) return -1;                                                    \
        const int dim = in->dim;                                                                 \
        const int64_t fd = field_volume(sp, dim), nin = in->data_acc[in->batch],                 \
                      nout = out->data_acc[out->batch];                                          \
        memset(dst, 0, sizeof(T) * (size_t)(sp.in_channels * fd * nout));                        \
        col_table ct = columns_of(out);                                                          \
        int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)fd);                          \
        int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)fd);                          \
        for (int64_t col = 0; col < nout; ++col) {                                               \
            int32_t base[3];                                                                     \
            field_origin(ct.xyz + 3 * col, sp, dim, base);                                       \
            const int k = field_hits(in, ct.model[col], base, sp, rows, cols);                   \
            for (int64_t c = 0; c < sp.in_channels; ++c)                                         \
                for (int h = 0; h < k; ++h)                                                      \
                    dst[(c * fd + rows[h]) * nout + col] = data[c * nin + cols[h]];              \
        }                                                                                        \
        free(rows);                                                                              \
        free(cols);                                                                              \
        drop(ct);                                                                                \
        return 0;                                                                                \
    }                                                                                            \
    /* cnn_ops.cpp:160-204 col2hash (Alg. 2): pull per input column, covering \
     * outputs in ascending (z,y,x) order */                                                     \
    int hco_col2hash_##SUF(const T* g, const hco_super* in, const hco_super* out, hco_spec sp,  \
                           T* res) {                                                             \
        if (!pair_ok(in, out, sp)) return -1;                                                    \
        const int dim = in->dim;                                                                 \
        const int64_t fd = field_volume(sp, dim), nin = in->data_acc[in->batch],                 \
                      nout = out->data_acc[out->batch];                                          \
        col_table ct = columns_of(in);                                                           \
        T* acc = (T*)malloc(sizeof(T) * (size_t)(sp.in_channels + 1));                           \
        for (int64_t gi = 0; gi < nin; ++gi) {                                                   \
            const int32_t* pi = ct.xyz + 3 * gi;                                                 \
            int32_t lo[3], hi[3], po[3] = {0, 0, 0}, base[3];                                    \
            for (int64_t c = 0; c < sp.in_channels; ++c) acc[c] = (T)0;                          \
            cover_range(pi, sp, dim, out->resolution, lo, hi);                                   \
            for (po[2] = lo[2]; po[2] <= hi[2]; ++po[2])                                         \
                for (po[1] = lo[1]; po[1] <= hi[1]; ++po[1])                                     \
                    for (po[0] = lo[0]; po[0] <= hi[0]; ++po[0]) {                               \
                        const int64_t col = hco_locate(out, ct.model[gi], po[0], po[1], po[2]);  \
                        if (col < 0) continue;                                                   \
                        field_origin(po, sp, dim, base);                                         \
                        const int64_t row = row_in_field(pi, base, sp.kernel, dim);              \
                        for (int64_t c = 0; c < sp.in_channels; ++c)                             \
                            acc[c] += g[(c * fd + row) * nout + col];                            \
                    }                                                                            \
            for (int64_t c = 0; c < sp.in_channels; ++c) res[c * nin + gi] = acc[c];             \
        }                                                                                        \
        free(acc);                                                                               \
        drop(ct);                                                                                \
        return 0;                                                                                \
    }                                                                                            \
    /* cnn_ops.cpp:234-284 max_pool: seed with the first present tap, strict '>' */             \
    int hco_max_pool_##SUF(const hco_super* in, const T* data, const hco_super* out, hco_spec sp, \
                           T* res, int32_t* sw) {                                                \
        if (!pair_ok(in, out, sp) || sp.stride < 2) return -1;                                   \
        const int dim = in->dim;                                                                 \
        const int64_t fd = field_volume(sp, dim), nin = in->data_acc[in->batch],                 \
                      nout = out->data_acc[out->batch];                                          \
        memset(res, 0, sizeof(T) * (size_t)(sp.in_channels * nout));                             \
        for (int64_t i = 0; i < sp.in_channels * nout; ++i) sw[i] = -1;                          \
        col_table ct = columns_of(out);                                                          \
        int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)fd);                          \
        int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)fd);                          \
        for (int64_t col = 0; col < nout; ++col) {                                               \
            int32_t base[3];                                                                     \
            field_origin(ct.xyz + 3 * col, sp, dim, base);                                       \
            const int k = field_hits(in, ct.model[col], base, sp, rows, cols);                   \
            if (k == 0) continue;                                                                \
            for (int64_t c = 0; c < sp.in_channels; ++c) {                                       \
                T best = data[c * nin + cols[0]];                                                \
                int64_t arg = rows[0];                                                           \
                for (int h = 1; h < k; ++h) {                                                    \
                    const T x = data[c * nin + cols[h]];                                         \
                    if (x > best) {                                                              \
                        best = x;                                                                \
                        arg = rows[h];                                                           \
                    }                                                                            \
                }                                                                                \
                res[c * nout + col] = best;                                                      \
                sw[c * nout + col] = (int32_t)arg;                                               \
            }                                                                                    \
        }                                                                                        \
        free(rows);                                                                              \
        free(cols);                                                                              \
        drop(ct);                                                                                \
        return 0;                                                                                \
    }                                                                                            \
    /* cnn_ops.cpp:286-322 avg_pool: (sum of present taps) * (1/F^dim) */                        \
    int hco_avg_pool_##SUF(const hco_super* in, const T* data, const hco_super* out, hco_spec sp, \
                           T* res) {                                                             \
        if (!pair_ok(in, out, sp) || sp.stride < 2) return -1;                                   \
        const int dim = in->dim;                                                                 \
        const int64_t fd = field_volume(sp, dim), nin = in->data_acc[in->batch],                 \
                      nout = out->data_acc[out->batch];                                          \
        const T inv = (T)1 / (T)fd;                                                              \
        col_table ct = columns_of(out);                                                          \
        int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)fd);                          \
        int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)fd);                          \
        for (int64_t col = 0; col < nout; ++col) {                                               \
            int32_t base[3];                                                                     \
            field_origin(ct.xyz + 3 * col, sp, dim, base);                                       \
            const int k = field_hits(in, ct.model[col], base, sp, rows, cols);                   \
            for (int64_t c = 0; c < sp.in_channels; ++c) {                                       \
                T s = (T)0;                                                                      \
                for (int h = 0; h < k; ++h) s += data[c * nin + cols[h]];                        \
                res[c * nout + col] = s * inv;                                                   \
            }                                                                                    \
        }                                                                                        \
        free(rows);                                                                              \
        free(cols);                                                                              \
        drop(ct);                                                                                \
        return 0;                                                                                \
    }                                                                                            \
    /* cnn_ops.cpp:336-372 max_unpool: out[c,g] += coarse iff switch == row(p_i) */              \
    int hco_max_unpool_##SUF(const T* coarse, const int32_t* sw, const hco_super* fine,          \
                             const hco_super* cs, hco_spec sp, T* res) {                         \
        if (!pair_ok(fine, cs, sp)) return -1;                                                   \
        const int dim = fine->dim;                                                               \
        const int64_t fd = field_volume(sp, dim), nf = fine->data_acc[fine->batch],              \
                      nc = cs->data_acc[cs->batch];                                              \
        for (int64_t i = 0; i < sp.in_channels * nc; ++i)                                        \
            if (sw[i] >= fd || sw[i] < -1) return -2; /* cnn_ops.cpp:326-332 */                  \
        memset(res, 0, sizeof(T) * (size_t)(sp.in_channels * nf));                               \
        col_table ct = columns_of(fine);                                                         \
        for (int64_t gi = 0; gi < nf; ++gi) {                                                    \
            const int32_t* pi = ct.xyz + 3 * gi;                                                 \
            int32_t lo[3], hi[3], po[3] = {0, 0, 0}, base[3];                                    \
            cover_range(pi, sp, dim, cs->resolution, lo, hi);                                    \
            for (po[2] = lo[2]; po[2] <= hi[2]; ++po[2])                                         \
                for (po[1] = lo[1]; po[1] <= hi[1]; ++po[1])                                     \
                    for (po[0] = lo[0]; po[0] <= hi[0]; ++po[0]) {                               \
                        const int64_t col = hco_locate(cs, ct.model[gi], po[0], po[1], po[2]);   \
                        if (col < 0) continue;                                                   \
                        field_origin(po, sp, dim, base);                                         \
                        const int32_t row = (int32_t)row_in_field(pi, base, sp.kernel, dim);     \
                        for (int64_t c = 0; c < sp.in_channels; ++c)                             \
                            if (sw[c * nc + col] == row) res[c * nf + gi] += coarse[c * nc + col]; \
                    }                                                                            \
        }                                                                                        \
        drop(ct);                                                                                \
        return 0;                                                                                \
    }                                                                                            \
    /* cnn_ops.cpp:374-406 avg_unpool: out[c,g] += coarse * (1/F^dim) (mul, then add) */         \
    int hco_avg_unpool_##SUF(const T* coarse, const hco_super* fine, const hco_super* cs,        \
                             hco_spec sp, T* res) {                                              \
        if (!pair_ok(fine, cs, sp)) return -1;                                                   \
        const int dim = fine->dim;                                                               \
        const int64_t fd = field_volume(sp, dim), nf = fine->data_acc[fine->batch],              \
                      nc = cs->data_acc[cs->batch];                                              \
        const T inv = (T)1 / (T)fd;                                                              \
        memset(res, 0, sizeof(T) * (size_t)(sp.in_channels * nf));                               \
        col_table ct = columns_of(fine);                                                         \
        for (int64_t gi = 0; gi < nf; ++gi) {                                                    \
            const int32_t* pi = ct.xyz + 3 * gi;                                                 \
            int32_t lo[3], hi[3], po[3] = {0, 0, 0};                                             \
            cover_range(pi, sp, dim, cs->resolution, lo, hi);                                    \
            for (po[2] = lo[2]; po[2] <= hi[2]; ++po[2])                                         \
                for (po[1] = lo[1]; po[1] <= hi[1]; ++po[1])                                     \
                    for (po[0] = lo[0]; po[0] <= hi[0]; ++po[0]) {                               \
                        const int64_t col = hco_locate(cs, ct.model[gi], po[0], po[1], po[2]);   \
                        if (col < 0) continue;                                                   \
                        for (int64_t c = 0; c < sp.in_channels; ++c) {                           \
                            const T scaled = coarse[c * nc + col] * inv;                         \
                            res[c * nf + gi] += scaled;                                          \
                        }                                                                        \
                    }                                                                            \
        }                                                                                        \
        drop(ct);                                                                                \
        return 0;                                                                                \
    }                                                                                            \
    /* gemm.cpp:14-35: row i of c accumulates a[i,k]*b[k,:], k ascending, zero a skipped */      \
    void hco_matmul_##SUF(const T* a, const T* b, T* c, int64_t ra, int64_t k, int64_t cb) {     \
        for (int64_t i = 0; i < ra; ++i) {                                                       \
            T* ci = c + i * cb;                                                                  \
            for (int64_t j = 0; j < cb; ++j) ci[j] = (T)0;                                       \
            for (int64_t kk = 0; kk < k; ++kk) {                                                 \
                const T av = a[i * k + kk];                                                      \
                if (av == (T)0) continue;                                                        \
                const T* bk = b + kk * cb;                                                       \
                for (int64_t j = 0; j < cb; ++j) {                                               \
                    const T prod = av * bk[j];                                                   \
                    ci[j] += prod;                                                               \
                }                                                                                \
            }                                                                                    \
        }                                                                                        \
    }                                                                                            \
    /* gemm.cpp:37-52: c[r,:] = sum_i a[i,r]*b[i,:], i ascending, zero a skipped */              \
    void hco_matmul_trans_a_##SUF(const T* a, const T* b, T* c, int64_t ra, int64_t k,           \
                                  int64_t cb) {                                                  \
        for (int64_t r = 0; r < k; ++r) {                                                        \
            T* cr = c + r * cb;                                                                  \
            for (int64_t j = 0; j < cb; ++j) cr[j] = (T)0;                                       \
            for (int64_t i = 0; i < ra; ++i) {                                                   \
                const T av = a[i * k + r];                                                       \
                if (av == (T)0) continue;                                                        \
                const T* bi = b + i * cb;                                                        \
                for (int64_t j = 0; j < cb; ++j) {                                               \
                    const T prod = av * bi[j];                                                   \
                    cr[j] += prod;                                                               \
                }                                                                                \
            }                                                                                    \
        }                                                                                        \
    }                                                                                            \
    /* gemm.cpp:54-69: c[i,j] = dot(a[i,:], b[j,:]) sequentially */                              \
    void hco_matmul_trans_b_##SUF(const T* a, const T* b, T* c, int64_t ra, int64_t k,           \
                                  int64_t rb) {                                                  \
        for (int64_t i = 0; i < ra; ++i)                                                         \
            for (int64_t j = 0; j < rb; ++j) {                                                   \
                T s = (T)0;                                                                      \
                for (int64_t kk = 0; kk < k; ++kk) {                                             \
                    const T prod = a[i * k + kk] * b[j * k + kk];                                \
                    s += prod;                                                                   \
                }                                                                                \
                c[i * rb + j] = s;                                                               \
            }                                                                                    \
    }

HCO_TYPED(float, f32)
HCO_TYPED(double, f64)
