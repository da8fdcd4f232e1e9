/* hc_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (H-CNN hash2col / col2hash /
 * conv contraction / hash pooling), used as the CPU checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg. The product never
 * links this. Parity of this restatement is pinned against the reference
 * library itself (oracle/_ref/libhcref.so, built from /root/reference) and the
 * golden fixtures in tests/golden/ — see tests/test_oracle.py.
 *
 * Layouts are the reference's: feature matrices are channels x columns,
 * row-major (feature_matrix.hpp:14-40); column matrices are (C*F^3) x N_out
 * with row c*F^3 + field_row (cnn_ops.hpp:32-37).
 */
#ifndef HC_ORACLE_H
#define HC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* psh_batch.hpp:15-38 (SuperPsh), as flat arrays. */
typedef struct {
    int32_t dim, resolution, batch, reserved;
    const int32_t* hash;          /* H*  [M]          */
    const uint8_t* offsets;       /* Phi* [R*dim]     */
    const uint16_t* tags;         /* T*  [M*dim]      */
    const int32_t* model_of_slot; /* V*  [M], 1-based */
    const int64_t* hash_acc;      /* M*  [batch+1]    */
    const int64_t* offset_acc;    /* R*  [batch+1]    */
    const int64_t* data_acc;      /* N*  [batch+1]    */
    const int32_t* hash_dims;     /* m_bar [batch]    */
    const int32_t* offset_dims;   /* r_bar [batch]    */
} hco_super;

/* cnn_ops.hpp:11-17 */
typedef struct {
    int32_t kernel, stride, pad, in_channels, out_channels;
} hco_spec;

int64_t hco_locate(const hco_super* s, int32_t model, int32_t x, int32_t y, int32_t z);
/* field map: for every output column, F^dim entries (row order) = input column or -1 */
int hco_field_map(const hco_super* in, const hco_super* out, hco_spec spec, int64_t* map);

int hco_hash2col_f32(const hco_super* in, const float* data, const hco_super* out, hco_spec spec, float* cols);
int hco_hash2col_f64(const hco_super* in, const double* data, const hco_super* out, hco_spec spec, double* cols);
int hco_col2hash_f32(const float* g, const hco_super* in, const hco_super* out, hco_spec spec, float* res);
int hco_col2hash_f64(const double* g, const hco_super* in, const hco_super* out, hco_spec spec, double* res);
int hco_max_pool_f32(const hco_super* in, const float* data, const hco_super* out, hco_spec spec, float* res, int32_t* sw);
int hco_max_pool_f64(const hco_super* in, const double* data, const hco_super* out, hco_spec spec, double* res, int32_t* sw);
int hco_avg_pool_f32(const hco_super* in, const float* data, const hco_super* out, hco_spec spec, float* res);
int hco_avg_pool_f64(const hco_super* in, const double* data, const hco_super* out, hco_spec spec, double* res);
int hco_max_unpool_f32(const float* coarse, const int32_t* sw, const hco_super* fine, const hco_super* cs, hco_spec spec, float* res);
int hco_max_unpool_f64(const double* coarse, const int32_t* sw, const hco_super* fine, const hco_super* cs, hco_spec spec, double* res);
int hco_avg_unpool_f32(const float* coarse, const hco_super* fine, const hco_super* cs, hco_spec spec, float* res);
int hco_avg_unpool_f64(const double* coarse, const hco_super* fine, const hco_super* cs, hco_spec spec, double* res);

/* gemm.hpp:15-33: c = a*b ; c = a^T*b ; c = a*b^T (row-major) */
void hco_matmul_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k, int64_t cb);
void hco_matmul_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k, int64_t cb);
void hco_matmul_trans_a_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k, int64_t cb);
void hco_matmul_trans_a_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k, int64_t cb);
void hco_matmul_trans_b_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k, int64_t rb);
void hco_matmul_trans_b_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k, int64_t rb);

#ifdef __cplusplus
}
#endif
#endif
