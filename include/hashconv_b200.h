/* hashconv_b200.h — C ABI of the B200-native H-CNN hot path (libhcb200.so).
 *
 * Drop-in boundary for the reference operator surface in
 * /root/reference/proj/include/hashconv/{cnn_ops,gemm,psh_batch,psh,psh_io,voxel,bench}.hpp.
 * Each entry point below names the reference function it replaces (file:line,
 * paths relative to proj/). Conventions:
 *
 *   - Plain pointers and sizes only; no C++ or torch types cross this ABI.
 *   - Every call returns an hc_status. HC_ERR_INVALID_ARGUMENT corresponds to the
 *     reference's std::invalid_argument and HC_ERR_RUNTIME to std::runtime_error;
 *     hc_last_error() returns the exact reference message text (thread-local).
 *   - Device entry points take DEVICE pointers in the reference's layouts
 *     (feature matrices: channels x columns, row-major — feature_matrix.hpp:14-40;
 *     column matrices: (C*F^3) x N_out, row c*F^3 + field_row — cnn_ops.hpp:32-37)
 *     and are stream-ordered on `stream` (a cudaStream_t; NULL = legacy default).
 *     Outputs are caller-allocated (the reference returns by value; sizes follow
 *     from hc_psh_info). Device-side-only validation (switch range, cnn_ops.cpp:326-332)
 *     synchronises the stream.
 *   - Results are deterministic for a fixed input on any grid: no floating-point
 *     atomics in the order-defined kernels.
 *   - HC_MATH_EXACT (default) reproduces the reference's fp32 results bit-for-bit
 *     (same accumulation order, separate mul/add rounding). HC_MATH_FAST routes the
 *     contraction to tcgen05 tensor cores as 3xTF32 (operands split hi + lo in shared
 *     memory; <= 1e-5 normwise vs double) when the matrices are TMA-eligible (inner
 *     dimensions % 4 == 0, 16-byte aligned), else to FFMA tiles (same bar).
 *     HC_MATH_TF32 is the single-pass tf32 product (~1e-3 normwise).
 */
#ifndef HASHCONV_B200_H
#define HASHCONV_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the ABI is exported from a -fvisibility=hidden build */
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* hc_stream; /* == cudaStream_t */

typedef enum {
    HC_OK = 0,
    HC_ERR_INVALID_ARGUMENT = 1, /* reference std::invalid_argument */
    HC_ERR_RUNTIME = 2,          /* reference std::runtime_error    */
    HC_ERR_CUDA = 3,             /* CUDA error (no reference counterpart) */
} hc_status;

typedef enum { HC_MATH_EXACT = 0, HC_MATH_FAST = 1, HC_MATH_TF32 = 2 } hc_math;
/* HC_DTYPE_SPLIT (outputs of some native layers only): fp32 values written as the split-precision
 * rows the x2 conv kernels consume — bf16 [N][2C], hi = rn(v), lo = rn(v - hi), hi and lo planes
 * interleaved per 64 channels (hc_native_split's layout). */
typedef enum { HC_DTYPE_F32 = 0, HC_DTYPE_BF16 = 1, HC_DTYPE_SPLIT = 2 } hc_dtype;

/* Thread-local text of the last error (exact reference message for 1/2). */
const char* hc_last_error(void);
const char* hc_version(void);
/* Total kernels this library has enqueued in the process (for launch accounting). */
int64_t hc_launch_count(void);
/* Reference-signature conv_forward / conv_backward calls (fp32, HC_MATH_FAST) served by the
 * fused split-precision tensor-core conv instead of hash2col + GEMMs (stride-1 layer over one
 * structure handle, <= 128 channels; HCB_FAST_FUSED=0 disables the route). */
int64_t hc_fused_route_count(void);
/* Deferred argument checks (max_unpool's switch range): HC_ERR_INVALID_ARGUMENT with the
 * reference's message if a check run since the last call failed, else HC_OK; clears the flag.
 * Call after synchronising the stream(s) that ran the checked operators. */
hc_status hc_deferred_status(void);
/* Math mode for the reference-layout contraction (thread-local; default EXACT). */
hc_status hc_set_math(hc_math mode);
hc_math hc_get_math(void);

/* Device-memory plumbing for hosts that do not link CUDA themselves (the header-only
 * C++ drop-in shim include/hashconv_b200.hpp uses only these). */
hc_status hc_malloc(void** ptr, size_t bytes);
hc_status hc_free(void* ptr);
hc_status hc_memcpy_h2d(void* dst, const void* src, size_t bytes, hc_stream stream);
hc_status hc_memcpy_d2h(void* dst, const void* src, size_t bytes, hc_stream stream);
hc_status hc_stream_synchronize(hc_stream stream);

/* cnn_ops.hpp:11-17 ConvSpec */
typedef struct {
    int32_t kernel, stride, pad, in_channels, out_channels;
} hc_conv_spec;

/* =========================================================== host-side input producers
 * Host C++ (not on the GPU hot path); these restate the reference producers so the
 * framework can make its own tables. They reproduce the reference tables byte-for-byte. */

typedef struct hc_voxel_set hc_voxel_set; /* voxel.hpp:16-25 SparseVoxelSet */
typedef struct hc_psh_level hc_psh_level; /* psh.hpp:21-35 PshLevel         */

/* bench.cpp:33-77 sphere_voxels */
hc_status hc_sphere_voxels(int32_t resolution, int shell, hc_voxel_set** out);
/* voxel.cpp:76-110 make_sparse_set (coords: n x 3 int32 (x,y,z); features: channels x n) */
hc_status hc_voxel_set_make(int32_t dim, int32_t resolution, int64_t n, const int32_t* coords,
                            int64_t channels, const float* features, hc_voxel_set** out);
/* voxel.cpp:218-268 coarsen */
hc_status hc_coarsen(const hc_voxel_set* s, hc_voxel_set** out);
/* info: dim, resolution, n, channels */
hc_status hc_voxel_set_info(const hc_voxel_set* s, int64_t info[4]);
hc_status hc_voxel_set_copy(const hc_voxel_set* s, int32_t* coords, float* features);
void hc_voxel_set_free(hc_voxel_set* s);

/* psh.cpp:179-227 build_psh (greedy; deterministic per (set, seed)). `injected` /
 * `injected_dim` mirror PshBuildOptions::injected_offsets (psh.hpp:55-58); pass NULL/0. */
hc_status hc_build_psh(const hc_voxel_set* s, uint64_t seed, const uint8_t* injected,
                       int64_t injected_len, int32_t injected_dim, hc_psh_level** out);
/* The same construction on the GPU: identical sizing, growth schedule
 * and lookup semantics (psh.cpp:170-227), offsets found by a parallel CAS-claimed search
 * instead of the sequential greedy scan -> a different but equally perfect table (every
 * lookup returns the reference's column). Returns a host PshLevel like hc_build_psh. */
hc_status hc_build_psh_device(const hc_voxel_set* s, uint64_t seed, hc_psh_level** out);
/* info: dim, resolution, n, hash_dim (m_bar), offset_dim (r_bar), channels */
hc_status hc_psh_level_info(const hc_psh_level* l, int64_t info[6]);
hc_status hc_psh_level_copy(const hc_psh_level* l, int32_t* hash, uint8_t* offsets, uint16_t* tags,
                            float* data);
void hc_psh_level_free(hc_psh_level* l);
/* psh_io.hpp:11-17 ".psh" container; psh_io.cpp:45-63 / 65-90 */
hc_status hc_write_psh_file(const char* path, const hc_psh_level* const* levels, int32_t count);
hc_status hc_read_psh_file(const char* path, hc_psh_level** levels, int32_t max_levels,
                           int32_t* count);
/* mix_seed (rng.hpp:53-58), exposed so callers derive per-level seeds like build_pyramid */
uint64_t hc_mix_seed(uint64_t seed, uint64_t item);

/* =========================================================== device super-PSH
 * psh_batch.hpp:15-38 SuperPsh as flat host arrays (lengths: M = hash_acc[batch],
 * R = offset_acc[batch]; hash/model_of_slot M, tags M*dim, offsets R*dim). */
typedef struct {
    int32_t dim, resolution, batch, reserved;
    const int32_t* hash;
    const uint8_t* offsets;
    const uint16_t* tags;
    const int32_t* model_of_slot; /* may be NULL: derived from hash_acc */
    const int64_t* hash_acc;
    const int64_t* offset_acc;
    const int64_t* data_acc;
    const int32_t* hash_dims;
    const int32_t* offset_dims;
} hc_super_psh_host;

typedef struct hc_psh hc_psh; /* opaque device-resident super-PSH */

/* Upload an already-concatenated super-PSH (replaces passing `const SuperPsh&`). */
hc_status hc_psh_upload(const hc_super_psh_host* host, hc_psh** out, hc_stream stream);
/* psh_batch.cpp:8-54 build_super, done on the device: concatenates the levels'
 * tables straight into device memory (no host-side SuperPsh). */
hc_status hc_psh_upload_levels(const hc_psh_level* const* levels, int32_t count, hc_psh** out,
                               hc_stream stream);
/* info: dim, resolution, batch, total_slots M, offset cells R, total_columns N */
hc_status hc_psh_info(const hc_psh* p, int64_t info[6]);
/* Copy the device super-PSH back (any pointer may be NULL). */
hc_status hc_psh_download(const hc_psh* p, int32_t* hash, uint8_t* offsets, uint16_t* tags,
                          int32_t* model_of_slot, int64_t* hash_acc, int64_t* offset_acc,
                          int64_t* data_acc, int32_t* hash_dims, int32_t* offset_dims);
/* psh_batch.cpp:80-102 split_super: the batch's models as host PshLevels (free each with
 * hc_psh_level_free); `data` (device, channels x N) optional, supplies the levels' data. */
hc_status hc_split_super(const hc_psh* p, const float* data, int64_t channels, hc_psh_level** out,
                         int32_t max_levels, int32_t* count);
/* Device pointers of the column table (cnn_ops.cpp:50-66 column_info): per data
 * column, int4 {x, y, z, model} (model 1-based). Valid until hc_psh_free. */
hc_status hc_psh_columns(const hc_psh* p, const void** xyzm);
hc_status hc_psh_free(hc_psh* p);

/* psh_batch.cpp:56-78 locate, batched: queries is n x 4 int32 {model, x, y, z};
 * result[i] = global data column or -1. Device pointers. */
hc_status hc_locate(const hc_psh* p, const int32_t* queries, int64_t n, int64_t* result,
                    hc_stream stream);

/* K0 — field ("kernel") map: map[col * F^dim + row] = global input column of field
 * row `row` of output column `col`, or -1 (cnn_ops.cpp:100-119 collect_field_hits for
 * every output voxel). This is the paper's pre-stored neighbour map. */
hc_status hc_field_map(const hc_psh* in, const hc_psh* out, hc_conv_spec spec, int32_t* map,
                       hc_stream stream);
/* Same map, tap-major: map[row * N_out + col] (coalesced stores; the native conv layout). */
hc_status hc_field_map_tap_major(const hc_psh* in, const hc_psh* out, hc_conv_spec spec,
                                 int32_t* map, hc_stream stream);
/* Same map, tile-major: 128-column tiles, map[((col/128)*F^dim + row)*128 + col%128], padded
 * to a multiple of 128 columns with -1 (one contiguous block per tile; the native conv's
 * preferred layout, fetched with one bulk copy per tile). */
hc_status hc_field_map_tiled(const hc_psh* in, const hc_psh* out, hc_conv_spec spec, int32_t* map,
                             hc_stream stream);

/* =========================================================== reference-layout operators
 * fp32, device pointers, shapes passed explicitly so shape errors carry the
 * reference's messages. */

/* cnn_ops.cpp:123-158 hash2col: cols is (C_in*F^dim) x N_out */
hc_status hc_hash2col_f32(const hc_psh* in, const float* data, int64_t data_rows,
                          int64_t data_cols, const hc_psh* out, hc_conv_spec spec, float* cols,
                          hc_stream stream);
/* cnn_ops.cpp:160-204 col2hash: result is C_in x N_in (ascending-output order) */
hc_status hc_col2hash_f32(const float* col_grads, int64_t rows, int64_t cols, const hc_psh* in,
                          const hc_psh* out, hc_conv_spec spec, float* result, hc_stream stream);
/* cnn_ops.cpp:206-215 conv_forward: result C_out x N_out; w is C_out x (C_in*F^dim) */
hc_status hc_conv_forward_f32(const hc_psh* in, const float* data, int64_t data_rows,
                              int64_t data_cols, const hc_psh* out, const float* w, int64_t w_rows,
                              int64_t w_cols, hc_conv_spec spec, float* result, hc_stream stream);
/* cnn_ops.cpp:217-232 conv_backward: dw same shape as w, dx C_in x N_in */
hc_status hc_conv_backward_f32(const float* output_grad, int64_t g_rows, int64_t g_cols,
                               const float* w, int64_t w_rows, int64_t w_cols,
                               const float* cached_cols, int64_t c_rows, int64_t c_cols,
                               const hc_psh* in, const hc_psh* out, hc_conv_spec spec, float* dw,
                               float* dx, hc_stream stream);
/* cnn_ops.cpp:234-284 max_pool: result and switches C x N_coarse */
hc_status hc_max_pool_f32(const hc_psh* in, const float* data, int64_t data_rows,
                          int64_t data_cols, const hc_psh* out, hc_conv_spec spec, float* result,
                          int32_t* switches, hc_stream stream);
/* cnn_ops.cpp:286-322 avg_pool */
hc_status hc_avg_pool_f32(const hc_psh* in, const float* data, int64_t data_rows,
                          int64_t data_cols, const hc_psh* out, hc_conv_spec spec, float* result,
                          hc_stream stream);
/* cnn_ops.cpp:336-372 max_unpool. The switch range check (cnn_ops.cpp:326-332) is stream-ordered
 * and never synchronises: an out-of-range switch is reported by hc_deferred_status() after the
 * caller synchronises the stream (the C++ shim and ops.py do, so they throw the reference's
 * std::invalid_argument / ValueError at the call as the reference does). */
hc_status hc_max_unpool_f32(const float* coarse_data, int64_t c_rows, int64_t c_cols,
                            const int32_t* switches, int64_t s_rows, int64_t s_cols,
                            const hc_psh* fine, const hc_psh* coarse, hc_conv_spec spec,
                            float* result, hc_stream stream);
/* cnn_ops.cpp:374-406 avg_unpool */
hc_status hc_avg_unpool_f32(const float* coarse_data, int64_t c_rows, int64_t c_cols,
                            const hc_psh* fine, const hc_psh* coarse, hc_conv_spec spec,
                            float* result, hc_stream stream);
/* cnn_ops.cpp:408-419 deconv_forward: result C_in x N_fine */
hc_status hc_deconv_forward_f32(const hc_psh* coarse, const float* coarse_data, int64_t d_rows,
                                int64_t d_cols, const hc_psh* fine, const float* w,
                                int64_t w_rows, int64_t w_cols, hc_conv_spec spec, float* result,
                                hc_stream stream);
/* cnn_ops.cpp:421-435 deconv_backward: dw same shape as w, dx C_out x N_coarse */
hc_status hc_deconv_backward_f32(const float* fine_grad, int64_t g_rows, int64_t g_cols,
                                 const float* w, int64_t w_rows, int64_t w_cols,
                                 const float* cached_coarse, int64_t c_rows, int64_t c_cols,
                                 const hc_psh* coarse, const hc_psh* fine, hc_conv_spec spec,
                                 float* dw, float* dx, hc_stream stream);

/* gemm.hpp:15-26 / gemm.cpp:30-69 (row-major; device pointers):
 *   matmul:          c[ra x cb] = a[ra x k] * b[k x cb]
 *   matmul_trans_a:  c[k  x cb] = a[ra x k]^T * b[ra x cb]
 *   matmul_trans_b:  c[ra x rb] = a[ra x k] * b[rb x k]^T
 * EXACT mode: the reference accumulation order, bit-identical. */
hc_status hc_matmul_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k,
                        int64_t cb, hc_stream stream);
hc_status hc_matmul_trans_a_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k,
                                int64_t cb, hc_stream stream);
hc_status hc_matmul_trans_b_f32(const float* a, const float* b, float* c, int64_t ra, int64_t k,
                                int64_t rb, hc_stream stream);


/* fp64: the reference's double instantiation (cnn_ops.cpp:652-653, gemm.cpp:117-118) —
 * the same operators with double data; always order-exact (bit-identical to the
 * reference's double results; the math mode applies to fp32 only). Generic kernels:
 * a parity / gradient-check path, not tuned for throughput. */
hc_status hc_hash2col_f64(const hc_psh* in, const double* data, int64_t data_rows,
                          int64_t data_cols, const hc_psh* out, hc_conv_spec spec, double* cols,
                          hc_stream stream);
hc_status hc_col2hash_f64(const double* col_grads, int64_t rows, int64_t cols, const hc_psh* in,
                          const hc_psh* out, hc_conv_spec spec, double* result, hc_stream stream);
hc_status hc_conv_forward_f64(const hc_psh* in, const double* data, int64_t data_rows,
                              int64_t data_cols, const hc_psh* out, const double* w, int64_t w_rows,
                              int64_t w_cols, hc_conv_spec spec, double* result, hc_stream stream);
hc_status hc_conv_backward_f64(const double* output_grad, int64_t g_rows, int64_t g_cols,
                               const double* w, int64_t w_rows, int64_t w_cols,
                               const double* cached_cols, int64_t c_rows, int64_t c_cols,
                               const hc_psh* in, const hc_psh* out, hc_conv_spec spec, double* dw,
                               double* dx, hc_stream stream);
hc_status hc_max_pool_f64(const hc_psh* in, const double* data, int64_t data_rows,
                          int64_t data_cols, const hc_psh* out, hc_conv_spec spec, double* result,
                          int32_t* switches, hc_stream stream);
hc_status hc_avg_pool_f64(const hc_psh* in, const double* data, int64_t data_rows,
                          int64_t data_cols, const hc_psh* out, hc_conv_spec spec, double* result,
                          hc_stream stream);
hc_status hc_max_unpool_f64(const double* coarse_data, int64_t c_rows, int64_t c_cols,
                            const int32_t* switches, int64_t s_rows, int64_t s_cols,
                            const hc_psh* fine, const hc_psh* coarse, hc_conv_spec spec,
                            double* result, hc_stream stream);
hc_status hc_avg_unpool_f64(const double* coarse_data, int64_t c_rows, int64_t c_cols,
                            const hc_psh* fine, const hc_psh* coarse, hc_conv_spec spec,
                            double* result, hc_stream stream);
hc_status hc_deconv_forward_f64(const hc_psh* coarse, const double* coarse_data, int64_t d_rows,
                                int64_t d_cols, const hc_psh* fine, const double* w,
                                int64_t w_rows, int64_t w_cols, hc_conv_spec spec, double* result,
                                hc_stream stream);
hc_status hc_deconv_backward_f64(const double* fine_grad, int64_t g_rows, int64_t g_cols,
                                 const double* w, int64_t w_rows, int64_t w_cols,
                                 const double* cached_coarse, int64_t c_rows, int64_t c_cols,
                                 const hc_psh* coarse, const hc_psh* fine, hc_conv_spec spec,
                                 double* dw, double* dx, hc_stream stream);
hc_status hc_matmul_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k,
                        int64_t cb, hc_stream stream);
hc_status hc_matmul_trans_a_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k,
                                int64_t cb, hc_stream stream);
hc_status hc_matmul_trans_b_f64(const double* a, const double* b, double* c, int64_t ra, int64_t k,
                                int64_t rb, hc_stream stream);


/* The rest of cnn_ops.hpp (cnn_ops.hpp:118-170, cnn_ops.cpp:437-608), reference layout
 * (channel-major C x N), fp32 and fp64, same error messages:
 *   batch_norm_forward  per-channel stats over N (training: double two-pass mean / biased var,
 *                       running stats updated in T) or the running stats (inference);
 *                       y = (x - T(mean)) * T(1/sqrt(var + eps)); inv_std = the cache's
 *                       inv_std (optional), y doubles as the cache's `normalized`.
 *   batch_norm_backward dx = T(inv_std * (dy - s1/n - xhat * s2/n)), s1/s2 double sums.
 *   scale_forward/backward, relu_forward/backward (std::max(T(0), x)), and inverted dropout
 *   whose keep mask (uint8, one per element) is the reference's std::mt19937_64(seed) stream,
 *   bit-exact; training = 0 or ratio = 0: identity, mask all ones. */
hc_status hc_batch_norm_forward_f32(const float* x, int64_t c, int64_t n, float* running_mean,
                                      float* running_var, int64_t stats_channels, float eps, float momentum,
                                      int32_t training, float* y, float* inv_std, hc_stream stream);
hc_status hc_batch_norm_backward_f32(const float* dy, int64_t c, int64_t n, const float* normalized,
                                       int64_t n_rows, int64_t n_cols, const float* inv_std, float* dx,
                                       hc_stream stream);
hc_status hc_scale_forward_f32(const float* x, int64_t rows, int64_t cols, const float* gamma, int64_t n_gamma,
                                 const float* beta, int64_t n_beta, float* y, hc_stream stream);
hc_status hc_scale_backward_f32(const float* dy, const float* x, int64_t rows, int64_t cols, const float* gamma,
                                  float* d_gamma, float* d_beta, float* dx, hc_stream stream);
hc_status hc_relu_forward_f32(const float* x, int64_t total, float* y, hc_stream stream);
hc_status hc_relu_backward_f32(const float* dy, int64_t rows, int64_t cols, const float* forward_out,
                                 int64_t o_rows, int64_t o_cols, float* dx, hc_stream stream);
hc_status hc_dropout_forward_f32(const float* x, int64_t total, float ratio, uint64_t seed, int32_t training,
                                   float* y, uint8_t* keep, hc_stream stream);
hc_status hc_dropout_backward_f32(const float* dy, int64_t total, const uint8_t* keep, int64_t keep_size,
                                    float ratio, float* dx, hc_stream stream);
hc_status hc_batch_norm_forward_f64(const double* x, int64_t c, int64_t n, double* running_mean,
                                      double* running_var, int64_t stats_channels, double eps, double momentum,
                                      int32_t training, double* y, double* inv_std, hc_stream stream);
hc_status hc_batch_norm_backward_f64(const double* dy, int64_t c, int64_t n, const double* normalized,
                                       int64_t n_rows, int64_t n_cols, const double* inv_std, double* dx,
                                       hc_stream stream);
hc_status hc_scale_forward_f64(const double* x, int64_t rows, int64_t cols, const double* gamma, int64_t n_gamma,
                                 const double* beta, int64_t n_beta, double* y, hc_stream stream);
hc_status hc_scale_backward_f64(const double* dy, const double* x, int64_t rows, int64_t cols, const double* gamma,
                                  double* d_gamma, double* d_beta, double* dx, hc_stream stream);
hc_status hc_relu_forward_f64(const double* x, int64_t total, double* y, hc_stream stream);
hc_status hc_relu_backward_f64(const double* dy, int64_t rows, int64_t cols, const double* forward_out,
                                 int64_t o_rows, int64_t o_cols, double* dx, hc_stream stream);
hc_status hc_dropout_forward_f64(const double* x, int64_t total, double ratio, uint64_t seed, int32_t training,
                                   double* y, uint8_t* keep, hc_stream stream);
hc_status hc_dropout_backward_f64(const double* dy, int64_t total, const uint8_t* keep, int64_t keep_size,
                                    double ratio, double* dx, hc_stream stream);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* HASHCONV_B200_H */
