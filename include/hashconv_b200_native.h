/* hashconv_b200_native.h — native (voxel-major) fused hash-conv on tcgen05 tensor cores.
 *
 * The B200-first form of the reference's conv contraction (cnn_ops.cpp:206-232 =
 * hash2col + matmul / matmul_trans_b / matmul_trans_a + col2hash): an implicit GEMM
 * whose A operand is gathered through the field map (hc_field_map) straight into
 * shared memory, so the (C*F^3) x N column matrix never exists in HBM.
 *
 * Layouts: features are voxel-major bf16 [N][C] (C a multiple of 8); the field map
 * is int32 [N_out][taps] (fmap_layout 0, hc_field_map), [taps][N_out] (layout 1,
 * hc_field_map_tap_major) or tile-major (layout 2, hc_field_map_tiled), -1 = empty cell; weights are packed once per update from
 * the reference layout W[co][ci*taps + t] (cnn_ops.hpp:21-27) by
 * hc_native_pack_weights. Device pointers, stream-ordered, deterministic.
 */
#ifndef HASHCONV_B200_NATIVE_H
#define HASHCONV_B200_NATIVE_H

#include "hashconv_b200.h"

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Packed K extent (taps * channels rounded up to 64). */
int64_t hc_native_packed_k(int32_t channels, int32_t taps);

/* backward = 0: Wp[co][t*C_in + ci] = W[co][ci*taps + t]           (forward operand)
 * backward = 1: Wp[ci][t*C_out + co] = W[co][ci*taps + taps-1-t]    (stride-1 input-gradient
 *               operand: the transposed, tap-flipped kernel)
 * backward = 2: Wp[ci][t*C_out + co] = W[co][ci*taps + t]           (deconvolution operand W^T,
 *               cnn_ops.cpp:408-419, with the transposed field map below)
 * w_packed: bf16, rows x hc_native_packed_k(...) */
hc_status hc_native_pack_weights(const float* w_ref, int32_t c_out, int32_t c_in, int32_t taps,
                                 int32_t backward, void* w_packed, hc_stream stream);

/* Y[n][0:c_out] = sum_{t,ci} X[fmap[n][t]][ci] * Wp[co][t*c_in + ci]  (gather-GEMM, tcgen05).
 * Forward conv: (fmap of (in,out), X, forward pack). Stride-1 input gradient:
 * (fmap of the structure, dY, backward pack) gives dX. c_out in {16,32,64,128,256}. */
hc_status hc_native_gather_gemm(const int32_t* fmap, int32_t fmap_layout, int64_t n_out,
                                int32_t taps, const void* x, int32_t c_in, const void* w_packed, int32_t c_out, void* y,
                                hc_dtype y_dtype, hc_stream stream);

/* dW in the reference layout (C_out x C_in*taps, fp32):
 * dW[co][ci*taps + t] = sum_n dY[n][co] * X[fmap[n][t]][ci]  (cnn_ops.cpp:228 matmul_trans_b).
 * Split-K over voxels on tcgen05, partials reduced in a fixed order (deterministic). */
size_t hc_native_dw_workspace(int64_t n_out, int32_t taps, int32_t c_in, int32_t c_out);
hc_status hc_native_conv_dw(const int32_t* fmap, int32_t fmap_layout, int64_t n_out,
                            int32_t taps, const void* x,
                            int32_t c_in, const void* dy, int32_t c_out, float* dw_ref,
                            void* workspace, size_t ws_bytes, hc_stream stream);

/* ---- Split precision (fp32-accurate contraction on the bf16 tensor-core path) ----------
 * An fp32 operand v is carried as two bf16 planes hi = rn(v), lo = rn(v - hi)
 * (|v - hi - lo| <= 2^-17 |v|); features become split rows [N][2C] = [hi | lo], weights
 * [2 R][hc_native_packed_k_x2] (hi rows then lo rows). The contraction accumulates
 * hi.hi + hi.lo + lo.hi (+ lo.lo for dW) in fp32 on tcgen05 — the reference's fp32
 * conv_forward / conv_backward (cnn_ops.cpp:206-232) within 1e-5 relative (normwise) of the
 * float64 instantiation on unquantised fp32 inputs. c_in, c_out <= 128 (multiples of 8;
 * forward c_out in {16, 32, 64, 128}). */
int64_t hc_native_packed_k_x2(int32_t channels, int32_t taps);
/* src fp32 channel-major C x N (channel_major = 1, the reference layout) or voxel-major
 * N x C (0) -> out bf16 [N][2C]. c a multiple of 4. */
hc_status hc_native_split(const float* src, int32_t channel_major, int64_t c, int64_t n, void* out,
                          hc_stream stream);
/* Same modes as hc_native_pack_weights; w_packed: bf16 [2*rows][hc_native_packed_k_x2(...)]. */
hc_status hc_native_pack_weights_x2(const float* w_ref, int32_t c_out, int32_t c_in, int32_t taps,
                                    int32_t mode, void* w_packed, hc_stream stream);
/* Both split operands of one layer in one launch: forward (mode 0) into w_fwd and flipped dX
 * (mode 1) into w_bwd, the latter zero-padded to c_in_bwd >= c_in rows (a multiple of 8). */
hc_status hc_native_pack_weights_x2_fb(const float* w_ref, int32_t c_out, int32_t c_in, int32_t taps,
                                       int32_t c_in_bwd, void* w_fwd, void* w_bwd, hc_stream stream);
/* The forward with batch-norm statistics from the epilogue: besides y, per
 * 128-row tile of the output and output channel, tile_stats[(tile * c_out + co) * 2 + {0, 1}] =
 * {sum, sum of squares about the tile mean} of the fp32 values (rows >= n_out excluded);
 * hc_native_bn_relu_forward_tiles folds them (replaces cnn_ops.cpp:455-466's two passes). */
hc_status hc_native_gather_gemm_stats(const int32_t* fmap, int32_t fmap_layout, int64_t n_out,
                                      int32_t taps, const void* x, int32_t c_in, const void* w_packed,
                                      int32_t c_out, void* y, hc_dtype y_dtype, float* tile_stats,
                                      hc_stream stream);
hc_status hc_native_gather_gemm_x2_stats(const int32_t* fmap, int32_t fmap_layout, int64_t n_out,
                                         int32_t taps, const void* x_split, int32_t c_in,
                                         const void* w_packed_x2, int32_t c_out, float* y,
                                         float* tile_stats, hc_stream stream);
/* y fp32 [n_out][c_out] = gather-GEMM of the split rows (hc_native_gather_gemm semantics). */
hc_status hc_native_gather_gemm_x2(const int32_t* fmap, int32_t fmap_layout, int64_t n_out,
                                   int32_t taps, const void* x_split, int32_t c_in,
                                   const void* w_packed_x2, int32_t c_out, float* y, hc_stream stream);
/* dW (reference layout, fp32) from split rows of X and dY (hc_native_conv_dw semantics). The
 * workspace query returns 0 for an unsupported shape. */
size_t hc_native_dw_workspace_x2(int64_t n_out, int32_t taps, int32_t c_in, int32_t c_out);
hc_status hc_native_conv_dw_x2(const int32_t* fmap, int32_t fmap_layout, int64_t n_out, int32_t taps,
                               const void* x_split, int32_t c_in, const void* dy_split, int32_t c_out,
                               float* dw_ref, void* workspace, size_t ws_bytes, hc_stream stream);

/* ---- Native net layers (voxel-major [N][C], C a multiple of 8) ----------------------
 * The block operators of net.cpp:181-323 around the conv: max pool / unpool
 * (cnn_ops.cpp:234-284, 336-372), batch norm + ReLU (cnn_ops.cpp:437-489, 542-561) and
 * the final 2^3 dense pool (net.cpp:69-122). Switches are int8 field rows (-1 = empty).
 *
 * Pool map: hc_field_map(fine, coarse, {2,2,0,C,C}) -> [n_coarse][8] fine columns.
 * hc_native_pool_parents inverts it (F == S fields tile the fine level): parent[g] =
 * coarse column covering g or -1, prow[g] = g's field row in it. */
hc_status hc_native_pool_parents(const int32_t* pmap, int64_t n_coarse, int32_t fd, int64_t n_fine,
                                 int32_t* parent, int8_t* prow, hc_stream stream);
/* y[p][c] = max over present field rows (first seeds, strict '>'), 0 if empty; switches[p][c]
 * = winning row or -1 (cnn_ops.cpp:234-284). x, y: dtype (bf16 or f32), fd must be 8. */
hc_status hc_native_max_pool(const int32_t* pmap, int64_t n_coarse, int32_t fd, const void* x,
                             hc_dtype dtype, int32_t c, void* y, int8_t* switches, hc_stream stream);
/* dx[g][c] = dy[parent[g]][c] if switches[parent[g]][c] == prow[g], else 0 (cnn_ops.cpp:336-372). */
hc_status hc_native_max_unpool(const int32_t* parent, const int8_t* prow, int64_t n_fine, const void* dy,
                               hc_dtype dtype, int32_t c, const int8_t* switches, void* dx,
                               hc_stream stream);
/* hc_native_max_unpool accumulated into an fp32 [n_fine][c] buffer: acc += unpooled rows, in one
 * pass (acc.add_(hc_native_max_unpool(...)) without materialising the unpooled rows). Used where an
 * unpooled branch joins a skip branch (the segmentation decoder). */
hc_status hc_native_max_unpool_add(const int32_t* parent, const int8_t* prow, int64_t n_fine, const void* dy,
                                   hc_dtype dtype, int32_t c, const int8_t* switches, float* acc,
                                   hc_stream stream);
/* Adjoint of hc_native_max_unpool: out[p][c] = fine[pmap[p][switches[p][c]]][c] (0 for -1). */
hc_status hc_native_switch_gather(const int32_t* pmap, int64_t n_coarse, int32_t fd, const void* fine,
                                  hc_dtype dtype, int32_t c, const int8_t* switches, void* out,
                                  hc_stream stream);
/* Training-mode batch norm over the N rows + ReLU: batch mean / biased variance (double,
 * two-pass), running stats updated with `momentum`, inv_std = 1/sqrt(var + eps);
 * xhat (fp32, optional) = (x - mean) * inv_std, out_bf16 = max(0, xhat). */
size_t hc_native_bn_workspace(int64_t n, int32_t c);
hc_status hc_native_bn_relu_forward(const float* x, int64_t n, int32_t c, int32_t training,
                                    float momentum, float eps, float* running_mean, float* running_var,
                                    float* inv_std, float* xhat, void* out_bf16, void* workspace,
                                    size_t ws_bytes, hc_stream stream);
/* d_conv = inv_std * (g - sum(g)/n - xhat * sum(g*xhat)/n), g = d_relu * (xhat > 0), bf16 out. */
hc_status hc_native_bn_relu_backward(const void* d_relu, hc_dtype dtype, const float* xhat,
                                     const float* inv_std, int64_t n, int32_t c, void* d_conv_bf16,
                                     void* workspace, size_t ws_bytes, hc_stream stream);
/* Inference-mode batch norm + ReLU (net_forward with training = false, cnn_ops.cpp:470-475):
 * the running statistics normalise; out_bf16 = max(0, (x - mean) * T(1/sqrt(var + eps))). */
hc_status hc_native_bn_relu_inference(const float* x, int64_t n, int32_t c, const float* running_mean,
                                      const float* running_var, float eps, void* out_bf16,
                                      hc_stream stream);
/* The same three with the output dtype explicit (HC_DTYPE_BF16 or HC_DTYPE_F32): the
 * split-precision (fp32) native net keeps fp32 activations and conv-output gradients. */
hc_status hc_native_bn_relu_forward_dt(const float* x, int64_t n, int32_t c, int32_t training,
                                       float momentum, float eps, float* running_mean, float* running_var,
                                       float* inv_std, float* xhat, void* out, hc_dtype out_dtype,
                                       void* workspace, size_t ws_bytes, hc_stream stream);
hc_status hc_native_bn_relu_backward_dt(const void* d_relu, hc_dtype dtype, const float* xhat,
                                        const float* inv_std, int64_t n, int32_t c, void* d_conv,
                                        hc_dtype out_dtype, void* workspace, size_t ws_bytes,
                                        hc_stream stream);
hc_status hc_native_bn_relu_inference_dt(const float* x, int64_t n, int32_t c, const float* running_mean,
                                         const float* running_var, float eps, void* out, hc_dtype out_dtype,
                                         hc_stream stream);
/* Synchronised batch norm for data parallelism (the reference normalises over
 * the whole batch, cnn_ops.cpp:456-470), in phases so the caller can sum the per-channel
 * statistics over ranks (e.g. ncclAllReduce, double) between them:
 *   forward:  bn_stat(0, x) -> sum -> bn_finalize(sum_x, NULL) [mean]
 *             bn_stat(1, x, mean) -> sum -> bn_finalize(sum_x, sum_sq) [running stats, inv_std]
 *             bn_relu_apply
 *   backward: bn_stat(2, xhat, d_relu) -> sum both rows -> bn_relu_backward_apply(n_total)
 * sums: double [2][c] (mode 0/1 use row 0). With one rank (n_total = n) the phases give the
 * fused calls' results bit for bit. */
hc_status hc_native_bn_stat(int32_t mode, const float* x, const void* d, hc_dtype dtype, int64_t n,
                            int32_t c, const double* mean, double* sums, void* workspace,
                            size_t ws_bytes, hc_stream stream);
hc_status hc_native_bn_finalize(const double* sum_x, const double* sum_sq, int64_t n_total, int32_t c,
                                float momentum, float eps, float* running_mean, float* running_var,
                                double* mean, float* inv_std, hc_stream stream);
hc_status hc_native_bn_relu_apply(const float* x, int64_t n, int32_t c, const double* mean,
                                  const float* inv_std, float* xhat, void* out_bf16, hc_stream stream);
hc_status hc_native_bn_relu_backward_apply(const void* d_relu, hc_dtype dtype, const float* xhat,
                                           const float* inv_std, int64_t n, int32_t c, const double* s1,
                                           const double* s2, int64_t n_total, void* d_conv_bf16,
                                           hc_stream stream);
hc_status hc_native_bn_relu_apply_dt(const float* x, int64_t n, int32_t c, const double* mean,
                                     const float* inv_std, float* xhat, void* out, hc_dtype out_dtype,
                                     hc_stream stream);
hc_status hc_native_bn_relu_backward_apply_dt(const void* d_relu, hc_dtype dtype, const float* xhat,
                                              const float* inv_std, int64_t n, int32_t c, const double* s1,
                                              const double* s2, int64_t n_total, void* d_conv,
                                              hc_dtype out_dtype, hc_stream stream);
/* Training batch norm + ReLU from the conv epilogue's tile statistics (hc_native_gather_gemm*
 * _stats on the same n x c output x): Chan's merge of the tiles in double (fixed order) ->
 * mean, biased variance, running stats, inv_std; then xhat / out as hc_native_bn_relu_forward_dt.
 * workspace: >= c doubles. Two launches instead of five. */
hc_status hc_native_bn_relu_forward_tiles(const float* tile_stats, int64_t n, int32_t c, float momentum,
                                          float eps, float* running_mean, float* running_var, float* inv_std,
                                          const float* x, float* xhat, void* out, hc_dtype out_dtype,
                                          void* workspace, size_t ws_bytes, hc_stream stream);
/* Final dense pool: cmap [b][8 cells][8 children] resolution-4 columns (or -1); head
 * [(c*8 + cell)][b] fp32 = max over present children, src = winning column or -1. */
hc_status hc_native_dense_pool(const int32_t* cmap, int32_t b, const void* x_bf16, int32_t c,
                               float* head, int32_t* src, hc_stream stream);
hc_status hc_native_dense_pool_dt(const int32_t* cmap, int32_t b, const void* x, hc_dtype dtype, int32_t c,
                                  float* head, int32_t* src, hc_stream stream);
hc_status hc_native_dense_pool_backward(const float* d_head, const int32_t* src, int32_t b, int32_t c,
                                        int64_t n_fine, float* dx, hc_stream stream);
/* Dropout (net.cpp:236-251) from uniform draws u[n]: mask = (u < keep) / keep, out = x * mask. */
hc_status hc_native_dropout_apply(const float* u, const float* x, int64_t n, float keep, float* mask, float* out,
                                  hc_stream stream);
/* Softmax cross-entropy (net.cpp:260-283): scores [classes][b] fp32, labels [b]; loss[0] (double)
 * = sum_j -log softmax(scores[:, j])[labels[j]] / denom, dscores = (softmax - onehot) / denom
 * (denom = the global batch under data parallelism). One launch, deterministic. */
hc_status hc_native_softmax_xent(const float* scores, int32_t classes, int32_t b, const int64_t* labels,
                                 int64_t denom, double* loss, float* dscores, hc_stream stream);
/* SGD with momentum and weight decay (net.cpp:339-346): v = momentum*v + lr*(g + wd*w); w -= v. */
/* The same update for `count` (<= 32) tensors in one launch (host arrays of device pointers / sizes). */
hc_status hc_native_sgd_update_multi(float* const* w, float* const* v, const float* const* g, const int64_t* n,
                                     int32_t count, float lr, float momentum, float weight_decay,
                                     hc_stream stream);
hc_status hc_native_sgd_update(float* w, float* v, const float* g, int64_t n, float lr, float momentum,
                               float weight_decay, hc_stream stream);

/* Transposed field map of a strided (coarsening) conv field: from pmap [n_coarse][taps]
 * (hc_field_map(fine, coarse, spec)) build the tile-major map tmap[g][t] = coarse voxel whose
 * field holds fine voxel g at row t (or -1). deconv_forward (cnn_ops.cpp:408-419) is then
 * hc_native_gather_gemm(tmap, D_coarse, pack mode 2, C_in); deconv_backward (:421-435) is
 * hc_native_conv_dw(pmap, fine_grad, D_coarse) for dW and hc_native_gather_gemm(pmap,
 * fine_grad, pack mode 0, C_out) for the coarse-data gradient. */
hc_status hc_native_transpose_map(const int32_t* pmap, int64_t n_coarse, int32_t taps, int64_t n_fine,
                                  int32_t* tmap_tiled, hc_stream stream);

/* Boundary transposes between the reference layout (C x N fp32) and the native layout. */
hc_status hc_native_to_voxel_major(const float* ref, int64_t c, int64_t n, void* out_bf16,
                                   hc_stream stream);
hc_status hc_native_to_channel_major(const void* native, hc_dtype dtype, int64_t n, int64_t c,
                                     float* out, hc_stream stream);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* HASHCONV_B200_NATIVE_H */
