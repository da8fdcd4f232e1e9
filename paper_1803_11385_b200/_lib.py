"""ctypes binding of libhcb200.so (the C ABI declared in include/hashconv_b200.h).

The product has no CPU fallback: if the library is missing this module raises
ImportError, and every device entry point fails loudly when no CUDA device is
present (HC_ERR_CUDA).
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HCB_LIB_PATH") or os.path.join(HERE, "_lib", "libhcb200.so")  # override: A/B builds
HEADERS = [os.path.join(os.path.dirname(HERE), "include", h)
           for h in ("hashconv_b200.h", "hashconv_b200_native.h")]

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the hash-conv path has no CPU fallback)")

lib = C.CDLL(LIB_PATH)

HC_OK, HC_ERR_INVALID_ARGUMENT, HC_ERR_RUNTIME, HC_ERR_CUDA = 0, 1, 2, 3
HC_MATH_EXACT, HC_MATH_FAST, HC_MATH_TF32 = 0, 1, 2
HC_DTYPE_F32, HC_DTYPE_BF16, HC_DTYPE_SPLIT = 0, 1, 2


class HashConvCudaError(RuntimeError):
    """A CUDA failure inside the library (no reference counterpart)."""


class ConvSpecC(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32),
                ("in_channels", C.c_int32), ("out_channels", C.c_int32)]


class SuperHostC(C.Structure):
    _fields_ = [("dim", C.c_int32), ("resolution", C.c_int32), ("batch", C.c_int32),
                ("reserved", C.c_int32),
                ("hash", C.c_void_p), ("offsets", C.c_void_p), ("tags", C.c_void_p),
                ("model_of_slot", C.c_void_p), ("hash_acc", C.c_void_p),
                ("offset_acc", C.c_void_p), ("data_acc", C.c_void_p),
                ("hash_dims", C.c_void_p), ("offset_dims", C.c_void_p)]


lib.hc_last_error.restype = C.c_char_p
lib.hc_version.restype = C.c_char_p
lib.hc_get_math.restype = C.c_int
lib.hc_mix_seed.restype = C.c_uint64
lib.hc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_SPEC = ConvSpecC

_SIGS = {
    "hc_set_math": [C.c_int],
    "hc_sphere_voxels": [_I32, C.c_int, _P],
    "hc_voxel_set_make": [_I32, _I32, _I64, _P, _I64, _P, _P],
    "hc_coarsen": [_P, _P],
    "hc_voxel_set_info": [_P, _P],
    "hc_voxel_set_copy": [_P, _P, _P],
    "hc_build_psh": [_P, C.c_uint64, _P, _I64, _I32, _P],
    "hc_build_psh_device": [_P, C.c_uint64, _P],
    "hc_psh_level_info": [_P, _P],
    "hc_psh_level_copy": [_P, _P, _P, _P, _P],
    "hc_write_psh_file": [C.c_char_p, _P, _I32],
    "hc_read_psh_file": [C.c_char_p, _P, _I32, _P],
    "hc_psh_upload": [_P, _P, _P],
    "hc_psh_upload_levels": [_P, _I32, _P, _P],
    "hc_malloc": [_P, C.c_size_t],
    "hc_free": [_P],
    "hc_psh_info": [_P, _P],
    "hc_split_super": [_P, _P, _I64, _P, _I32, _P],
    "hc_psh_download": [_P] * 10,
    "hc_psh_columns": [_P, _P],
    "hc_psh_free": [_P],
    "hc_locate": [_P, _P, _I64, _P, _P],
    "hc_field_map": [_P, _P, _SPEC, _P, _P],
    "hc_field_map_tap_major": [_P, _P, _SPEC, _P, _P],
    "hc_field_map_tiled": [_P, _P, _SPEC, _P, _P],
    "hc_hash2col_f32": [_P, _P, _I64, _I64, _P, _SPEC, _P, _P],
    "hc_col2hash_f32": [_P, _I64, _I64, _P, _P, _SPEC, _P, _P],
    "hc_conv_forward_f32": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _SPEC, _P, _P],
    "hc_conv_backward_f32": [_P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _SPEC, _P, _P, _P],
    "hc_max_pool_f32": [_P, _P, _I64, _I64, _P, _SPEC, _P, _P, _P],
    "hc_avg_pool_f32": [_P, _P, _I64, _I64, _P, _SPEC, _P, _P],
    "hc_max_unpool_f32": [_P, _I64, _I64, _P, _I64, _I64, _P, _P, _SPEC, _P, _P],
    "hc_avg_unpool_f32": [_P, _I64, _I64, _P, _P, _SPEC, _P, _P],
    "hc_deconv_forward_f32": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _SPEC, _P, _P],
    "hc_deconv_backward_f32": [_P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _SPEC, _P, _P, _P],
    "hc_matmul_f32": [_P, _P, _P, _I64, _I64, _I64, _P],
    "hc_matmul_trans_a_f32": [_P, _P, _P, _I64, _I64, _I64, _P],
    "hc_matmul_trans_b_f32": [_P, _P, _P, _I64, _I64, _I64, _P],
    "hc_hash2col_f64": [_P, _P, _I64, _I64, _P, _SPEC, _P, _P],
    "hc_col2hash_f64": [_P, _I64, _I64, _P, _P, _SPEC, _P, _P],
    "hc_conv_forward_f64": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _SPEC, _P, _P],
    "hc_conv_backward_f64": [_P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _SPEC, _P, _P, _P],
    "hc_max_pool_f64": [_P, _P, _I64, _I64, _P, _SPEC, _P, _P, _P],
    "hc_avg_pool_f64": [_P, _P, _I64, _I64, _P, _SPEC, _P, _P],
    "hc_max_unpool_f64": [_P, _I64, _I64, _P, _I64, _I64, _P, _P, _SPEC, _P, _P],
    "hc_avg_unpool_f64": [_P, _I64, _I64, _P, _P, _SPEC, _P, _P],
    "hc_deconv_forward_f64": [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _SPEC, _P, _P],
    "hc_deconv_backward_f64": [_P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _SPEC, _P, _P, _P],
    "hc_matmul_f64": [_P, _P, _P, _I64, _I64, _I64, _P],
    "hc_matmul_trans_a_f64": [_P, _P, _P, _I64, _I64, _I64, _P],
    "hc_matmul_trans_b_f64": [_P, _P, _P, _I64, _I64, _I64, _P],
}
_SIGS.update({
    "hc_native_pack_weights": [_P, _I32, _I32, _I32, _I32, _P, _P],
    "hc_native_gather_gemm": [_P, _I32, _I64, _I32, _P, _I32, _P, _I32, _P, C.c_int, _P],
    "hc_native_conv_dw": [_P, _I32, _I64, _I32, _P, _I32, _P, _I32, _P, _P, C.c_size_t, _P],
    "hc_native_to_voxel_major": [_P, _I64, _I64, _P, _P],
    "hc_native_to_channel_major": [_P, C.c_int, _I64, _I64, _P, _P],
    "hc_native_pool_parents": [_P, _I64, _I32, _I64, _P, _P, _P],
    "hc_native_transpose_map": [_P, _I64, _I32, _I64, _P, _P],
    "hc_native_max_pool": [_P, _I64, _I32, _P, C.c_int, _I32, _P, _P, _P],
    "hc_native_max_unpool": [_P, _P, _I64, _P, C.c_int, _I32, _P, _P, _P],
    "hc_native_max_unpool_add": [_P, _P, _I64, _P, C.c_int, _I32, _P, _P, _P],
    "hc_native_softmax_xent": [_P, _I32, _I32, _P, _I64, _P, _P, _P],
    "hc_native_dropout_apply": [_P, _P, _I64, C.c_float, _P, _P, _P],
    "hc_native_switch_gather": [_P, _I64, _I32, _P, C.c_int, _I32, _P, _P, _P],
    "hc_native_bn_relu_forward": [_P, _I64, _I32, _I32, C.c_float, C.c_float, _P, _P, _P, _P, _P, _P, C.c_size_t,
                                  _P],
    "hc_native_bn_relu_backward": [_P, C.c_int, _P, _P, _I64, _I32, _P, _P, C.c_size_t, _P],
    "hc_batch_norm_forward_f32": [_P, _I64, _I64, _P, _P, _I64, C.c_float, C.c_float, _I32, _P, _P, _P],
    "hc_batch_norm_backward_f32": [_P, _I64, _I64, _P, _I64, _I64, _P, _P, _P],
    "hc_scale_forward_f32": [_P, _I64, _I64, _P, _I64, _P, _I64, _P, _P],
    "hc_scale_backward_f32": [_P, _P, _I64, _I64, _P, _P, _P, _P, _P],
    "hc_relu_forward_f32": [_P, _I64, _P, _P],
    "hc_relu_backward_f32": [_P, _I64, _I64, _P, _I64, _I64, _P, _P],
    "hc_dropout_forward_f32": [_P, _I64, C.c_float, C.c_uint64, _I32, _P, _P, _P],
    "hc_dropout_backward_f32": [_P, _I64, _P, _I64, C.c_float, _P, _P],
    "hc_batch_norm_forward_f64": [_P, _I64, _I64, _P, _P, _I64, C.c_double, C.c_double, _I32, _P, _P, _P],
    "hc_batch_norm_backward_f64": [_P, _I64, _I64, _P, _I64, _I64, _P, _P, _P],
    "hc_scale_forward_f64": [_P, _I64, _I64, _P, _I64, _P, _I64, _P, _P],
    "hc_scale_backward_f64": [_P, _P, _I64, _I64, _P, _P, _P, _P, _P],
    "hc_relu_forward_f64": [_P, _I64, _P, _P],
    "hc_relu_backward_f64": [_P, _I64, _I64, _P, _I64, _I64, _P, _P],
    "hc_dropout_forward_f64": [_P, _I64, C.c_double, C.c_uint64, _I32, _P, _P, _P],
    "hc_dropout_backward_f64": [_P, _I64, _P, _I64, C.c_double, _P, _P],
    "hc_native_bn_relu_inference": [_P, _I64, _I32, _P, _P, C.c_float, _P, _P],
    "hc_native_bn_stat": [_I32, _P, _P, C.c_int, _I64, _I32, _P, _P, _P, C.c_size_t, _P],
    "hc_native_bn_finalize": [_P, _P, _I64, _I32, C.c_float, C.c_float, _P, _P, _P, _P, _P],
    "hc_native_bn_relu_apply": [_P, _I64, _I32, _P, _P, _P, _P, _P],
    "hc_native_bn_relu_backward_apply": [_P, C.c_int, _P, _P, _I64, _I32, _P, _P, _I64, _P, _P],
    "hc_native_dense_pool": [_P, _I32, _P, _I32, _P, _P, _P],
    "hc_native_dense_pool_dt": [_P, _I32, _P, C.c_int, _I32, _P, _P, _P],
    "hc_native_bn_relu_forward_tiles": [_P, _I64, _I32, C.c_float, C.c_float, _P, _P, _P, _P, _P, _P, C.c_int, _P,
                                        C.c_size_t, _P],
    "hc_native_gather_gemm_stats": [_P, _I32, _I64, _I32, _P, _I32, _P, _I32, _P, C.c_int, _P, _P],
    "hc_native_gather_gemm_x2_stats": [_P, _I32, _I64, _I32, _P, _I32, _P, _I32, _P, _P, _P],
    "hc_native_bn_relu_forward_dt": [_P, _I64, _I32, _I32, C.c_float, C.c_float, _P, _P, _P, _P, _P, C.c_int, _P,
                                     C.c_size_t, _P],
    "hc_native_bn_relu_backward_dt": [_P, C.c_int, _P, _P, _I64, _I32, _P, C.c_int, _P, C.c_size_t, _P],
    "hc_native_bn_relu_inference_dt": [_P, _I64, _I32, _P, _P, C.c_float, _P, C.c_int, _P],
    "hc_native_bn_relu_apply_dt": [_P, _I64, _I32, _P, _P, _P, _P, C.c_int, _P],
    "hc_native_bn_relu_backward_apply_dt": [_P, C.c_int, _P, _P, _I64, _I32, _P, _P, _I64, _P, C.c_int, _P],
    "hc_native_dense_pool_backward": [_P, _P, _I32, _I32, _I64, _P, _P],
    "hc_native_sgd_update": [_P, _P, _P, _I64, C.c_float, C.c_float, C.c_float, _P],
    "hc_native_sgd_update_multi": [_P, _P, _P, _P, _I32, C.c_float, C.c_float, C.c_float, _P],
    "hc_native_split": [_P, _I32, _I64, _I64, _P, _P],
    "hc_native_pack_weights_x2": [_P, _I32, _I32, _I32, _I32, _P, _P],
    "hc_native_pack_weights_x2_fb": [_P, _I32, _I32, _I32, _I32, _P, _P, _P],
    "hc_native_gather_gemm_x2": [_P, _I32, _I64, _I32, _P, _I32, _P, _I32, _P, _P],
    "hc_native_conv_dw_x2": [_P, _I32, _I64, _I32, _P, _I32, _P, _I32, _P, _P, C.c_size_t, _P],
})
lib.hc_native_bn_workspace.restype = C.c_size_t
lib.hc_native_bn_workspace.argtypes = [_I64, _I32]
lib.hc_native_packed_k.restype = C.c_int64
lib.hc_native_packed_k.argtypes = [_I32, _I32]
lib.hc_native_dw_workspace.restype = C.c_size_t
lib.hc_native_dw_workspace.argtypes = [_I64, _I32, _I32, _I32]
lib.hc_native_packed_k_x2.restype = C.c_int64
lib.hc_native_packed_k_x2.argtypes = [_I32, _I32]
lib.hc_native_dw_workspace_x2.restype = C.c_size_t
lib.hc_native_dw_workspace_x2.argtypes = [_I64, _I32, _I32, _I32]
lib.hc_launch_count.restype = C.c_int64
lib.hc_fused_route_count.restype = C.c_int64
lib.hc_deferred_status.restype = C.c_int
for _name, _args in _SIGS.items():
    fn = getattr(lib, _name)
    fn.argtypes = _args
    fn.restype = C.c_int
for _name in ("hc_voxel_set_free", "hc_psh_level_free"):
    getattr(lib, _name).argtypes = [_P]
    getattr(lib, _name).restype = None


def check(status: int) -> None:
    """Map hc_status to the reference's exception types (cnn_ops.cpp: std::invalid_argument
    -> ValueError, std::runtime_error -> RuntimeError)."""
    if status == HC_OK:
        return
    msg = lib.hc_last_error().decode()
    if status == HC_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == HC_ERR_CUDA:
        raise HashConvCudaError(msg)
    raise RuntimeError(msg)


def declared_symbols() -> list:
    """Every function name declared in include/*.h (for the ABI export test)."""
    names = []
    for h in HEADERS:
        if not os.path.exists(h):
            continue
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))
