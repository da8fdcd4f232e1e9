"""Reference operator surface (cnn_ops.hpp / gemm.hpp) on the B200 path.

Same names, argument meaning and error behaviour as `namespace hashconv`:
structures are device super-PSHs (psh.SuperPsh), feature matrices are
channels x columns fp32 tensors (feature_matrix.hpp:14-40), column matrices are
(C*F^3) x N_out (cnn_ops.hpp:32-37). Spec/shape errors raise ValueError with the
reference's std::invalid_argument message. Outputs are returned by value (new
tensors), like the reference.

Inputs may be CUDA tensors (device-resident path) or host numpy arrays / CPU
tensors (end-to-end path: uploaded, computed on the GPU, downloaded). There is
no CPU fallback: every call runs the sm_100a kernels of libhcb200.so.
"""
from __future__ import annotations

import contextlib
import ctypes as C
from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .psh import SuperPsh


class ConvSpec(NamedTuple):
    """cnn_ops.hpp:11-17"""

    kernel: int = 3
    stride: int = 1
    pad: int = 0
    in_channels: int = 0
    out_channels: int = 0

    def c(self) -> _lib.ConvSpecC:
        return _lib.ConvSpecC(int(self.kernel), int(self.stride), int(self.pad), int(self.in_channels),
                              int(self.out_channels))


def field_size(spec: ConvSpec, dim: int = 3) -> int:
    """cnn_ops.hpp:19 field_size"""
    return int(spec.kernel) ** dim


class ConvGradients(NamedTuple):
    """cnn_ops.hpp:48-52"""

    weights: torch.Tensor
    input: torch.Tensor


class MaxPoolResult(NamedTuple):
    """cnn_ops.hpp:75-79 (switches: int32 C x N_coarse)"""

    output: torch.Tensor
    switches: torch.Tensor


# ------------------------------------------------------------------ plumbing
def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.HashConvCudaError("no CUDA device: the hash-conv path runs on sm_100a only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class _Args:
    """Tracks whether the call came with host inputs (=> host outputs) and the call's
    precision: like the reference's templates (instantiated for float and double,
    cnn_ops.cpp:652-653), the first floating input picks T — float64 inputs run the fp64
    entry points, anything else fp32 — and the other floating inputs follow it."""

    def __init__(self):
        self.host = False
        self.dtype = None

    def fp(self, x) -> torch.Tensor:
        if isinstance(x, np.ndarray):
            self.host = True
            x = torch.from_numpy(np.ascontiguousarray(x, np.float64 if x.dtype == np.float64 else np.float32))
        if self.dtype is None:
            self.dtype = torch.float64 if x.dtype == torch.float64 else torch.float32
        if not x.is_cuda:
            self.host = True
            x = x.to(_dev(), non_blocking=True)
        if x.dtype != self.dtype:
            x = x.to(self.dtype)
        return x.contiguous()

    def fn(self, name: str):
        """The entry point of this call's precision: name_f32 or name_f64."""
        return getattr(lib, name + ("_f64" if self.dtype == torch.float64 else "_f32"))

    def i32(self, x) -> torch.Tensor:
        if isinstance(x, np.ndarray):
            self.host = True
            x = torch.from_numpy(np.ascontiguousarray(x, np.int32))
        if not x.is_cuda:
            self.host = True
            x = x.to(_dev(), non_blocking=True)
        return x.to(torch.int32).contiguous()

    def out(self, t: torch.Tensor):
        return t.cpu().numpy() if self.host else t


def _shape(t: torch.Tensor):
    if t.dim() != 2:
        raise ValueError("feature matrices are 2-D (rows x cols)")
    return int(t.shape[0]), int(t.shape[1])


def _p(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def _empty(rows, cols, dtype=torch.float32):
    return torch.empty((int(rows), int(cols)), dtype=dtype, device=_dev())


@contextlib.contextmanager
def math_mode(mode: str):
    """'exact' (bit-identical to src/gemm.cpp order), 'fast' (3xTF32 tensor cores, FFMA tiles
    for shapes TMA cannot stage; <= 1e-5 normwise) or 'tf32' (single-pass tf32, ~1e-3)."""
    modes = {"exact": _lib.HC_MATH_EXACT, "fast": _lib.HC_MATH_FAST, "tf32": _lib.HC_MATH_TF32}
    if mode not in modes:
        raise ValueError(f"unknown math mode {mode!r}")
    prev = lib.hc_get_math()
    check(lib.hc_set_math(modes[mode]))
    try:
        yield
    finally:
        lib.hc_set_math(prev)


# ------------------------------------------------------------------ operators
def field_map(input: SuperPsh, output: SuperPsh, spec: ConvSpec, tap_major: bool = False) -> torch.Tensor:
    """K0: int32 N_out x F^dim (or F^dim x N_out when tap_major), input column or -1
    (cnn_ops.cpp:100-119 collect_field_hits for every output voxel)."""
    spec = ConvSpec(*spec)
    fd = field_size(spec, input.dim)
    if tap_major:
        m = _empty(fd, output.total_columns(), torch.int32)
        check(lib.hc_field_map_tap_major(input._h, output._h, spec.c(), _p(m), _stream()))
    else:
        m = _empty(output.total_columns(), fd, torch.int32)
        check(lib.hc_field_map(input._h, output._h, spec.c(), _p(m), _stream()))
    return m


def locate(structure: SuperPsh, queries) -> torch.Tensor:
    """psh_batch.cpp:56-78 batched: queries n x 4 int32 {model, x, y, z} -> int64 column or -1."""
    a = _Args()
    q = a.i32(queries)
    r = torch.empty(q.shape[0], dtype=torch.int64, device=_dev())
    check(lib.hc_locate(structure._h, _p(q), q.shape[0], _p(r), _stream()))
    return a.out(r)


def hash2col(input: SuperPsh, input_data, output: SuperPsh, spec: ConvSpec):
    """cnn_ops.cpp:123-158"""
    spec = ConvSpec(*spec)
    a = _Args()
    d = a.fp(input_data)
    cols = _empty(spec.in_channels * field_size(spec, input.dim), output.total_columns(), a.dtype)
    check(a.fn("hc_hash2col")(input._h, _p(d), *_shape(d), output._h, spec.c(), _p(cols), _stream()))
    return a.out(cols)


def col2hash(col_grads, input: SuperPsh, output: SuperPsh, spec: ConvSpec):
    """cnn_ops.cpp:160-204"""
    spec = ConvSpec(*spec)
    a = _Args()
    g = a.fp(col_grads)
    res = _empty(spec.in_channels, input.total_columns(), a.dtype)
    check(a.fn("hc_col2hash")(_p(g), *_shape(g), input._h, output._h, spec.c(), _p(res), _stream()))
    return a.out(res)


def conv_forward(input: SuperPsh, input_data, output: SuperPsh, weights, spec: ConvSpec):
    """cnn_ops.cpp:206-215 (weights: C_out x C_in*F^dim)"""
    spec = ConvSpec(*spec)
    a = _Args()
    d, w = a.fp(input_data), a.fp(weights)
    res = _empty(spec.out_channels, output.total_columns(), a.dtype)
    check(a.fn("hc_conv_forward")(input._h, _p(d), *_shape(d), output._h, _p(w), *_shape(w), spec.c(), _p(res),
                                  _stream()))
    return a.out(res)


def conv_backward(output_grad, weights, cached_cols, input: SuperPsh, output: SuperPsh, spec: ConvSpec):
    """cnn_ops.cpp:217-232 -> ConvGradients(weights=dW, input=dX)"""
    spec = ConvSpec(*spec)
    a = _Args()
    g, w, cc = a.fp(output_grad), a.fp(weights), a.fp(cached_cols)
    gr, gc = _shape(g)
    wr, wc = _shape(w)
    dw = _empty(gr, _shape(cc)[0], a.dtype)
    dx = _empty(spec.in_channels, input.total_columns(), a.dtype)
    check(a.fn("hc_conv_backward")(_p(g), gr, gc, _p(w), wr, wc, _p(cc), *_shape(cc), input._h, output._h,
                                   spec.c(), _p(dw), _p(dx), _stream()))
    return ConvGradients(a.out(dw), a.out(dx))


def max_pool(input: SuperPsh, input_data, output: SuperPsh, spec: ConvSpec) -> MaxPoolResult:
    """cnn_ops.cpp:234-284"""
    spec = ConvSpec(*spec)
    a = _Args()
    d = a.fp(input_data)
    res = _empty(spec.in_channels, output.total_columns(), a.dtype)
    sw = _empty(spec.in_channels, output.total_columns(), torch.int32)
    check(a.fn("hc_max_pool")(input._h, _p(d), *_shape(d), output._h, spec.c(), _p(res), _p(sw), _stream()))
    return MaxPoolResult(a.out(res), a.out(sw))


def avg_pool(input: SuperPsh, input_data, output: SuperPsh, spec: ConvSpec):
    """cnn_ops.cpp:286-322"""
    spec = ConvSpec(*spec)
    a = _Args()
    d = a.fp(input_data)
    res = _empty(spec.in_channels, output.total_columns(), a.dtype)
    check(a.fn("hc_avg_pool")(input._h, _p(d), *_shape(d), output._h, spec.c(), _p(res), _stream()))
    return a.out(res)


def max_unpool(coarse_data, switches, fine: SuperPsh, coarse: SuperPsh, spec: ConvSpec, check_now: bool = True):
    """cnn_ops.cpp:336-372. The switch range check (cnn_ops.cpp:326-332) runs on the stream
    without a host round trip; with check_now (the reference's semantics: raise at the call)
    the stream is synchronised and hc_deferred_status() raises ValueError for an out-of-range
    switch. check_now=False keeps the call asynchronous (graph capture, pipelines): call
    check_deferred() after a later synchronisation."""
    spec = ConvSpec(*spec)
    a = _Args()
    cd, sw = a.fp(coarse_data), a.i32(switches)
    res = _empty(spec.in_channels, fine.total_columns(), a.dtype)
    check(a.fn("hc_max_unpool")(_p(cd), *_shape(cd), _p(sw), *_shape(sw), fine._h, coarse._h, spec.c(), _p(res),
                                _stream()))
    if check_now:
        torch.cuda.current_stream().synchronize()
        check_deferred()
    return a.out(res)


def check_deferred() -> None:
    """Raise the first deferred argument error (ValueError, the reference's message) recorded
    by a stream-ordered check since the last call (hc_deferred_status)."""
    check(lib.hc_deferred_status())


def avg_unpool(coarse_data, fine: SuperPsh, coarse: SuperPsh, spec: ConvSpec):
    """cnn_ops.cpp:374-406"""
    spec = ConvSpec(*spec)
    a = _Args()
    cd = a.fp(coarse_data)
    res = _empty(spec.in_channels, fine.total_columns(), a.dtype)
    check(a.fn("hc_avg_unpool")(_p(cd), *_shape(cd), fine._h, coarse._h, spec.c(), _p(res), _stream()))
    return a.out(res)


def deconv_forward(coarse: SuperPsh, coarse_data, fine: SuperPsh, weights, spec: ConvSpec):
    """cnn_ops.cpp:408-419"""
    spec = ConvSpec(*spec)
    a = _Args()
    d, w = a.fp(coarse_data), a.fp(weights)
    res = _empty(spec.in_channels, fine.total_columns(), a.dtype)
    check(a.fn("hc_deconv_forward")(coarse._h, _p(d), *_shape(d), fine._h, _p(w), *_shape(w), spec.c(), _p(res),
                                    _stream()))
    return a.out(res)


def deconv_backward(fine_grad, weights, cached_coarse_data, coarse: SuperPsh, fine: SuperPsh, spec: ConvSpec):
    """cnn_ops.cpp:421-435 -> ConvGradients(weights=dW, input=dX(coarse))"""
    spec = ConvSpec(*spec)
    a = _Args()
    g, w, cd = a.fp(fine_grad), a.fp(weights), a.fp(cached_coarse_data)
    dw = _empty(_shape(cd)[0], spec.in_channels * field_size(spec, fine.dim), a.dtype)
    dx = _empty(_shape(w)[0], coarse.total_columns(), a.dtype)
    check(a.fn("hc_deconv_backward")(_p(g), *_shape(g), _p(w), *_shape(w), _p(cd), *_shape(cd), coarse._h, fine._h,
                                     spec.c(), _p(dw), _p(dx), _stream()))
    return ConvGradients(a.out(dw), a.out(dx))


def matmul(a_, b_):
    """gemm.cpp:71-77: c = a * b"""
    a = _Args()
    x, y = a.fp(a_), a.fp(b_)
    if x.shape[1] != y.shape[0]:
        raise ValueError("matmul: shape mismatch")
    c = _empty(x.shape[0], y.shape[1], a.dtype)
    check(a.fn("hc_matmul")(_p(x), _p(y), _p(c), x.shape[0], x.shape[1], y.shape[1], _stream()))
    return a.out(c)


def matmul_trans_a(a_, b_):
    """gemm.cpp:79-85: c = a^T * b"""
    a = _Args()
    x, y = a.fp(a_), a.fp(b_)
    if x.shape[0] != y.shape[0]:
        raise ValueError("matmul_trans_a: shape mismatch")
    c = _empty(x.shape[1], y.shape[1], a.dtype)
    check(a.fn("hc_matmul_trans_a")(_p(x), _p(y), _p(c), x.shape[0], x.shape[1], y.shape[1], _stream()))
    return a.out(c)


def matmul_trans_b(a_, b_):
    """gemm.cpp:87-93: c = a * b^T"""
    a = _Args()
    x, y = a.fp(a_), a.fp(b_)
    if x.shape[1] != y.shape[1]:
        raise ValueError("matmul_trans_b: shape mismatch")
    c = _empty(x.shape[0], y.shape[0], a.dtype)
    check(a.fn("hc_matmul_trans_b")(_p(x), _p(y), _p(c), x.shape[0], x.shape[1], y.shape[0], _stream()))
    return a.out(c)


# ------------------------------------------------------------------ cnn_ops.hpp:118-170
class BatchNormStats:
    """cnn_ops.hpp:118-127: per-channel running statistics (updated in place by training
    batch_norm_forward). running_mean / running_var: CUDA tensors or numpy arrays."""

    def __init__(self, channels: int = 0, eps: float = 1e-5, momentum: float = 0.1, dtype=np.float32):
        self.running_mean = np.zeros(channels, dtype)
        self.running_var = np.ones(channels, dtype)
        self.eps, self.momentum = eps, momentum


class BatchNormCache:
    """cnn_ops.hpp:129-133: normalized (C x N) and inv_std (C)."""

    def __init__(self):
        self.normalized = None
        self.inv_std = None


class ScaleGradients(NamedTuple):  # cnn_ops.hpp:143-148
    gamma: object
    beta: object
    input: object


class DropoutMask:  # cnn_ops.hpp:160-162 (keep: uint8 per element)
    def __init__(self):
        self.keep = None


def _vec(a: _Args, v, n_expected=None):
    """A per-channel parameter vector in the call's precision (device)."""
    t = torch.as_tensor(np.asarray(v)) if not isinstance(v, torch.Tensor) else v
    t = t.to(device=_dev(), dtype=a.dtype).contiguous()
    return t


def _scalar(a: _Args):
    return C.c_double if a.dtype == torch.float64 else C.c_float


def batch_norm_forward(x, stats: BatchNormStats, training: bool, cache: BatchNormCache = None):
    """cnn_ops.cpp:437-482 (channel-major C x N)."""
    a = _Args()
    xt = a.fp(x)
    c, n = _shape(xt)
    rm, rv = _vec(a, stats.running_mean), _vec(a, stats.running_var)
    y = _empty(c, n, a.dtype)
    inv = torch.empty(c, dtype=a.dtype, device=_dev())
    S = _scalar(a)
    check(a.fn("hc_batch_norm_forward")(_p(xt), c, n, _p(rm), _p(rv), rm.numel(), S(stats.eps), S(stats.momentum),
                                        int(bool(training)), _p(y), _p(inv), _stream()))
    if training:  # write the updated running statistics back where they live
        for dst, src in ((stats.running_mean, rm), (stats.running_var, rv)):
            if isinstance(dst, torch.Tensor):
                dst.copy_(src)
            else:
                dst[...] = src.cpu().numpy()
    if cache is not None:
        cache.normalized = a.out(y)
        cache.inv_std = a.out(inv)
    return a.out(y)


def batch_norm_backward(dy, cache: BatchNormCache):
    """cnn_ops.cpp:484-507."""
    a = _Args()
    d = a.fp(dy)
    xh, inv = a.fp(cache.normalized), _vec(a, cache.inv_std)
    c, n = _shape(d)
    dx = _empty(c, n, a.dtype)
    check(a.fn("hc_batch_norm_backward")(_p(d), c, n, _p(xh), *_shape(xh), _p(inv), _p(dx), _stream()))
    return a.out(dx)


def scale_forward(x, gamma, beta):
    """cnn_ops.cpp:509-522: y = gamma * x + beta per channel."""
    a = _Args()
    xt = a.fp(x)
    g, b = _vec(a, gamma), _vec(a, beta)
    r, c = _shape(xt)
    y = _empty(r, c, a.dtype)
    check(a.fn("hc_scale_forward")(_p(xt), r, c, _p(g), g.numel(), _p(b), b.numel(), _p(y), _stream()))
    return a.out(y)


def scale_backward(dy, x, gamma) -> ScaleGradients:
    """cnn_ops.cpp:525-546."""
    a = _Args()
    d, xt = a.fp(dy), a.fp(x)
    g = _vec(a, gamma)
    r, c = _shape(d)
    dg = torch.empty(r, dtype=a.dtype, device=_dev())
    db = torch.empty(r, dtype=a.dtype, device=_dev())
    dx = _empty(r, c, a.dtype)
    check(a.fn("hc_scale_backward")(_p(d), _p(xt), r, c, _p(g), _p(dg), _p(db), _p(dx), _stream()))
    return ScaleGradients(a.out(dg), a.out(db), a.out(dx))


def relu_forward(x):
    """cnn_ops.cpp:548-559: max(0, x)."""
    a = _Args()
    xt = a.fp(x)
    y = torch.empty_like(xt)
    check(a.fn("hc_relu_forward")(_p(xt), xt.numel(), _p(y), _stream()))
    return a.out(y)


def relu_backward(dy, forward_out):
    """cnn_ops.cpp:561-573: dy where forward_out > 0."""
    a = _Args()
    d, fo = a.fp(dy), a.fp(forward_out)
    dx = torch.empty_like(d)
    check(a.fn("hc_relu_backward")(_p(d), *_shape(d), _p(fo), *_shape(fo), _p(dx), _stream()))
    return a.out(dx)


def dropout_forward(x, ratio: float, seed: int, training: bool, mask: DropoutMask = None):
    """cnn_ops.cpp:575-596: inverted dropout; the mask is the reference's mt19937_64(seed)
    stream (bit-exact)."""
    a = _Args()
    xt = a.fp(x)
    y = torch.empty_like(xt)
    keep = torch.empty(xt.numel(), dtype=torch.uint8, device=_dev())
    check(a.fn("hc_dropout_forward")(_p(xt), xt.numel(), _scalar(a)(ratio), C.c_uint64(seed & (2 ** 64 - 1)),
                                     int(bool(training)), _p(y), _p(keep), _stream()))
    if mask is not None:
        mask.keep = a.out(keep)
    return a.out(y)


def dropout_backward(dy, mask: DropoutMask, ratio: float):
    """cnn_ops.cpp:598-608."""
    a = _Args()
    d = a.fp(dy)
    k = mask.keep
    k = (torch.from_numpy(np.ascontiguousarray(k, np.uint8)) if isinstance(k, np.ndarray) else k)
    k = k.to(_dev()).contiguous()
    dx = torch.empty_like(d)
    check(a.fn("hc_dropout_backward")(_p(d), d.numel(), _p(k), k.numel(), _scalar(a)(ratio), _p(dx), _stream()))
    return a.out(dx)
