"""Native fused hash-conv layer on tcgen05 tensor cores (include/hashconv_b200_native.h).

The B200-first form of conv_forward / conv_backward (cnn_ops.cpp:206-232):
features are voxel-major bf16 tensors [N][C]; the field map (K0) is computed once
per structure pair and reused by forward, input-gradient and weight-gradient; the
column matrix is never materialised. Weights and weight gradients use the
reference layout W[co][ci*F^3 + t] (cnn_ops.hpp:21-27).
"""
from __future__ import annotations

import ctypes as C
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .ops import ConvSpec, field_map, field_size
from .psh import SuperPsh


def _p(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_voxel_major(ref: torch.Tensor) -> torch.Tensor:
    """C x N fp32 (reference layout) -> N x C bf16."""
    ref = ref.contiguous().float()
    c, n = ref.shape
    out = torch.empty((n, c), dtype=torch.bfloat16, device=ref.device)
    check(lib.hc_native_to_voxel_major(_p(ref), c, n, _p(out), _s()))
    return out


def to_channel_major(nat: torch.Tensor) -> torch.Tensor:
    """N x C (fp32 or bf16) -> C x N fp32 (reference layout)."""
    nat = nat.contiguous()
    n, c = nat.shape
    out = torch.empty((c, n), dtype=torch.float32, device=nat.device)
    dt = _lib.HC_DTYPE_F32 if nat.dtype == torch.float32 else _lib.HC_DTYPE_BF16
    check(lib.hc_native_to_channel_major(_p(nat), dt, n, c, _p(out), _s()))
    return out


PACK_FORWARD, PACK_BACKWARD, PACK_TRANSPOSE = 0, 1, 2


def pack_weights(w_ref: torch.Tensor, c_out: int, c_in: int, taps: int, backward: bool = False,
                 mode: int = None) -> torch.Tensor:
    """W[co][ci*taps + t] -> the bf16 GEMM operand (hc_native_pack_weights): forward
    (mode 0), flipped transpose for the stride-1 input gradient (1, `backward=True`), or the
    plain transpose W^T for the deconvolution (2)."""
    mode = (PACK_BACKWARD if backward else PACK_FORWARD) if mode is None else mode
    w_ref = w_ref.contiguous().float()
    rows = c_in if mode else c_out
    kp = int(lib.hc_native_packed_k(c_out if mode else c_in, taps))
    wp = torch.empty((rows, kp), dtype=torch.bfloat16, device=w_ref.device)
    check(lib.hc_native_pack_weights(_p(w_ref), c_out, c_in, taps, mode, _p(wp), _s()))
    return wp


class FieldMap(NamedTuple):
    """K0 field map on the device: `data` int32 in one of three layouts (0 row-major
    [n][taps], 1 tap-major [taps][n], 2 tile-major [ceil(n/128)][taps][128])."""

    data: torch.Tensor
    n: int
    taps: int
    layout: int


ROW_MAJOR, TAP_MAJOR, TILED = 0, 1, 2


def as_field_map(fmap) -> FieldMap:
    if isinstance(fmap, FieldMap):
        return fmap
    return FieldMap(fmap, fmap.shape[0], fmap.shape[1], ROW_MAJOR)


def field_map_native(inp: SuperPsh, out: SuperPsh, spec: ConvSpec, layout: int = TILED) -> FieldMap:
    """K0 for the native conv (tile-major by default: one contiguous block per 128-voxel tile)."""
    spec = ConvSpec(*spec)
    taps = field_size(spec, inp.dim)
    n = out.total_columns()
    if layout == TILED:
        m = torch.empty(((n + 127) // 128, taps, 128), dtype=torch.int32, device="cuda")
        check(lib.hc_field_map_tiled(inp._h, out._h, spec.c(), _p(m), _s()))
        return FieldMap(m, n, taps, TILED)
    m = field_map(inp, out, spec, tap_major=layout == TAP_MAJOR)
    return FieldMap(m, n, taps, layout)


def gather_gemm(fmap, x: torch.Tensor, wp: torch.Tensor, c_out: int, out_dtype=torch.float32) -> torch.Tensor:
    """Y[n] = sum_t X[fmap(n,t)] . Wp_t  on tcgen05 (hc_native_gather_gemm)."""
    fm = as_field_map(fmap)
    y = torch.empty((fm.n, c_out), dtype=out_dtype, device=x.device)
    dt = _lib.HC_DTYPE_F32 if out_dtype == torch.float32 else _lib.HC_DTYPE_BF16
    check(lib.hc_native_gather_gemm(_p(fm.data), fm.layout, fm.n, fm.taps, _p(x), x.shape[1], _p(wp), c_out, _p(y),
                                    dt, _s()))
    return y


# ---------------------------------------------------------------- split precision (fp32 accurate)
def split(t: torch.Tensor, channel_major: bool = False) -> torch.Tensor:
    """fp32 features -> split rows [N][2C] bf16 = [hi | lo], hi = rn(v), lo = rn(v - hi)
    (hc_native_split). `t` is voxel-major [N][C], or channel-major C x N (the reference
    layout) with channel_major=True."""
    t = t.contiguous().float()
    c, n = (t.shape[0], t.shape[1]) if channel_major else (t.shape[1], t.shape[0])
    out = torch.empty((n, 2 * c), dtype=torch.bfloat16, device=t.device)
    check(lib.hc_native_split(_p(t), int(channel_major), c, n, _p(out), _s()))
    return out


def pack_weights_x2(w_ref: torch.Tensor, c_out: int, c_in: int, taps: int, mode: int = PACK_FORWARD) -> torch.Tensor:
    """W[co][ci*taps + t] -> the split-precision operand [2 rows][Kp2] (hi rows, lo rows)."""
    w_ref = w_ref.contiguous().float()
    rows = c_in if mode else c_out
    kp = int(lib.hc_native_packed_k_x2(c_out if mode else c_in, taps))
    wp = torch.empty((2 * rows, kp), dtype=torch.bfloat16, device=w_ref.device)
    check(lib.hc_native_pack_weights_x2(_p(w_ref), c_out, c_in, taps, mode, _p(wp), _s()))
    return wp


def pack_weights_x2_fb(w_ref: torch.Tensor, c_out: int, c_in: int, taps: int, c_in_bwd: int = None):
    """Forward and flipped (dX) split operands in one launch (hc_native_pack_weights_x2_fb); the dX
    operand zero-padded to c_in_bwd >= c_in rows."""
    w_ref = w_ref.contiguous().float()
    c_in_bwd = c_in if c_in_bwd is None else c_in_bwd
    wf = torch.empty((2 * c_out, int(lib.hc_native_packed_k_x2(c_in, taps))), dtype=torch.bfloat16,
                     device=w_ref.device)
    wb = torch.empty((2 * c_in_bwd, int(lib.hc_native_packed_k_x2(c_out, taps))), dtype=torch.bfloat16,
                     device=w_ref.device)
    check(lib.hc_native_pack_weights_x2_fb(_p(w_ref), c_out, c_in, taps, c_in_bwd, _p(wf), _p(wb), _s()))
    return wf, wb


def gather_gemm_x2(fmap, xs: torch.Tensor, wp2: torch.Tensor, c_out: int) -> torch.Tensor:
    """fp32 Y[n] = sum_t X[fmap(n,t)] . W_t from split operands (hc_native_gather_gemm_x2)."""
    fm = as_field_map(fmap)
    y = torch.empty((fm.n, c_out), dtype=torch.float32, device=xs.device)
    check(lib.hc_native_gather_gemm_x2(_p(fm.data), fm.layout, fm.n, fm.taps, _p(xs), xs.shape[1] // 2, _p(wp2),
                                       c_out, _p(y), _s()))
    return y


def conv_dw_x2(fmap, xs: torch.Tensor, dys: torch.Tensor, ws: "DwWorkspace" = None) -> torch.Tensor:
    """fp32 dW[co][ci*taps + t] from split rows of X and dY (hc_native_conv_dw_x2)."""
    fm = as_field_map(fmap)
    c_in, c_out = xs.shape[1] // 2, dys.shape[1] // 2
    nbytes = int(lib.hc_native_dw_workspace_x2(fm.n, fm.taps, c_in, c_out))
    w = (ws or _WS).get(nbytes, xs.device)
    dw = torch.empty((c_out, c_in * fm.taps), dtype=torch.float32, device=xs.device)
    check(lib.hc_native_conv_dw_x2(_p(fm.data), fm.layout, fm.n, fm.taps, _p(xs), c_in, _p(dys), c_out, _p(dw),
                                   _p(w), w.numel(), _s()))
    return dw


class DwWorkspace:
    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
        return self.buf


_WS = DwWorkspace()


def conv_dw(fmap, x: torch.Tensor, dy: torch.Tensor, ws: DwWorkspace = None) -> torch.Tensor:
    """dW[co][ci*taps + t] = sum_n dY[n,co] X[fmap(n,t),ci]  (reference layout, fp32)."""
    fm = as_field_map(fmap)
    c_in, c_out = x.shape[1], dy.shape[1]
    nbytes = int(lib.hc_native_dw_workspace(fm.n, fm.taps, c_in, c_out))
    w = (ws or _WS).get(nbytes, x.device)
    dw = torch.empty((c_out, c_in * fm.taps), dtype=torch.float32, device=x.device)
    check(lib.hc_native_conv_dw(_p(fm.data), fm.layout, fm.n, fm.taps, _p(x), c_in, _p(dy), c_out, _p(dw), _p(w),
                                w.numel(), _s()))
    return dw


class HashConv:
    """One hash-conv layer in the native layout.

    forward(x) -> y          : conv_forward (cnn_ops.cpp:206-215)
    backward(dy, x) -> dw, dx: conv_backward (cnn_ops.cpp:217-232). Stride 1 (same structure):
                               dx via the flipped transposed kernel on the same field map.
                               Strided (output = a coarser structure): dx is the gather-GEMM
                               over the TRANSPOSED field map (fine voxel, tap -> the coarse voxel
                               whose field holds it), the col2hash of cnn_ops.cpp:229-231 without
                               a column matrix.
    """

    def __init__(self, structure: SuperPsh, weights: torch.Tensor, spec: ConvSpec, out_dtype=torch.bfloat16,
                 precision: str = "bf16", output: Optional[SuperPsh] = None):
        """precision "bf16": bf16 operands (features voxel-major bf16), fp32 accumulation;
        "f32": fp32 features and weights carried as bf16 hi/lo planes (hc_native_*_x2),
        fp32 outputs within 1e-5 of the float64 reference — the reference's own precision.
        output: the output structure of a strided conv (e.g. the next-coarser level for
        stride 2; cnn_ops.cpp:20-33 check_pair); None = `structure` (stride 1)."""
        spec = ConvSpec(*spec)
        if precision not in ("bf16", "f32"):
            raise ValueError("HashConv: precision must be 'bf16' or 'f32'")
        if spec.stride != 1 and output is None:
            raise ValueError("HashConv: a strided conv needs its output structure (output=...)")
        self.precision = precision
        self.s, self.spec = structure, spec
        self.out = output if output is not None else structure
        self.strided = output is not None and (spec.stride != 1 or output is not structure)
        self.out_dtype = torch.float32 if precision == "f32" else out_dtype
        self.taps = field_size(spec, structure.dim)
        if self.taps > 27:
            raise ValueError("native conv: at most 27 field taps (3x3x3)")
        self.tmap = None
        # any channel counts (the reference takes e.g. 3 -> 2): the tensor-core tile set is
        # {16, 32, 64, 128, 256} channels, so both sides are zero-padded to it; padded weight
        # rows/columns are zero, so the padded outputs and gradients are exactly zero
        self.cin_p, self.cout_p = _tile_channels(spec.in_channels), _tile_channels(spec.out_channels)
        if precision == "f32" and max(self.cin_p, self.cout_p) > 128:
            raise ValueError("native conv (split precision): at most 128 channels")
        self.fmap = None
        self._xs = None  # split rows of the last forward input (f32)
        self.set_weights(weights)

    def set_weights(self, w: torch.Tensor):
        sp = self.spec
        if tuple(w.shape) != (sp.out_channels, sp.in_channels * self.taps):
            raise ValueError("conv_forward: weight shape mismatch")
        self.w = w
        wp = w
        if (self.cin_p, self.cout_p) != (sp.in_channels, sp.out_channels):
            wp = torch.zeros((self.cout_p, self.cin_p * self.taps), dtype=w.dtype, device=w.device)
            wp.view(self.cout_p, self.cin_p, self.taps)[:sp.out_channels, :sp.in_channels] = \
                w.view(sp.out_channels, sp.in_channels, self.taps)
        # dX operand: the flipped kernel on the same map (stride 1), or the unflipped transpose on
        # the transposed map (strided)
        back = PACK_TRANSPOSE if self.strided else PACK_BACKWARD
        if self.precision == "f32":
            if back == PACK_BACKWARD:  # both operands in one launch
                self.wf, self.wb = pack_weights_x2_fb(wp, self.cout_p, self.cin_p, self.taps)
            else:
                self.wf = pack_weights_x2(wp, self.cout_p, self.cin_p, self.taps, PACK_FORWARD)
                self.wb = pack_weights_x2(wp, self.cout_p, self.cin_p, self.taps, back)
        else:
            self.wf = pack_weights(wp, self.cout_p, self.cin_p, self.taps, False)
            self.wb = pack_weights(wp, self.cout_p, self.cin_p, self.taps, mode=back)

    def build_map(self) -> FieldMap:
        """K0 in the tile-major layout (coalesced build; one bulk copy per tile in the GEMM);
        strided: also its transpose (input voxel, tap -> output voxel) for the input gradient."""
        self.fmap = field_map_native(self.s, self.out, self.spec, TILED)
        if self.strided:
            rows = field_map(self.s, self.out, self.spec)  # same map, row-major [n_out][taps]
            n_in = self.s.total_columns()
            tm = torch.empty(((n_in + 127) // 128, self.taps, 128), dtype=torch.int32, device=rows.device)
            check(lib.hc_native_transpose_map(_p(rows), rows.shape[0], self.taps, n_in, _p(tm), _s()))
            self.tmap = FieldMap(tm, n_in, self.taps, TILED)
        return self.fmap

    @staticmethod
    def _pad(t: torch.Tensor, c: int) -> torch.Tensor:
        if t.shape[1] == c:
            return t
        out = torch.zeros((t.shape[0], c), dtype=t.dtype, device=t.device)
        out[:, :t.shape[1]] = t
        return out

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x: voxel-major [N][C_in] (bf16, or fp32 for precision "f32")."""
        if self.fmap is None:
            self.build_map()
        if self.precision == "f32":
            self._xs = split(self._pad(x, self.cin_p))
            y = gather_gemm_x2(self.fmap, self._xs, self.wf, self.cout_p)
        else:
            y = gather_gemm(self.fmap, self._pad(x, self.cin_p), self.wf, self.cout_p, self.out_dtype)
        return y if self.cout_p == self.spec.out_channels else y[:, :self.spec.out_channels].contiguous()

    def backward(self, dy: torch.Tensor, x: torch.Tensor, dx_dtype=None):
        """-> (dW fp32 [C_out][C_in*taps], dX [N][C_in]). f32: x is the forward input (its
        split rows from forward() are reused when x is that same tensor's data)."""
        sp = self.spec
        if self.precision == "f32":
            xs = self._xs if self._xs is not None and x is None else split(self._pad(x, self.cin_p))
            dys = split(self._pad(dy, self.cout_p))
            dw = conv_dw_x2(self.fmap, xs, dys)
            if (self.cin_p, self.cout_p) != (sp.in_channels, sp.out_channels):
                dw = dw.view(self.cout_p, self.cin_p, self.taps)[:sp.out_channels, :sp.in_channels].reshape(
                    sp.out_channels, sp.in_channels * self.taps)
            dx = gather_gemm_x2(self.tmap if self.strided else self.fmap, dys, self.wb, self.cin_p)
            if self.cin_p != sp.in_channels:
                dx = dx[:, :sp.in_channels].contiguous()
            return dw, dx
        dyp, xp = self._pad(dy, self.cout_p), self._pad(x, self.cin_p)
        dw = conv_dw(self.fmap, xp, dyp)
        if (self.cin_p, self.cout_p) != (sp.in_channels, sp.out_channels):
            dw = dw.view(self.cout_p, self.cin_p, self.taps)[:sp.out_channels, :sp.in_channels].reshape(
                sp.out_channels, sp.in_channels * self.taps)
        dx = gather_gemm(self.tmap if self.strided else self.fmap, dyp, self.wb, self.cin_p, dx_dtype or self.out_dtype)
        if self.cin_p != sp.in_channels:
            dx = dx[:, :sp.in_channels].contiguous()
        return dw, dx


def _tile_channels(c: int) -> int:
    for t in (16, 32, 64, 128, 256):
        if c <= t:
            return t
    raise ValueError("native conv: at most 256 channels")


class HashDeconv:
    """Native deconvolution onto the finer structure (cnn_ops.cpp:408-435): the transpose
    of the strided conv `spec` (fine -> coarse field). Forward Y_fine = col2hash(W^T D_coarse)
    is a gather-GEMM over the TRANSPOSED field map (fine voxel g, row t -> the coarse voxel
    whose field holds g at t) with the W^T operand; backward is the strided conv's own
    structure: dW by the split-K dW kernel on the field map, dD_coarse by the gather-GEMM
    with the forward operand. Nothing is materialised (no column matrix, no col2hash)."""

    def __init__(self, coarse: SuperPsh, fine: SuperPsh, weights: torch.Tensor, spec: ConvSpec,
                 out_dtype=torch.bfloat16, precision: str = "bf16"):
        """precision "f32": fp32 data carried as bf16 hi/lo planes through the split-precision
        kernels (fp32 outputs within 1e-5 of float64); "bf16": bf16 operands."""
        spec = ConvSpec(*spec)
        if precision not in ("bf16", "f32"):
            raise ValueError("HashDeconv: precision must be 'bf16' or 'f32'")
        self.f32 = precision == "f32"
        self.coarse, self.fine, self.spec = coarse, fine, spec
        self.out_dtype = torch.float32 if self.f32 else out_dtype
        self.taps = field_size(spec, fine.dim)
        if tuple(weights.shape) != (spec.out_channels, spec.in_channels * self.taps):
            raise ValueError("deconv_forward: weight shape mismatch")
        self.w = weights
        self.pmap = field_map_native(fine, coarse, spec, TILED)  # coarse voxel p, row t -> fine column
        rows = field_map(fine, coarse, spec)                     # same map, row-major
        nf = fine.total_columns()
        tm = torch.empty(((nf + 127) // 128, self.taps, 128), dtype=torch.int32, device=weights.device)
        check(lib.hc_native_transpose_map(_p(rows), rows.shape[0], self.taps, nf, _p(tm), _s()))
        self.tmap = FieldMap(tm, nf, self.taps, TILED)

    def forward(self, coarse_data: torch.Tensor) -> torch.Tensor:
        """[N_coarse][C_out] bf16 -> [N_fine][C_in]   (cnn_ops.cpp:408-419)"""
        sp = self.spec
        if self.f32:
            wt = pack_weights_x2(self.w, sp.out_channels, sp.in_channels, self.taps, PACK_TRANSPOSE)
            return gather_gemm_x2(self.tmap, split(coarse_data), wt, sp.in_channels)
        wt = pack_weights(self.w, sp.out_channels, sp.in_channels, self.taps, mode=PACK_TRANSPOSE)
        return gather_gemm(self.tmap, coarse_data, wt, sp.in_channels, self.out_dtype)

    def backward(self, fine_grad: torch.Tensor, coarse_data: torch.Tensor, d_dtype=None):
        """-> (dW [C_out][C_in*taps] fp32, dD_coarse [N_coarse][C_out])   (cnn_ops.cpp:421-435)"""
        sp = self.spec
        if self.f32:
            fs = split(fine_grad)
            dw = conv_dw_x2(self.pmap, fs, split(coarse_data))
            wf = pack_weights_x2(self.w, sp.out_channels, sp.in_channels, self.taps, PACK_FORWARD)
            return dw, gather_gemm_x2(self.pmap, fs, wf, sp.out_channels)
        dw = conv_dw(self.pmap, fine_grad, coarse_data)
        wf = pack_weights(self.w, sp.out_channels, sp.in_channels, self.taps, mode=PACK_FORWARD)
        dd = gather_gemm(self.pmap, fine_grad, wf, sp.out_channels, d_dtype or self.out_dtype)
        return dw, dd


def smoke_check(structure: SuperPsh, x: np.ndarray, w: np.ndarray, dy: np.ndarray, y64: np.ndarray,
                dw64: np.ndarray = None, dx64: np.ndarray = None) -> None:
    """Native forward on tensor cores vs the double oracle: the bf16-operand layer (bf16
    tolerance) and the split-precision fp32 layer (forward, dW, dX within 1e-5)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    c_in, c_out = x.shape[0], w.shape[0]
    spec = ConvSpec(3, 1, 0, c_in, c_out)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    layer = HashConv(structure, torch.from_numpy(w).to(dev), spec, torch.float32)
    xv = to_voxel_major(torch.from_numpy(x).to(dev))
    y = to_channel_major(layer.forward(xv)).cpu().numpy().astype(np.float64)
    err = rel(y, y64)
    # bf16 operands (2^-9 relative each) accumulated in fp32
    assert err < 2e-2, f"native conv forward rel err {err}"
    f32 = HashConv(structure, torch.from_numpy(w).to(dev), spec, precision="f32")
    xf = torch.from_numpy(x).to(dev).t().contiguous()
    y = f32.forward(xf).t().cpu().numpy().astype(np.float64)
    assert rel(y, y64) <= 1e-5, f"native fp32 (split) conv forward rel err {rel(y, y64)}"
    if dw64 is not None:
        dw, dx = f32.backward(torch.from_numpy(dy).to(dev).t().contiguous(), xf)
        assert rel(dw.cpu().numpy().astype(np.float64), dw64) <= 1e-5, "native fp32 (split) dW"
        assert rel(dx.t().cpu().numpy().astype(np.float64), dx64) <= 1e-5, "native fp32 (split) dX"
