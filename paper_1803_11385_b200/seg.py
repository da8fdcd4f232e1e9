"""Segmentation-style composition on the native path (BASELINE config 4).

A SegNet / DeconvNet-style encoder-decoder on two PSH levels (PAPER.md:381 DeconvNet:
unpooling with the encoder's switches followed by convolution, plus a learned stride-2
deconvolution), built only from the reference's operators in their native form:

    encoder   x -> conv1 (fine, Cin->C) -> BN -> ReLU -> max_pool (switches) ->
              conv2 (coarse, C->2C) -> BN -> ReLU = e2
    decoder   max_unpool(conv3(e2): coarse 2C->C, the encoder's switches)   (cnn_ops.cpp:336-372)
              + deconv(e2): coarse 2C -> fine C, spec {2,2,0}                (cnn_ops.cpp:408-419)
              -> BN -> ReLU -> conv4 (fine, C->K) = per-voxel scores
    loss      per-voxel softmax cross-entropy against labels, mean over voxels

forward + backward of every layer (the unpool's backward is the pool's gather through the
same switches, the deconvolution's backward is the strided conv) — the col2hash-heavy
backward of config 4 without ever materialising a column matrix. Maps are built once per
batch. Weights are plain SGD-updated fp32 in the reference layout W[co][ci*taps + t].
"""
from __future__ import annotations

import math

import torch

from . import _lib
from . import conv as nconv
from ._lib import check, lib
from .net import BF16, _p, _s
from .ops import ConvSpec, field_map
from .psh import SuperPsh


class NativeSegNet:
    def __init__(self, fine: SuperPsh, coarse: SuperPsh, c_in: int = 8, c: int = 32, classes: int = 16,
                 seed: int = 0, lr: float = 0.01, precision: str = "bf16"):
        """precision "bf16": bf16 activations and conv operands; "f32": fp32 activations and
        gradients, every conv / deconv through the split-precision tcgen05 kernels (the
        reference's precision, within 1e-5 of float64 per operator)."""
        if c_in % 8 or c % 16 or classes % 16:
            raise ValueError("native seg net: c_in % 8, c % 16, classes % 16 (tensor-core tile set)")
        if precision not in ("bf16", "f32"):
            raise ValueError("precision must be 'bf16' or 'f32'")
        self.f32 = precision == "f32"
        self.adt = torch.float32 if self.f32 else BF16
        self.adt_code = _lib.HC_DTYPE_F32 if self.f32 else _lib.HC_DTYPE_BF16
        self._splits = {}
        self.fine, self.coarse, self.c_in, self.c, self.k, self.lr = fine, coarse, c_in, c, classes, lr
        g = torch.Generator(device="cuda").manual_seed(seed)

        def xavier(co, ci, taps):
            b = math.sqrt(6.0 / ((ci + co) * taps))
            return (torch.rand((co, ci * taps), device="cuda", generator=g) * 2 - 1) * b

        self.w = {"conv1": xavier(c, c_in, 27), "conv2": xavier(2 * c, c, 27), "conv3": xavier(c, 2 * c, 27),
                  "deconv": xavier(2 * c, c, 8), "conv4": xavier(classes, c, 27)}
        nf, nc = fine.total_columns(), coarse.total_columns()
        self.nf, self.nc = nf, nc
        # per-batch maps
        self.fmap_f = nconv.field_map_native(fine, fine, ConvSpec(3, 1, 0, 8, 8), nconv.TILED)
        self.fmap_c = nconv.field_map_native(coarse, coarse, ConvSpec(3, 1, 0, 8, 8), nconv.TILED)
        self.pmap = field_map(fine, coarse, ConvSpec(2, 2, 0, 8, 8))
        self.parent = torch.empty(nf, dtype=torch.int32, device="cuda")
        self.prow = torch.empty(nf, dtype=torch.int8, device="cuda")
        check(lib.hc_native_pool_parents(_p(self.pmap), nc, 8, nf, _p(self.parent), _p(self.prow), _s()))
        self.deconv = nconv.HashDeconv(coarse, fine, self.w["deconv"], ConvSpec(2, 2, 0, c, 2 * c), torch.float32,
                                       precision="f32" if self.f32 else "bf16")
        self.bn = {k: dict(mean=torch.zeros(n, device="cuda"), var=torch.ones(n, device="cuda"),
                           inv=torch.empty(n, device="cuda"))
                   for k, n in (("bn1", c), ("bn2", 2 * c), ("bn3", c))}
        self._dw = nconv.DwWorkspace()
        self._bnws = None
        self._neg = None

    # ------------------------------------------------------------------ pieces
    def _bnws_for(self, n, c):
        need = int(lib.hc_native_bn_workspace(n, c))
        if self._bnws is None or self._bnws.numel() < need:
            self._bnws = torch.empty(need, dtype=torch.uint8, device="cuda")
        return self._bnws

    def _conv(self, fmap, x, name, c_out, dtype=torch.float32, pre_split=False, stats=None):
        """stats: [tiles][c_out][2] fp32 receives the epilogue's per-tile batch-norm statistics
        (hc_native_gather_gemm[_x2]_stats; fp32 output only)."""
        w = self.w[name]
        fm = nconv.as_field_map(fmap)
        if self.f32:  # split rows kept for the layer's dW (pre_split: x already holds them)
            xs = self._splits[name] = x if pre_split else nconv.split(x)
            c_in = w.shape[1] // 27
            wf = nconv.pack_weights_x2(w, c_out, c_in, 27, nconv.PACK_FORWARD)
            if stats is None:
                return nconv.gather_gemm_x2(fmap, xs, wf, c_out)
            y = torch.empty((fm.n, c_out), dtype=torch.float32, device="cuda")
            check(lib.hc_native_gather_gemm_x2_stats(_p(fm.data), fm.layout, fm.n, fm.taps, _p(xs), c_in, _p(wf),
                                                     c_out, _p(y), _p(stats), _s()))
            return y
        wf = nconv.pack_weights(w, c_out, x.shape[1], 27, False)
        if stats is None:
            return nconv.gather_gemm(fmap, x, wf, c_out, dtype)
        y = torch.empty((fm.n, c_out), dtype=torch.float32, device="cuda")
        check(lib.hc_native_gather_gemm_stats(_p(fm.data), fm.layout, fm.n, fm.taps, _p(x), x.shape[1], _p(wf), c_out,
                                              _p(y), _lib.HC_DTYPE_F32, _p(stats), _s()))
        return y

    def _conv_bwd(self, fmap, x, dy, name, need_dx=True, dy_split=False):
        w = self.w[name]
        c_out, c_in = w.shape[0], w.shape[1] // 27
        dx = None
        if self.f32:
            xs = self._splits.pop(name, None)
            dys = dy if dy_split else nconv.split(dy)
            dw = nconv.conv_dw_x2(fmap, xs if xs is not None else nconv.split(x), dys, self._dw)
            if need_dx:
                wb = nconv.pack_weights_x2(w, c_out, c_in, 27, nconv.PACK_BACKWARD)
                dx = nconv.gather_gemm_x2(fmap, dys, wb, c_in)
            return dw, dx
        dw = nconv.conv_dw(fmap, x, dy, self._dw)
        if need_dx:
            wb = nconv.pack_weights(w, c_out, c_in, 27, True)
            dx = nconv.gather_gemm(fmap, dy, wb, c_in, BF16)
        return dw, dx

    def _bn_relu(self, y, name, stats=None):
        """stats: the producing conv's epilogue tile statistics — merged in double in a fixed
        order (hc_native_bn_relu_forward_tiles), no statistics pass over y."""
        n, c = y.shape
        b = self.bn[name]
        xhat = torch.empty_like(y)
        out = torch.empty((n, c), dtype=self.adt, device="cuda")
        ws = self._bnws_for(n, c)
        if stats is not None:
            check(lib.hc_native_bn_relu_forward_tiles(_p(stats), n, c, 0.1, 1e-5, _p(b["mean"]), _p(b["var"]),
                                                      _p(b["inv"]), _p(y), _p(xhat), _p(out), self.adt_code, _p(ws),
                                                      ws.numel(), _s()))
            return out, xhat
        check(lib.hc_native_bn_relu_forward_dt(_p(y), n, c, 1, 0.1, 1e-5, _p(b["mean"]), _p(b["var"]), _p(b["inv"]),
                                               _p(xhat), _p(out), self.adt_code, _p(ws), ws.numel(), _s()))
        return out, xhat

    def _bn_relu_bwd(self, d, dtype, xhat, name, split=False):
        """split (fp32 only): write the split-precision rows the conv backward consumes
        (HC_DTYPE_SPLIT, no separate split pass)."""
        n, c = xhat.shape
        if split:
            out, code = torch.empty((n, 2 * c), dtype=BF16, device="cuda"), _lib.HC_DTYPE_SPLIT
        else:
            out, code = torch.empty((n, c), dtype=self.adt, device="cuda"), self.adt_code
        ws = self._bnws_for(n, c)
        check(lib.hc_native_bn_relu_backward_dt(_p(d), dtype, _p(xhat), _p(self.bn[name]["inv"]), n, c, _p(out),
                                                code, _p(ws), ws.numel(), _s()))
        return out

    # ------------------------------------------------------------------ step
    def step(self, x: torch.Tensor, labels: torch.Tensor, allreduce=None, world: int = 1, trace: dict = None):
        """One training step; x [N_fine][c_in] (bf16, or fp32 at precision f32), labels [N_fine]
        int64. Returns the loss.
        Data parallel: `allreduce` sums the weight gradients over `world` equal shards, which
        are then averaged (the loss is the mean over all voxels of the global batch).
        `trace` (a dict) receives every layer's inputs and outputs and the weight gradients
        (before the update) for the layer-by-layer oracle comparison (tests/test_seg_parity.py)."""
        c, nc, nf = self.c, self.nc, self.nf
        A, AC = self.adt, self.adt_code
        rec = trace.__setitem__ if trace is not None else (lambda k, v: None)
        if trace is not None:
            trace["w"] = {k: v.clone() for k, v in self.w.items()}
        # ---- encoder
        st1 = torch.empty(((nf + 127) // 128, c, 2), device="cuda")  # conv epilogue BN statistics
        y1 = self._conv(self.fmap_f, x, "conv1", c, stats=st1)
        r1, h1 = self._bn_relu(y1, "bn1", st1)
        sw = torch.empty((nc, c), dtype=torch.int8, device="cuda")
        if self.f32:  # the pool writes the split rows conv2 consumes (no split pass)
            p1 = torch.empty((nc, 2 * c), dtype=BF16, device="cuda")
            check(lib.hc_native_max_pool(_p(self.pmap), nc, 8, _p(r1), _lib.HC_DTYPE_SPLIT, c, _p(p1), _p(sw), _s()))
            st2 = torch.empty(((nc + 127) // 128, 2 * c, 2), device="cuda")
            y2 = self._conv(self.fmap_c, p1, "conv2", 2 * c, pre_split=True, stats=st2)
        else:
            p1 = torch.empty((nc, c), dtype=A, device="cuda")
            check(lib.hc_native_max_pool(_p(self.pmap), nc, 8, _p(r1), AC, c, _p(p1), _p(sw), _s()))
            st2 = torch.empty(((nc + 127) // 128, 2 * c, 2), device="cuda")
            y2 = self._conv(self.fmap_c, p1, "conv2", 2 * c, stats=st2)
        e2, h2 = self._bn_relu(y2, "bn2", st2)
        # ---- decoder: unpool(conv3(e2)) + deconv(e2)
        d3 = self._conv(self.fmap_c, e2, "conv3", c, A)
        s3 = self.deconv.forward(e2)  # fp32 (the deconvolution's output dtype)
        up = None
        if trace is not None:  # the unpooled branch on its own (trace only)
            up = torch.empty((nf, c), dtype=A, device="cuda")
            check(lib.hc_native_max_unpool(_p(self.parent), _p(self.prow), nf, _p(d3), AC, c, _p(sw), _p(up), _s()))
        if trace is not None:
            p1t = p1
            if self.f32:  # the fp32 pooled rows the split rows hold (trace only)
                p1t = torch.empty((nc, c), dtype=torch.float32, device="cuda")
                swt = torch.empty_like(sw)
                check(lib.hc_native_max_pool(_p(self.pmap), nc, 8, _p(r1), AC, c, _p(p1t), _p(swt), _s()))
            for k, v in dict(x=x, y1=y1, r1=r1, p1=p1t, sw=sw, y2=y2, e2=e2, d3=d3, up=up, dc=s3.clone()).items():
                rec(k, v)
        # + the unpooled branch, accumulated in place (no unpooled tensor, no separate add pass)
        check(lib.hc_native_max_unpool_add(_p(self.parent), _p(self.prow), nf, _p(d3), AC, c, _p(sw), _p(s3), _s()))
        r3, h3 = self._bn_relu(s3, "bn3")
        scores = self._conv(self.fmap_f, r3, "conv4", self.k)  # [N_fine][K] fp32
        rec("r3", r3)
        rec("scores", scores)
        # ---- per-voxel softmax cross-entropy (mean over voxels)
        logp = torch.log_softmax(scores, dim=1)
        loss = -logp.gather(1, labels[:, None]).mean()
        dscores = logp.exp_()  # softmax, in place (the loss has been gathered)
        if self._neg is None or self._neg.shape[0] != nf:
            self._neg = torch.full((nf, 1), -1.0, device="cuda")
        dscores.scatter_add_(1, labels[:, None], self._neg)
        dscores = dscores.mul_(1.0 / nf).to(A)
        # ---- backward
        g = {}
        g["conv4"], d_r3 = self._conv_bwd(self.fmap_f, r3, dscores, "conv4")
        d_s3 = self._bn_relu_bwd(d_r3, AC, h3, "bn3")                          # [N_fine][C]
        g["deconv"], d_e2a = self.deconv.backward(d_s3, e2)                    # deconv branch
        d_d3 = torch.empty((nc, c), dtype=A, device="cuda")                     # unpool branch: adjoint =
        check(lib.hc_native_switch_gather(_p(self.pmap), nc, 8, _p(d_s3), AC, c, _p(sw), _p(d_d3), _s()))
        g["conv3"], d_e2b = self._conv_bwd(self.fmap_c, e2, d_d3, "conv3")
        if trace is not None:
            for k, v in dict(dscores=dscores, d_r3=d_r3, d_s3=d_s3, d_e2a=d_e2a.clone(), d_d3=d_d3,
                             d_e2b=d_e2b).items():
                rec(k, v)
        d_e2 = d_e2a.float()  # fp32 already (no copy)
        d_e2.add_(d_e2b)
        d_e2 = d_e2.contiguous()
        d_y2 = self._bn_relu_bwd(d_e2, _lib.HC_DTYPE_F32, h2, "bn2", split=self.f32)
        g["conv2"], d_p1 = self._conv_bwd(self.fmap_c, p1, d_y2, "conv2", dy_split=self.f32)
        if trace is not None and self.f32:  # fp32 rows for the oracle comparison (trace only)
            d_y2 = self._bn_relu_bwd(d_e2, _lib.HC_DTYPE_F32, h2, "bn2")
        d_r1 = torch.empty((nf, c), dtype=A, device="cuda")                    # pool backward = unpool
        check(lib.hc_native_max_unpool(_p(self.parent), _p(self.prow), nf, _p(d_p1), AC, c, _p(sw), _p(d_r1), _s()))
        d_y1 = self._bn_relu_bwd(d_r1, AC, h1, "bn1", split=self.f32)
        g["conv1"], _ = self._conv_bwd(self.fmap_f, x, d_y1, "conv1", need_dx=False, dy_split=self.f32)
        if trace is not None and self.f32:
            d_y1 = self._bn_relu_bwd(d_r1, AC, h1, "bn1")
        if trace is not None:
            for k, v in dict(d_y2=d_y2, d_p1=d_p1, d_r1=d_r1, d_y1=d_y1).items():
                rec(k, v)
            trace["grads"] = {k: v.clone() for k, v in g.items()}
        if allreduce is not None:
            allreduce(list(g.values()))
        for k, gr in g.items():  # plain SGD
            self.w[k].sub_((self.lr / world) * gr)
        return loss
