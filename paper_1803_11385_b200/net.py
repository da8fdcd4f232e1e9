"""Native H-CNN classification net on the B200 path.

The LeNet-style hierarchy of net.hpp:40-60 / net.cpp:181-375 — per level, finest to
resolution 4: hash conv 3^3 -> batch norm -> ReLU -> 2^3 max pool; the last level's
output goes through the final 2^3 dense pool, dropout -> FC(128) -> dropout ->
FC(classes) -> softmax cross-entropy; SGD with momentum and weight decay — built from the
native kernels: tcgen05 implicit-GEMM conv (conv.py), and voxel-major pooling, batch
norm + ReLU, dense pool and SGD (csrc/net_ops.cu). The two FC layers (b x 1024 -> 128 ->
classes) are plain cuBLAS GEMMs through torch.

Layout: features are voxel-major [N][C]; channel counts are padded to the tensor-core
tile set (input 3 -> 8 channels, 8 output channels -> 16) with zero weights, so padded
channels stay exactly zero through conv, batch norm (xhat = 0), pooling and SGD.
Field maps (conv K0 tile-major, pool maps and their inverses, the dense-pool child map)
depend only on the batch's PSH tables and are built once per batch (`NetBatch`).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from . import conv as nconv
from ._lib import check, lib
from .ops import ConvSpec, field_map, locate
from .psh import SuperPsh

BF16 = torch.bfloat16


def _p(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def channels_at_level(level: int) -> int:
    """net.cpp:15-17: max{2, 2^(9-l)}."""
    return max(2, 1 << max(0, 9 - level))


def _pad_in(c: int) -> int:
    return (c + 7) // 8 * 8


def _pad_out(c: int) -> int:
    for t in (16, 32, 64, 128, 256):
        if c <= t:
            return t
    raise ValueError("native net: at most 256 channels per level")


_QUERIES = {}


def _dense_queries(b: int) -> torch.Tensor:
    """{model, x, y, z} of every (model, cell, child) of the final dense pool (device, cached)."""
    if b not in _QUERIES:
        q = []
        for v in range(1, b + 1):
            for cell in range(8):
                qx, qy, qz = cell & 1, (cell >> 1) & 1, (cell >> 2) & 1
                for dz in range(2):
                    for dy in range(2):
                        for dx in range(2):
                            q.append((v, qx * 2 + dx, qy * 2 + dy, qz * 2 + dz))
        _QUERIES[b] = torch.tensor(q, dtype=torch.int32, device="cuda")
    return _QUERIES[b]


@dataclass
class NetBatch:
    """Device-side per-batch structure: one SuperPsh per level (finest first) plus the maps
    every layer needs. Mirrors net.hpp:22-31 MultiLevelBatch."""

    levels: List[SuperPsh]
    conv_maps: list
    pool_maps: list
    parents: list
    dense_children: torch.Tensor

    @classmethod
    def build(cls, levels: Sequence[SuperPsh]) -> "NetBatch":
        levels = list(levels)
        if levels[-1].resolution != 4:
            raise RuntimeError("final pool expects the resolution-4 level")
        conv_maps, pool_maps, parents = [], [], []
        for i, s in enumerate(levels):
            conv_maps.append(nconv.field_map_native(s, s, ConvSpec(3, 1, 0, 8, 8), nconv.TILED))
            if i + 1 < len(levels):
                c = levels[i + 1]
                pm = field_map(s, c, ConvSpec(2, 2, 0, 8, 8))  # [N_coarse][8] fine columns
                par = torch.empty(s.total_columns(), dtype=torch.int32, device="cuda")
                prow = torch.empty(s.total_columns(), dtype=torch.int8, device="cuda")
                check(lib.hc_native_pool_parents(_p(pm), pm.shape[0], 8, s.total_columns(), _p(par), _p(prow), _s()))
                pool_maps.append(pm)
                parents.append((par, prow))
        # dense-pool children: [b][8 cells][8 kids] (net.cpp:76-88: cell q unflattened x-fastest,
        # kids in (dz, dy, dx) order)
        last = levels[-1]
        b = last.batch
        kids = locate(last, _dense_queries(b)).to(torch.int32)
        return cls(levels, conv_maps, pool_maps, parents, kids.view(b, 8, 8).contiguous())

    @property
    def batch(self) -> int:
        return self.levels[0].batch


class NativeHashNet:
    """net.hpp:40-60 LayerGraph + net.cpp training step on the native path."""

    def __init__(self, level_max: int, num_classes: int, seed: int = 0, input_channels: int = 3,
                 dropout: float = 0.5, lr: float = 0.1, momentum: float = 0.9, weight_decay: float = 5e-4,
                 bn_momentum: float = 0.1, bn_eps: float = 1e-5, sync_bn=None, precision: str = "bf16"):
        """sync_bn: data parallelism with whole-batch statistics — a callable
        that sums a float64 CUDA tensor in place over the ranks (e.g. dist.sum_over_ranks);
        batch norm then normalises over the global batch, as the reference does for one
        process (cnn_ops.cpp:456-470). None: statistics over this process's batch.
        precision: "bf16" — bf16 conv operands and activations (fp32 accumulation); "f32" — the
        reference's precision: fp32 activations and gradients, every conv (forward, dW, dX)
        through the split-precision tcgen05 kernels (bf16 hi/lo planes, within 1e-5 of fp64)."""
        if precision not in ("bf16", "f32"):
            raise ValueError("precision must be 'bf16' or 'f32'")
        self.f32 = precision == "f32"
        self.adt = torch.float32 if self.f32 else BF16  # activation / conv-gradient dtype
        self.adt_code = _lib.HC_DTYPE_F32 if self.f32 else _lib.HC_DTYPE_BF16
        # batch-norm statistics from the conv epilogue (per-tile sums merged in double) instead of
        # two passes over the conv output; sync BN keeps the phased path (its sums are all-reduced)
        self.epilogue_stats = True
        if level_max < 2 or level_max > 16:
            raise ValueError("level_max out of range")
        if num_classes < 2:
            raise ValueError("need at least two classes")
        self.level_max, self.num_classes, self.input_channels = level_max, num_classes, input_channels
        self.dropout, self.lr, self.momentum, self.wd = dropout, lr, momentum, weight_decay
        self.bn_momentum, self.bn_eps = bn_momentum, bn_eps
        self.sync_bn = sync_bn
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.blocks = []
        for lvl in range(level_max, 1, -1):
            cin = input_channels if lvl == level_max else channels_at_level(lvl + 1)
            cout = channels_at_level(lvl)
            cin_p = _pad_in(cin) if lvl == level_max else _pad_out(cin)
            cout_p = _pad_out(cout)
            bound = math.sqrt(6.0 / (cin * 27 + cout * 27))  # net.cpp:60-65 xavier (fan = C*27)
            w = torch.zeros((cout_p, cin_p * 27), device="cuda")
            wr = (torch.rand((cout, cin * 27), device="cuda", generator=g) * 2 - 1) * bound
            w.view(cout_p, cin_p, 27)[:cout, :cin] = wr.view(cout, cin, 27)
            self.blocks.append(dict(level=lvl, cin=cin, cout=cout, cin_p=cin_p, cout_p=cout_p, w=w,
                                    v=torch.zeros_like(w),
                                    run_mean=torch.zeros(cout_p, device="cuda"),
                                    run_var=torch.ones(cout_p, device="cuda"),  # cnn_ops.hpp:125-127
                                    inv_std=torch.empty(cout_p, device="cuda")))
        head_in = channels_at_level(2) * 8
        b1 = math.sqrt(6.0 / (head_in + 128))
        b2 = math.sqrt(6.0 / (128 + num_classes))
        self.fc1_w = (torch.rand((128, head_in), device="cuda", generator=g) * 2 - 1) * b1
        self.fc1_b = torch.zeros(128, device="cuda")
        self.fc2_w = (torch.rand((num_classes, 128), device="cuda", generator=g) * 2 - 1) * b2
        self.fc2_b = torch.zeros(num_classes, device="cuda")
        self.head_v = [torch.zeros_like(t) for t in (self.fc1_w, self.fc1_b, self.fc2_w, self.fc2_b)]
        self._ws = {}
        self._dw_ws = nconv.DwWorkspace()
        self._wb = {}  # f32: dX weight operands packed in the forward pass
        self._seed = seed + 1
        self._gen = None  # dropout masks: a private generator in eager mode, the default one in graphs

    # ------------------------------------------------------------------ helpers
    def reference_weights(self, i: int) -> torch.Tensor:
        """Block i's conv weights in the reference layout W[co][ci*27 + t] (unpadded)."""
        b = self.blocks[i]
        return b["w"].view(b["cout_p"], b["cin_p"], 27)[:b["cout"], :b["cin"]].reshape(b["cout"], b["cin"] * 27)

    def set_reference_weights(self, i: int, w_ref: torch.Tensor) -> None:
        b = self.blocks[i]
        b["w"].zero_()
        b["w"].view(b["cout_p"], b["cin_p"], 27)[:b["cout"], :b["cin"]] = w_ref.view(b["cout"], b["cin"], 27)

    def _bn_ws(self, n: int, c: int) -> torch.Tensor:
        nbytes = int(lib.hc_native_bn_workspace(n, c))
        t = self._ws.get("bn")
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
            self._ws["bn"] = t
        return t

    def _sync_sums(self, buf: torch.Tensor, n: int, c: int) -> torch.Tensor:
        """All-reduce per-channel double sums buf[0:2c] TOGETHER with this rank's row count
        (buf[2c] = n), so every step's global count rides in the same collective (ranks whose
        shard sizes differ from step to step stay in lock step; no host synchronisation, so the
        step still captures into a CUDA graph). Returns the global count as a device scalar."""
        buf[2 * c:].fill_(float(n))
        self.sync_bn(buf)
        return buf[2 * c:]

    def _bn_relu_forward(self, i: int, y: torch.Tensor, xhat: torch.Tensor, r: torch.Tensor) -> None:
        blk = self.blocks[i]
        n, c = y.shape
        ws = self._bn_ws(n, c)
        if self.sync_bn is None:
            check(lib.hc_native_bn_relu_forward_dt(_p(y), n, c, 1, self.bn_momentum, self.bn_eps,
                                                   _p(blk["run_mean"]), _p(blk["run_var"]), _p(blk["inv_std"]),
                                                   _p(xhat), _p(r), self.adt_code, _p(ws), ws.numel(), _s()))
            return
        # the sums are divided by the global count on the device (the same IEEE double ops
        # hc_native_bn_finalize applies), then finalised with n_total = 1
        sxb = torch.empty(2 * c + 1, dtype=torch.float64, device="cuda")
        sq = torch.empty((2, c), dtype=torch.float64, device="cuda")
        mean = torch.empty(c, dtype=torch.float64, device="cuda")
        check(lib.hc_native_bn_stat(0, _p(y), None, 0, n, c, None, _p(sxb), _p(ws), ws.numel(), _s()))
        nt = self._sync_sums(sxb, n, c)
        sx = (sxb[:c] / nt).contiguous()
        check(lib.hc_native_bn_finalize(_p(sx), None, 1, c, 0.0, 0.0, None, None, _p(mean), None, _s()))
        check(lib.hc_native_bn_stat(1, _p(y), None, 0, n, c, _p(mean), _p(sq), _p(ws), ws.numel(), _s()))
        self.sync_bn(sq)
        sq0 = (sq[0] / nt).contiguous()
        check(lib.hc_native_bn_finalize(_p(sx), _p(sq0), 1, c, self.bn_momentum, self.bn_eps, _p(blk["run_mean"]),
                                        _p(blk["run_var"]), _p(mean), _p(blk["inv_std"]), _s()))
        check(lib.hc_native_bn_relu_apply_dt(_p(y), n, c, _p(mean), _p(blk["inv_std"]), _p(xhat), _p(r), self.adt_code,
                                             _s()))

    def _bn_relu_backward(self, i: int, d_relu: torch.Tensor, d_dtype: int, xhat: torch.Tensor,
                          d_conv: torch.Tensor, out_code: Optional[int] = None) -> None:
        blk = self.blocks[i]
        out_code = self.adt_code if out_code is None else out_code
        n, c = xhat.shape
        ws = self._bn_ws(n, c)
        if self.sync_bn is None:
            check(lib.hc_native_bn_relu_backward_dt(_p(d_relu), d_dtype, _p(xhat), _p(blk["inv_std"]), n, c,
                                                    _p(d_conv), out_code, _p(ws), ws.numel(), _s()))
            return
        stb = torch.empty(2 * c + 1, dtype=torch.float64, device="cuda")
        check(lib.hc_native_bn_stat(2, _p(xhat), _p(d_relu), d_dtype, n, c, None, _p(stb), _p(ws), ws.numel(), _s()))
        nt = self._sync_sums(stb, n, c)
        st = (stb[:2 * c].view(2, c) * (1.0 / nt)).contiguous()  # s * inv_n, as the kernel forms it
        check(lib.hc_native_bn_relu_backward_apply_dt(_p(d_relu), d_dtype, _p(xhat), _p(blk["inv_std"]), n, c,
                                                      _p(st[0]), _p(st[1]), 1, _p(d_conv), out_code, _s()))

    def input_features(self, ref: torch.Tensor) -> torch.Tensor:
        """Finest-level data (C x N fp32, psh data array) -> padded voxel-major (bf16, or fp32 at
        precision f32)."""
        c, n = ref.shape
        x = torch.zeros((n, self.blocks[0]["cin_p"]), dtype=self.adt, device="cuda")
        x[:, :c] = nconv.to_voxel_major(ref) if not self.f32 else ref.t()
        return x

    def _conv_forward(self, i: int, x: torch.Tensor, stats: Optional[torch.Tensor] = None):
        """Block i's conv: returns (fp32 output, what the backward needs of the input). stats:
        [tiles][c_out][2] fp32 receives the epilogue's per-tile batch-norm statistics."""
        blk = self.blocks[i]
        fm = self._maps[i]
        n, co = fm.n, blk["cout_p"]
        y = torch.empty((n, co), dtype=torch.float32, device="cuda")
        if self.f32:
            # split rows arrive straight from the previous level's pool (HC_DTYPE_SPLIT output)
            xs = x if x.dtype == BF16 else nconv.split(x)
            # forward and dX operands in one launch; the dX one is kept for the backward pass (the
            # tensor-core tile set starts at 16 output channels: an 8-channel input level takes its
            # gradient through a zero-padded 16-channel kernel)
            cin_g = max(16, blk["cin_p"])
            wf = torch.empty((2 * co, int(lib.hc_native_packed_k_x2(blk["cin_p"], 27))), dtype=BF16, device="cuda")
            wb = torch.empty((2 * cin_g, int(lib.hc_native_packed_k_x2(co, 27))), dtype=BF16, device="cuda")
            check(lib.hc_native_pack_weights_x2_fb(_p(blk["w"]), co, blk["cin_p"], 27, cin_g, _p(wf), _p(wb), _s()))
            self._wb[i] = wb
            check(lib.hc_native_gather_gemm_x2_stats(_p(fm.data), fm.layout, n, fm.taps, _p(xs), blk["cin_p"], _p(wf),
                                                     co, _p(y), _p(stats) if stats is not None else None, _s()))
            return y, xs
        wf = nconv.pack_weights(blk["w"], co, blk["cin_p"], 27, False)
        check(lib.hc_native_gather_gemm_stats(_p(fm.data), fm.layout, n, fm.taps, _p(x), blk["cin_p"], _p(wf), co,
                                              _p(y), _lib.HC_DTYPE_F32, _p(stats) if stats is not None else None,
                                              _s()))
        return y, x

    # ------------------------------------------------------------------ forward / backward
    def forward(self, nb: NetBatch, x: torch.Tensor, training: bool = True, cache: Optional[dict] = None):
        """net.cpp:181-258 net_forward: class scores (classes x b). training=True: batch
        statistics (running stats updated) and dropout; training=False: the running statistics
        normalise and dropout is the identity (net.cpp:203-208, 232-241)."""
        acts = []
        self._maps = nb.conv_maps
        for i, blk in enumerate(self.blocks):
            s = nb.levels[i]
            n = s.total_columns()
            fused = training and self.sync_bn is None and self.epilogue_stats
            stats = torch.empty(((n + 127) // 128, blk["cout_p"], 2), device="cuda") if fused else None
            y, x_saved = self._conv_forward(i, x, stats)
            r = torch.empty((n, blk["cout_p"]), dtype=self.adt, device="cuda")
            if fused:  # batch-norm statistics from the conv epilogue: fold + apply (2 launches)
                xhat = torch.empty_like(y)
                ws = self._bn_ws(n, blk["cout_p"])
                check(lib.hc_native_bn_relu_forward_tiles(_p(stats), n, blk["cout_p"], self.bn_momentum, self.bn_eps,
                                                          _p(blk["run_mean"]), _p(blk["run_var"]), _p(blk["inv_std"]),
                                                          _p(y), _p(xhat), _p(r), self.adt_code, _p(ws), ws.numel(),
                                                          _s()))
            elif training:
                xhat = torch.empty_like(y)
                self._bn_relu_forward(i, y, xhat, r)
            else:
                xhat = None
                check(lib.hc_native_bn_relu_inference_dt(_p(y), n, blk["cout_p"], _p(blk["run_mean"]),
                                                         _p(blk["run_var"]), self.bn_eps, _p(r), self.adt_code, _s()))
            acts.append(dict(x=x_saved, xhat=xhat))
            if cache is not None and cache.get("trace") is not None:
                cache["trace"].setdefault("blocks", []).append(dict(x=x, y=y.clone(), r=r))
            if i + 1 < len(self.blocks):
                pm = nb.pool_maps[i]
                nc = pm.shape[0]
                sw = torch.empty((nc, blk["cout_p"]), dtype=torch.int8, device="cuda")
                if self.f32:  # fp32 max, written as the split rows the next conv consumes
                    pooled = torch.empty((nc, 2 * blk["cout_p"]), dtype=BF16, device="cuda")
                    code = _lib.HC_DTYPE_SPLIT
                else:
                    pooled = torch.empty((nc, blk["cout_p"]), dtype=self.adt, device="cuda")
                    code = self.adt_code
                check(lib.hc_native_max_pool(_p(pm), nc, 8, _p(r), code, blk["cout_p"], _p(pooled), _p(sw), _s()))
                acts[-1]["sw"] = sw
                if cache is not None and cache.get("trace") is not None:
                    cache["trace"]["blocks"][-1].update(pooled=pooled, sw=sw)
                x = pooled
            else:
                b = nb.batch
                c = blk["cout_p"]
                head = torch.empty((c * 8, b), device="cuda")
                src = torch.empty((c * 8, b), dtype=torch.int32, device="cuda")
                check(lib.hc_native_dense_pool_dt(_p(nb.dense_children), b, _p(r), self.adt_code, c, _p(head), _p(src),
                                                  _s()))
                acts[-1]["src"] = src
                x = head
        # head: dropout -> FC(128) -> dropout -> FC(classes)   (net.cpp:236-251)
        if not training:
            fc1_out = self.fc1_w @ x + self.fc1_b[:, None]
            return self.fc2_w @ fc1_out + self.fc2_b[:, None]
        keep = 1.0 - self.dropout
        if self._gen is None and not torch.cuda.is_current_stream_capturing():
            self._gen = torch.Generator(device="cuda").manual_seed(self._seed)
        gen = None if torch.cuda.is_current_stream_capturing() else self._gen
        def dropout(t):  # uniform draws from torch's (graph-safe) generator; mask and product in one launch
            t = t.contiguous()
            u = torch.rand(t.shape, device="cuda", generator=gen)
            m, o = torch.empty_like(t), torch.empty_like(t)
            check(lib.hc_native_dropout_apply(_p(u), _p(t), t.numel(), keep, _p(m), _p(o), _s()))
            return m, o
        m1, fc1_in = dropout(x)
        fc1_out = torch.addmm(self.fc1_b[:, None], self.fc1_w, fc1_in)  # bias in the GEMM epilogue
        m2, fc2_in = dropout(fc1_out)
        scores = torch.addmm(self.fc2_b[:, None], self.fc2_w, fc2_in)
        if cache is not None:
            cache.update(acts=acts, m1=m1, m2=m2, fc1_in=fc1_in, fc2_in=fc2_in)
        return scores

    def predict(self, nb: NetBatch, x: torch.Tensor) -> torch.Tensor:
        """Inference (running statistics, no dropout): predicted class per shape."""
        return self.forward(nb, x, training=False).argmax(0)

    def loss_and_gradients(self, nb: NetBatch, x: torch.Tensor, labels: torch.Tensor,
                           global_batch: Optional[int] = None, trace: Optional[dict] = None):
        """net.cpp:260-323: softmax cross-entropy (mean over the batch), gradients of every
        conv and FC weight; returns (loss tensor, conv weight gradients (padded ref layout),
        FC gradients). With data parallelism the scores' gradient is divided by the GLOBAL
        batch (net.cpp:281 divides by b; shards must not divide by their local b)."""
        cache = {"trace": trace}
        scores = self.forward(nb, x, True, cache)
        classes, b = scores.shape
        # softmax cross-entropy and its gradient in one launch (hc_native_softmax_xent, double
        # log-sum-exp per shape). The reference's loss is the mean over the whole batch
        # (net.cpp:283): with data parallelism each rank returns its share, sum / global_batch,
        # so the ranks' losses add up to the global mean
        scores = scores.contiguous()
        lab = labels.to(device="cuda", dtype=torch.int64).contiguous()
        loss_t = torch.empty(1, dtype=torch.float64, device="cuda")
        dscores = torch.empty_like(scores)
        check(lib.hc_native_softmax_xent(_p(scores), classes, b, _p(lab), int(global_batch or b), _p(loss_t),
                                         _p(dscores), _s()))
        loss = loss_t[0]
        g_fc2_w = dscores @ cache["fc2_in"].t()
        g_fc2_b = dscores.sum(1)
        d_fc1_out = (self.fc2_w.t() @ dscores) * cache["m2"]
        g_fc1_w = d_fc1_out @ cache["fc1_in"].t()
        g_fc1_b = d_fc1_out.sum(1)
        d_head = ((self.fc1_w.t() @ d_fc1_out) * cache["m1"]).contiguous()
        acts = cache["acts"]
        conv_grads = [None] * len(self.blocks)
        d_relu, d_dtype = None, None
        for i in range(len(self.blocks) - 1, -1, -1):
            blk, a = self.blocks[i], acts[i]
            s = nb.levels[i]
            n, c = s.total_columns(), blk["cout_p"]
            if i == len(self.blocks) - 1:  # net.cpp:301-304 final_dense_pool_backward
                d_relu = torch.empty((n, c), device="cuda")
                check(lib.hc_native_dense_pool_backward(_p(d_head), _p(a["src"]), nb.batch, c, n, _p(d_relu), _s()))
                d_dtype = _lib.HC_DTYPE_F32
            if self.f32:  # the BN backward writes the split rows dW / dX consume (no split pass)
                d_conv = d_conv_s = torch.empty((n, 2 * c), dtype=BF16, device="cuda")
                self._bn_relu_backward(i, d_relu, d_dtype, a["xhat"], d_conv, _lib.HC_DTYPE_SPLIT)
            else:
                d_conv = torch.empty((n, c), dtype=self.adt, device="cuda")
                self._bn_relu_backward(i, d_relu, d_dtype, a["xhat"], d_conv)
            if self.f32:  # a["x"] holds the split input rows
                conv_grads[i] = nconv.conv_dw_x2(nb.conv_maps[i], a["x"], d_conv_s, self._dw_ws)
            else:
                conv_grads[i] = nconv.conv_dw(nb.conv_maps[i], a["x"], d_conv, self._dw_ws)
            if trace is not None:
                trace["blocks"][i].update(d_relu=d_relu, d_conv=d_conv, dw=conv_grads[i].clone())
            # input gradient (net.cpp:316-317; the finest one is the net's input gradient, g.input).
            # The tensor-core tile set starts at 16 output channels: an 8-channel input level
            # takes its gradient through a zero-padded 16-channel kernel.
            cin_g = max(16, blk["cin_p"])
            if self.f32:  # the operand packed with the forward one (_conv_forward)
                dx = nconv.gather_gemm_x2(nb.conv_maps[i], d_conv_s, self._wb.pop(i), cin_g)[:, :blk["cin_p"]]
            else:
                w = blk["w"]
                if cin_g != blk["cin_p"]:
                    w = torch.zeros((blk["cout_p"], cin_g * 27), device="cuda")
                    w.view(blk["cout_p"], cin_g, 27)[:, :blk["cin_p"]] = blk["w"].view(blk["cout_p"], blk["cin_p"], 27)
                wb = nconv.pack_weights(w, blk["cout_p"], cin_g, 27, True)
                dx = nconv.gather_gemm(nb.conv_maps[i], d_conv, wb, cin_g, BF16)[:, :blk["cin_p"]]
            if trace is not None:
                trace["blocks"][i]["dx"] = dx
            if i > 0:  # net.cpp:296-300: unpool through the finer level's switches
                prev = self.blocks[i - 1]
                par, prow = nb.parents[i - 1]
                nf = nb.levels[i - 1].total_columns()
                d_relu = torch.empty((nf, prev["cout_p"]), dtype=self.adt, device="cuda")
                check(lib.hc_native_max_unpool(_p(par), _p(prow), nf, _p(dx.contiguous()), self.adt_code,
                                               prev["cout_p"], _p(acts[i - 1]["sw"]), _p(d_relu), _s()))
                d_dtype = self.adt_code
        head_grads = (g_fc1_w, g_fc1_b, g_fc2_w, g_fc2_b)
        return loss, conv_grads, head_grads

    def train_step(self, nb: NetBatch, x: torch.Tensor, labels: torch.Tensor, allreduce=None,
                   global_batch: Optional[int] = None):
        """net.cpp:349-375 train_step: loss + SGD with momentum and weight decay. `allreduce`
        (e.g. dist.allreduce_gradients) sums the gradients over data-parallel ranks first."""
        loss, conv_grads, head_grads = self.loss_and_gradients(nb, x, labels, global_batch)
        head_grads = [g.contiguous() for g in head_grads]  # the tensors reduced ARE the ones applied
        if allreduce is not None:
            allreduce(list(conv_grads) + head_grads)
        # every conv and FC tensor in one multi-tensor launch (net.cpp:339-346 per tensor)
        ws = [blk["w"] for blk in self.blocks] + [self.fc1_w, self.fc1_b, self.fc2_w, self.fc2_b]
        vs = [blk["v"] for blk in self.blocks] + list(self.head_v)
        gs = list(conv_grads) + list(head_grads)
        k = len(ws)
        arr = lambda ts: (C.c_void_p * k)(*[t.data_ptr() for t in ts])  # noqa: E731
        ns = (C.c_int64 * k)(*[t.numel() for t in ws])
        check(lib.hc_native_sgd_update_multi(arr(ws), arr(vs), arr(gs), ns, k, self.lr, self.momentum, self.wd,
                                             _s()))
        return loss


class GraphedStep:
    """A whole training step (per-batch maps + forward + backward + [all-reduce] + SGD)
    captured once as a CUDA graph and replayed: ~100 launches per step become one graph
    launch, so small batches are not host-bound. Valid while the batch's structure
    tensors, the input features and the labels stay at the captured addresses (the
    tables of a new batch of the same shapes are copied in place)."""

    def __init__(self, net: NativeHashNet, levels: Sequence[SuperPsh], x: torch.Tensor, labels: torch.Tensor,
                 allreduce=None, global_batch: Optional[int] = None, warmup: int = 2):
        self.net, self.levels, self.x, self.labels = net, list(levels), x, labels
        self.allreduce, self.global_batch = allreduce, global_batch
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):  # allocator / attribute setup outside the capture
                self._step()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        before = int(lib.hc_launch_count())
        with torch.cuda.graph(self.graph):
            self.loss = self._step()
        # this library's kernels captured per step (replays do not pass through the host
        # launch counter; callers multiply by the replays they time)
        self.launches_per_step = int(lib.hc_launch_count()) - before

    def _step(self):
        nb = NetBatch.build(self.levels)
        return self.net.train_step(nb, self.x, self.labels, self.allreduce, self.global_batch)

    def __call__(self):
        self.graph.replay()
        return self.loss
