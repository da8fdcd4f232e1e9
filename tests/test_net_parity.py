"""The native classification net (net.py, net.cpp:181-323) layer by layer at BASELINE config 2
size — 64^3 shells x 32, five conv / BN+ReLU / max-pool levels — against the double oracle
(oracle/hc_oracle.c conv_forward / conv_backward / max_pool / max_unpool = cnn_ops.cpp:206-372).

Every oracle call takes the native step's own inputs for that layer (its bf16 activations and
gradients, bf16-quantised weights: exact in double), so each operator is checked on its own:
conv outputs (fp32) within 1e-5, weight gradients within 5e-5, bf16-output input gradients and
BN+ReLU outputs within 2^-8 (one bf16 rounding), pooling values / switches and the unpooling of
the backward pass bit-exact. (tests/test_net_gpu.py keeps the end-to-end comparison with the
unmodified reference net as a smoke test.)"""
import os
import sys

import numpy as np
import pytest
import torch

from helpers import levels_to_arrays

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200.ops import ConvSpec  # noqa: E402
from paper_1803_11385_b200.psh import SuperPsh  # noqa: E402

F64 = np.float64
TOL_F32, TOL_DW, TOL_BF16 = 1e-5, 5e-5, 2.0 ** -8


def cm(t: torch.Tensor) -> np.ndarray:
    return t.float().t().contiguous().cpu().numpy().astype(F64)


def rel(a, b) -> float:
    a, b = np.asarray(a, F64), np.asarray(b, F64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def cfg2_trace(cuda):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_1803_11385_b200 import net as nnet
    b = 32
    pyr = bench.shell_pyramid(64)
    levels = [SuperPsh.from_levels([lv] * b) for lv in pyr]
    arrays = [levels_to_arrays([lv] * b) for lv in pyr]
    net = nnet.NativeHashNet(6, 40, seed=3)
    feats = np.concatenate([pyr[0].arrays()[3]] * b, axis=1)
    x = net.input_features(torch.from_numpy(np.ascontiguousarray(feats)).cuda())
    labels = torch.arange(b, device="cuda") % 40
    nb = nnet.NetBatch.build(levels)
    net.train_step(nb, x, labels)  # one real step first: weights, momenta and running stats move
    tr = {}
    net.loss_and_gradients(nb, x, labels, trace=tr)
    torch.cuda.synchronize()
    assert [s.total_columns() for s in levels] == [451840, 103936, 27904, 7168, 1792]
    return net, arrays, tr


def test_cfg2_forward_layers_vs_oracle(cfg2_trace, restated):
    net, arrays, tr = cfg2_trace
    for i, (blk, t) in enumerate(zip(net.blocks, tr["blocks"])):
        s = arrays[i]
        spec = ConvSpec(3, 1, 0, blk["cin_p"], blk["cout_p"])
        w = blk["w"].to(torch.bfloat16).float().cpu().numpy().astype(F64)
        y64 = restated.conv_forward(s, cm(t["x"]), s, w, spec, F64)
        assert rel(cm(t["y"]), y64) <= TOL_F32, (i, rel(cm(t["y"]), y64))
        # BN (batch statistics, cnn_ops.cpp:456-475) + ReLU on the native conv output
        y = t["y"].double().cpu().numpy()
        mean, var = y.mean(0), y.var(0)
        want = np.maximum((y - mean) / np.sqrt(var + net.bn_eps), 0.0)
        assert rel(t["r"].float().cpu().numpy(), want) <= TOL_BF16, i
        if i + 1 < len(net.blocks):
            pool = ConvSpec(2, 2, 0, blk["cout_p"], blk["cout_p"])
            mp, sw = restated.max_pool(s, cm(t["r"]), arrays[i + 1], pool, F64)
            assert np.array_equal(cm(t["pooled"]), mp), i
            assert np.array_equal(t["sw"].t().cpu().numpy().astype(np.int32), sw), i


def test_cfg2_backward_layers_vs_oracle(cfg2_trace, restated):
    net, arrays, tr = cfg2_trace
    nblk = len(net.blocks)
    for i in range(nblk - 1, -1, -1):
        blk, t, s = net.blocks[i], tr["blocks"][i], arrays[i]
        spec = ConvSpec(3, 1, 0, blk["cin_p"], blk["cout_p"])
        w = blk["w"].to(torch.bfloat16).float().cpu().numpy().astype(F64)
        cols = restated.hash2col(s, cm(t["x"]), s, spec, F64)
        dw64, dx64 = restated.conv_backward(cm(t["d_conv"]), w, cols, s, s, spec, F64)
        assert rel(t["dw"].cpu().numpy(), dw64) <= TOL_DW, (i, rel(t["dw"].cpu().numpy(), dw64))
        assert rel(cm(t["dx"]), dx64) <= TOL_BF16, (i, rel(cm(t["dx"]), dx64))
        if i + 1 < nblk:  # this level's ReLU gradient = unpool of the coarser level's dX (net.cpp:296-300)
            pool = ConvSpec(2, 2, 0, blk["cout_p"], blk["cout_p"])
            sw = t["sw"].t().cpu().numpy().astype(np.int32)
            up = restated.max_unpool(cm(tr["blocks"][i + 1]["dx"]), sw, s, arrays[i + 1], pool, F64)
            assert np.array_equal(cm(t["d_relu"]), up), i
