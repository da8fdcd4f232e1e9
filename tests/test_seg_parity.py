"""Segmentation composition (BASELINE config 4): every hash operator of
one NativeSegNet training step (paper_1803_11385_b200/seg.py) against the SAME operator of the
double-precision oracle (oracle/hc_oracle.c: conv_forward / conv_backward, max_pool,
max_unpool, deconv_forward / deconv_backward = cnn_ops.cpp:206-435), layer by layer.

Each oracle call is fed the native path's own inputs for that layer (its bf16 activations and
bf16-quantised weights, exactly representable in double), so the comparison isolates the
operator: fp32-output contractions within 1e-5 (normwise), weight gradients within 5e-5,
bf16-output contractions within 2^-8 (one bf16 rounding of the output), pooling values,
switches and unpooling bit-exact. At precision "f32" (fp32 activations, every contraction through the
split-precision kernels) the oracle gets the unquantised fp32 weights and activations and every
contraction — outputs, input gradients and weight gradients — is within 1e-5 normwise."""
import numpy as np
import pytest
import torch

from helpers import levels_to_arrays, shell_pair

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200.ops import ConvSpec  # noqa: E402
from paper_1803_11385_b200.psh import SuperPsh  # noqa: E402

F64 = np.float64
TOL_F32, TOL_DW, TOL_BF16 = 1e-5, 5e-5, 2.0 ** -8


def cm(t: torch.Tensor) -> np.ndarray:
    """native voxel-major [N][C] -> reference channel-major C x N float64"""
    return t.float().t().contiguous().cpu().numpy().astype(F64)


def wq(w: torch.Tensor, f32: bool = False) -> np.ndarray:
    """weights as the tensor cores see them (bf16-quantised at packing; unchanged at f32)"""
    return (w if f32 else w.to(torch.bfloat16).float()).cpu().numpy().astype(F64)


def rel(a, b) -> float:
    a, b = np.asarray(a, F64), np.asarray(b, F64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", params=["bf16", "f32"])
def seg_trace(cuda, request):
    from paper_1803_11385_b200.seg import NativeSegNet
    f, cl = shell_pair(32, 2)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(cl)
    seg = NativeSegNet(fine, coarse, c_in=8, c=32, classes=16, seed=7, lr=0.1, precision=request.param)
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.rand((fine.total_columns(), 8), device="cuda", generator=g) * 2 - 1
    if request.param == "bf16":
        x = x.to(torch.bfloat16)
    labels = torch.randint(0, 16, (fine.total_columns(),), device="cuda", generator=g)
    seg.step(x, labels)  # one real step first: BN running stats and weights move
    tr = {}
    seg.step(x, labels, trace=tr)
    torch.cuda.synchronize()
    return tr, levels_to_arrays(f), levels_to_arrays(cl), seg


def test_seg_forward_layers_vs_oracle(seg_trace, restated):
    tr, fa, ca, seg = seg_trace
    c, k = seg.c, seg.k
    f32 = seg.f32
    TOL_BF16_ = TOL_F32 if f32 else TOL_BF16  # outputs that are bf16 at precision bf16

    def wq(w):  # noqa: F811 — the precision-aware weight view
        return globals()["wq"](w, f32)
    s1, s2 = ConvSpec(3, 1, 0, 8, c), ConvSpec(3, 1, 0, c, 2 * c)
    s3, s4 = ConvSpec(3, 1, 0, 2 * c, c), ConvSpec(3, 1, 0, c, k)
    pool, dspec = ConvSpec(2, 2, 0, c, c), ConvSpec(2, 2, 0, c, 2 * c)
    w = tr["w"]
    # conv1 (fine) and conv2 (coarse): fp32 outputs
    y1 = restated.conv_forward(fa, cm(tr["x"]), fa, wq(w["conv1"]), s1, F64)
    assert rel(cm(tr["y1"]), y1) <= TOL_F32
    # max pool with switches (cnn_ops.cpp:234-284): values and switches bit-exact
    mp, msw = restated.max_pool(fa, cm(tr["r1"]), ca, pool, F64)
    assert np.array_equal(cm(tr["p1"]), mp)
    assert np.array_equal(tr["sw"].t().cpu().numpy().astype(np.int32), msw)
    y2 = restated.conv_forward(ca, cm(tr["p1"]), ca, wq(w["conv2"]), s2, F64)
    assert rel(cm(tr["y2"]), y2) <= TOL_F32
    # conv3 (bf16 output) -> max unpool through the encoder's switches (bit-exact)
    d3 = restated.conv_forward(ca, cm(tr["e2"]), ca, wq(w["conv3"]), s3, F64)
    assert rel(cm(tr["d3"]), d3) <= TOL_BF16_
    up = restated.max_unpool(cm(tr["d3"]), msw, fa, ca, pool, F64)
    assert np.array_equal(cm(tr["up"]), up)
    # stride-2 deconvolution coarse -> fine (cnn_ops.cpp:408-419): col2hash(W^T D)
    dc = restated.deconv_forward(ca, cm(tr["e2"]), fa, wq(w["deconv"]), dspec, F64)
    assert rel(cm(tr["dc"]), dc) <= TOL_F32
    # skip join (the unpooled branch accumulated into the deconvolution's output in place,
    # hc_native_max_unpool_add) -> batch norm (biased batch statistics, eps 1e-5) -> ReLU
    s3v = tr["dc"].double() + tr["up"].double()
    xh = (s3v - s3v.mean(0)) / torch.sqrt(s3v.var(0, unbiased=False) + 1e-5)
    assert rel(cm(tr["r3"].float()), cm(torch.clamp(xh, min=0).float())) <= TOL_BF16_
    sc = restated.conv_forward(fa, cm(tr["r3"]), fa, wq(w["conv4"]), s4, F64)
    assert rel(cm(tr["scores"]), sc) <= TOL_F32


def test_seg_backward_layers_vs_oracle(seg_trace, restated):
    tr, fa, ca, seg = seg_trace
    c, k = seg.c, seg.k
    f32 = seg.f32
    TOL_BF16_ = TOL_F32 if f32 else TOL_BF16
    TOL_DW_ = TOL_F32 if f32 else TOL_DW

    def wq(w):  # noqa: F811
        return globals()["wq"](w, f32)
    s2, s3, s4 = ConvSpec(3, 1, 0, c, 2 * c), ConvSpec(3, 1, 0, 2 * c, c), ConvSpec(3, 1, 0, c, k)
    s1 = ConvSpec(3, 1, 0, 8, c)
    pool, dspec = ConvSpec(2, 2, 0, c, c), ConvSpec(2, 2, 0, c, 2 * c)
    w, gr = tr["w"], tr["grads"]

    def conv_bwd(x, dy, wname, spec, s):
        cols = restated.hash2col(s, cm(x), s, spec, F64)
        return restated.conv_backward(cm(dy), wq(w[wname]), cols, s, s, spec, F64)

    # conv4: dW and the input gradient (bf16 output)
    dw4, dx4 = conv_bwd(tr["r3"], tr["dscores"], "conv4", s4, fa)
    assert rel(gr["conv4"].cpu().numpy(), dw4) <= TOL_DW_
    assert rel(cm(tr["d_r3"]), dx4) <= TOL_BF16_
    # deconvolution backward (cnn_ops.cpp:421-435): hash2col of the fine gradient + 2 GEMMs
    dwd, dxd = restated.deconv_backward(cm(tr["d_s3"]), wq(w["deconv"]), cm(tr["e2"]), ca, fa, dspec, F64)
    assert rel(gr["deconv"].cpu().numpy(), dwd) <= TOL_DW_
    assert rel(cm(tr["d_e2a"]), dxd) <= TOL_F32
    # the unpool's adjoint: each coarse cell takes the gradient of the fine voxel its switch chose
    fm = restated.field_map(fa, ca, pool)  # [n_coarse][8] fine columns (cnn_ops.cpp:100-119)
    sw = tr["sw"].cpu().numpy().astype(np.int64)
    ds3 = tr["d_s3"].float().cpu().numpy().astype(F64)
    rows = np.arange(sw.shape[0])[:, None]
    src = np.where(sw >= 0, fm[rows, np.maximum(sw, 0)], -1)
    want = np.where(src >= 0, ds3[np.maximum(src, 0), np.arange(c)[None, :]], 0.0)
    assert np.array_equal(tr["d_d3"].float().cpu().numpy().astype(F64), want)
    dw3, dx3 = conv_bwd(tr["e2"], tr["d_d3"], "conv3", s3, ca)
    assert rel(gr["conv3"].cpu().numpy(), dw3) <= TOL_DW_
    assert rel(cm(tr["d_e2b"]), dx3) <= TOL_BF16_
    dw2, dx2 = conv_bwd(tr["p1"], tr["d_y2"], "conv2", s2, ca)
    assert rel(gr["conv2"].cpu().numpy(), dw2) <= TOL_DW_
    assert rel(cm(tr["d_p1"]), dx2) <= TOL_BF16_
    # the pool's backward is the unpool through the same switches (bit-exact)
    msw = sw.T.astype(np.int32)
    assert np.array_equal(cm(tr["d_r1"]), restated.max_unpool(cm(tr["d_p1"]), msw, fa, ca, pool, F64))
    dw1, _ = conv_bwd(tr["x"], tr["d_y1"], "conv1", s1, fa)
    assert rel(gr["conv1"].cpu().numpy(), dw1) <= TOL_DW_
