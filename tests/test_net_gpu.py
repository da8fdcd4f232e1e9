"""Native net layers (csrc/net_ops.cu) and the native classification net (net.py) against
the oracle and the unmodified reference net (oracle/_ref, net.cpp:260-323).

Bars: pooling / unpooling / switches / dense pool are copies and compares -> bit-exact
against the reference-layout oracle on identical fp32 inputs. Batch norm + ReLU against a
float64 restatement of cnn_ops.cpp:437-489 (<= 1e-6 relative). The whole net step uses
bf16 conv operands (tcgen05), so it is compared to the fp32 reference net within a stated
bf16 tolerance (loss 2e-2 relative, every conv weight gradient 8e-2 normwise)."""
import numpy as np
import pytest
import torch

from helpers import random_pair, levels_to_arrays

pytestmark = pytest.mark.gpu

from oracle.oracle import mix_seed  # noqa: E402
from paper_1803_11385_b200 import _lib  # noqa: E402
from paper_1803_11385_b200 import conv as nconv  # noqa: E402
from paper_1803_11385_b200 import net as nnet  # noqa: E402
from paper_1803_11385_b200.ops import ConvSpec, field_map  # noqa: E402
from paper_1803_11385_b200.psh import SuperPsh  # noqa: E402

import ctypes as C  # noqa: E402


def _p(t):
    return C.c_void_p(t.data_ptr())


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("c", [8, 16, 64])
def test_native_max_pool_unpool_bit_exact(cuda, restated, c):
    f, cl = random_pair(16, 3, seed=c, n_lo=300, n_hi=900)
    fa, ca = levels_to_arrays(f), levels_to_arrays(cl)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(cl)
    nf, nc = fine.total_columns(), coarse.total_columns()
    rng = np.random.default_rng(c)
    x = rng.integers(-3, 4, (c, nf)).astype(np.float32)  # few distinct values: many ties
    spec = ConvSpec(2, 2, 0, c, c)
    om, osw = restated.max_pool(fa, x, ca, spec)
    pm = field_map(fine, coarse, spec)
    xv = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    y = torch.empty((nc, c), device="cuda")
    sw = torch.empty((nc, c), dtype=torch.int8, device="cuda")
    _lib.check(_lib.lib.hc_native_max_pool(_p(pm), nc, 8, _p(xv), _lib.HC_DTYPE_F32, c, _p(y), _p(sw), None))
    assert np.array_equal(y.cpu().numpy().T, om)
    assert np.array_equal(sw.cpu().numpy().T.astype(np.int32), osw)
    # unpool: the reference's covering-output pull on the same switches
    dy = rng.uniform(-1, 1, (c, nc)).astype(np.float32)
    ou = restated.max_unpool(dy, osw, fa, ca, spec)
    par = torch.empty(nf, dtype=torch.int32, device="cuda")
    prow = torch.empty(nf, dtype=torch.int8, device="cuda")
    _lib.check(_lib.lib.hc_native_pool_parents(_p(pm), nc, 8, nf, _p(par), _p(prow), None))
    dyv = torch.from_numpy(np.ascontiguousarray(dy.T)).cuda()
    dx = torch.empty((nf, c), device="cuda")
    _lib.check(_lib.lib.hc_native_max_unpool(_p(par), _p(prow), nf, _p(dyv), _lib.HC_DTYPE_F32, c, _p(sw), _p(dx),
                                             None))
    assert np.array_equal(dx.cpu().numpy().T, ou)


def test_native_bn_relu_forward_backward(cuda):
    n, c = 70001, 32
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((n, c), device="cuda", generator=g) * 3 + 1
    rm, rv = torch.zeros(c, device="cuda"), torch.ones(c, device="cuda")
    inv = torch.empty(c, device="cuda")
    xhat = torch.empty_like(x)
    out = torch.empty((n, c), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(int(_lib.lib.hc_native_bn_workspace(n, c)), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib.hc_native_bn_relu_forward(_p(x), n, c, 1, 0.1, 1e-5, _p(rm), _p(rv), _p(inv), _p(xhat),
                                                  _p(out), _p(ws), ws.numel(), None))
    xd = x.double().cpu().numpy()
    mean, var = xd.mean(0), ((xd - xd.mean(0)) ** 2).mean(0)
    istd = 1.0 / np.sqrt(var + 1e-5)
    assert _rel(inv.cpu().numpy(), istd) < 1e-6
    assert _rel(xhat.cpu().numpy(), (xd - mean) * istd) < 1e-6
    assert _rel(rm.cpu().numpy(), 0.1 * mean) < 1e-6 and _rel(rv.cpu().numpy(), 0.9 + 0.1 * var) < 1e-6
    assert torch.equal(out, torch.relu(xhat).to(torch.bfloat16))
    # backward: cnn_ops.cpp:476-489 after relu_backward
    dr = torch.randn((n, c), device="cuda", generator=g)
    dconv = torch.empty((n, c), dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.lib.hc_native_bn_relu_backward(_p(dr), _lib.HC_DTYPE_F32, _p(xhat), _p(inv), n, c, _p(dconv),
                                                   _p(ws), ws.numel(), None))
    h = xhat.double().cpu().numpy()
    gd = np.where(h > 0, dr.double().cpu().numpy(), 0.0)
    want = inv.double().cpu().numpy() * (gd - gd.mean(0) - h * (gd * h).mean(0))
    assert _rel(dconv.float().cpu().numpy(), want) < 4e-3  # bf16 output rounding


def _ref_pyramid_batch(ref, nmodels, res, seed):
    pyr = []
    for k in range(nmodels):
        s = ref.random_set(res, 220 + 60 * k, mix_seed(seed, k))
        levels, cur, li = [], s, 0
        while True:
            levels.append(ref.build_psh(cur, mix_seed(seed + 100 + k, li)))
            if cur.resolution == 4:
                break
            cur = ref.coarsen(cur)
            li += 1
        pyr.append(levels)
    return [ref.build_super([p[lv] for p in pyr]) for lv in range(len(pyr[0]))]


def test_native_net_step_matches_reference_net(cuda, ref):
    level_max, classes, b = 4, 5, 3
    supers = _ref_pyramid_batch(ref, b, 1 << level_max, seed=11)
    labels = np.array([0, 3, 1], np.int32)
    rn = ref.net_make(level_max, classes, 7)
    rn.set_dropout(0.0)
    head_in = nnet.channels_at_level(2) * 8
    net = nnet.NativeHashNet(level_max, classes, seed=1, dropout=0.0)
    for i in range(rn.nblocks):
        net.set_reference_weights(i, torch.from_numpy(rn.conv(i)).cuda())
    for dst, src in zip((net.fc1_w, net.fc1_b, net.fc2_w, net.fc2_b), rn.fc(classes, head_in)):
        dst.copy_(torch.from_numpy(src))
    loss_r, grads_r, fc_r = rn.loss_and_gradients(supers, labels, classes, head_in)

    nb = nnet.NetBatch.build([SuperPsh.from_host(s) for s in supers])
    x = net.input_features(torch.from_numpy(supers[0].data).cuda())
    loss_n, grads_n, fc_n = net.loss_and_gradients(nb, x, torch.from_numpy(labels).long().cuda())
    assert abs(float(loss_n) - loss_r) / abs(loss_r) < 2e-2, (float(loss_n), loss_r)
    for i, gr in enumerate(grads_r):
        blk = net.blocks[i]
        gn = grads_n[i].view(blk["cout_p"], blk["cin_p"], 27)[:blk["cout"], :blk["cin"]].reshape(gr.shape)
        assert _rel(gn.cpu().numpy(), gr) < 8e-2, (i, _rel(gn.cpu().numpy(), gr))
        # padded rows / columns of the gradient stay exactly zero
        full = grads_n[i].view(blk["cout_p"], blk["cin_p"], 27)
        assert float(full[blk["cout"]:].abs().sum()) == 0.0 and float(full[:, blk["cin"]:].abs().sum()) == 0.0
        m_r, v_r = rn.bn(i)
        assert _rel(blk["run_mean"][:blk["cout"]].cpu().numpy(), m_r) < 5e-2
        assert _rel(blk["run_var"][:blk["cout"]].cpu().numpy(), v_r) < 5e-2
    for a, r in zip(fc_n, fc_r):
        assert _rel(a.cpu().numpy(), r) < 8e-2


def test_native_net_inference_matches_reference_net(cuda, ref):
    """net_forward with training = false (net.cpp:203-208, 232-241): running statistics
    normalise, dropout is off. The reference's running stats (after one training pass) are
    loaded into the native net, so the comparison isolates the inference path (bf16 conv
    operands: scores within 2e-2 normwise)."""
    level_max, classes, b = 4, 5, 3
    supers = _ref_pyramid_batch(ref, b, 1 << level_max, seed=13)
    labels = np.array([1, 4, 0], np.int32)
    rn = ref.net_make(level_max, classes, 9)
    rn.set_dropout(0.0)
    head_in = nnet.channels_at_level(2) * 8
    net = nnet.NativeHashNet(level_max, classes, seed=1, dropout=0.0)
    for i in range(rn.nblocks):
        net.set_reference_weights(i, torch.from_numpy(rn.conv(i)).cuda())
    for dst, src in zip((net.fc1_w, net.fc1_b, net.fc2_w, net.fc2_b), rn.fc(classes, head_in)):
        dst.copy_(torch.from_numpy(src))
    rn.loss_and_gradients(supers, labels, classes, head_in)  # training pass: running stats move
    for i in range(rn.nblocks):
        m_r, v_r = rn.bn(i)
        blk = net.blocks[i]
        assert np.abs(v_r - 1.0).max() > 1e-3  # the stats are not at their initial values
        blk["run_mean"][:blk["cout"]] = torch.from_numpy(m_r).cuda()
        blk["run_var"][:blk["cout"]] = torch.from_numpy(v_r).cuda()
    want = rn.forward(supers, classes)
    nb = nnet.NetBatch.build([SuperPsh.from_host(s) for s in supers])
    x = net.input_features(torch.from_numpy(supers[0].data).cuda())
    before = [blk["run_mean"].clone() for blk in net.blocks]
    got = net.forward(nb, x, training=False)
    assert _rel(got.cpu().numpy(), want) < 2e-2, _rel(got.cpu().numpy(), want)
    assert all(torch.equal(a, blk["run_mean"]) for a, blk in zip(before, net.blocks))  # inference: stats untouched
    assert net.predict(nb, x).shape == (b,)


def test_native_net_train_step_descends(cuda, ref):
    supers = _ref_pyramid_batch(ref, 4, 16, seed=5)
    net = nnet.NativeHashNet(4, 4, seed=2, dropout=0.0, lr=0.01)  # batch 4: lr 0.05 oscillates
    nb = nnet.NetBatch.build([SuperPsh.from_host(s) for s in supers])
    x = net.input_features(torch.from_numpy(supers[0].data).cuda())
    labels = torch.tensor([0, 1, 2, 3], device="cuda")
    losses = [float(net.train_step(nb, x, labels)) for _ in range(12)]
    assert all(np.isfinite(losses)) and max(losses[-3:]) < 0.5 * losses[0], losses


def test_graphed_step_matches_eager(cuda, ref):
    """The CUDA-graph step replays exactly the eager step's kernels (deterministic): same
    losses step for step (the graph's 2 warm-up steps are real training steps)."""
    supers = _ref_pyramid_batch(ref, 3, 16, seed=9)
    labels = torch.tensor([2, 0, 1], device="cuda")

    def fresh():
        net = nnet.NativeHashNet(4, 3, seed=4, dropout=0.0, lr=0.01)
        levels = [SuperPsh.from_host(s) for s in supers]
        x = net.input_features(torch.from_numpy(supers[0].data).cuda())
        return net, levels, x

    net_e, lev_e, x_e = fresh()
    eager = [float(net_e.train_step(nnet.NetBatch.build(lev_e), x_e, labels)) for _ in range(5)]
    net_g, lev_g, x_g = fresh()
    step = nnet.GraphedStep(net_g, lev_g, x_g, labels, warmup=2)
    graphed = [float(step()) for _ in range(3)]
    assert graphed == eager[2:], (graphed, eager)


def test_native_seg_step_descends(cuda):
    """Segmentation-style composition (conv/BN/ReLU/pool -> conv -> unpool + deconv -> conv,
    per-voxel softmax) trains on a 32^3 shell pair: the loss falls under SGD."""
    from helpers import shell_pair
    from paper_1803_11385_b200.seg import NativeSegNet
    f, cl = shell_pair(32, 2)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(cl)
    seg = NativeSegNet(fine, coarse, c_in=8, c=32, classes=16, seed=3, lr=0.5)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = (torch.rand((fine.total_columns(), 8), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    labels = (x[:, 0].float() > 0).long() + 2 * (x[:, 1].float() > 0).long()  # learnable from the input
    losses = [float(seg.step(x, labels)) for _ in range(15)]
    assert all(np.isfinite(losses)) and losses[-1] < 0.8 * losses[0], losses


def test_native_net_step_f32_matches_reference_net(cuda, ref):
    """precision="f32": fp32 activations, every conv through the split-precision tcgen05 kernels.
    The same step as above against the unmodified fp32 reference net, now at the reference's
    precision: loss 1e-6 relative, conv / FC weight gradients 5e-5 normwise, running statistics
    1e-5 (the remaining differences are the reference's own fp32 summation order)."""
    level_max, classes, b = 4, 5, 3
    supers = _ref_pyramid_batch(ref, b, 1 << level_max, seed=11)
    labels = np.array([0, 3, 1], np.int32)
    rn = ref.net_make(level_max, classes, 7)
    rn.set_dropout(0.0)
    head_in = nnet.channels_at_level(2) * 8
    net = nnet.NativeHashNet(level_max, classes, seed=1, dropout=0.0, precision="f32")
    for i in range(rn.nblocks):
        net.set_reference_weights(i, torch.from_numpy(rn.conv(i)).cuda())
    for dst, src in zip((net.fc1_w, net.fc1_b, net.fc2_w, net.fc2_b), rn.fc(classes, head_in)):
        dst.copy_(torch.from_numpy(src))
    loss_r, grads_r, fc_r = rn.loss_and_gradients(supers, labels, classes, head_in)

    nb = nnet.NetBatch.build([SuperPsh.from_host(s) for s in supers])
    x = net.input_features(torch.from_numpy(supers[0].data).cuda())
    assert x.dtype == torch.float32
    loss_n, grads_n, fc_n = net.loss_and_gradients(nb, x, torch.from_numpy(labels).long().cuda())
    errs = {"loss": abs(float(loss_n) - loss_r) / abs(loss_r)}
    for i, gr in enumerate(grads_r):
        blk = net.blocks[i]
        gn = grads_n[i].view(blk["cout_p"], blk["cin_p"], 27)[:blk["cout"], :blk["cin"]].reshape(gr.shape)
        errs[f"dw{i}"] = _rel(gn.cpu().numpy(), gr)
        full = grads_n[i].view(blk["cout_p"], blk["cin_p"], 27)
        assert float(full[blk["cout"]:].abs().sum()) == 0.0 and float(full[:, blk["cin"]:].abs().sum()) == 0.0
        m_r, v_r = rn.bn(i)
        errs[f"mean{i}"] = _rel(blk["run_mean"][:blk["cout"]].cpu().numpy(), m_r)
        errs[f"var{i}"] = _rel(blk["run_var"][:blk["cout"]].cpu().numpy(), v_r)
    for k, (a, r) in enumerate(zip(fc_n, fc_r)):
        errs[f"fc{k}"] = _rel(a.cpu().numpy(), r)
    print(errs)
    assert errs["loss"] < 1e-6, errs  # measured 1.0e-7
    assert all(v < 5e-5 for k, v in errs.items() if k.startswith(("dw", "fc"))), errs  # measured <= 1.0e-5
    assert all(v < 1e-5 for k, v in errs.items() if k.startswith(("mean", "var"))), errs  # measured <= 3.1e-6
