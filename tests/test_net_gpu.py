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
    # accumulating form (the segmentation decoder's skip join): acc += unpooled rows, bit for bit
    # what acc.add_(unpooled) gives, with -0.0 entries in acc
    acc = torch.randn((nf, c), device="cuda")
    acc[::7] = -0.0
    want = acc + dx
    _lib.check(_lib.lib.hc_native_max_unpool_add(_p(par), _p(prow), nf, _p(dyv), _lib.HC_DTYPE_F32, c, _p(sw),
                                                 _p(acc), None))
    assert torch.equal(acc.view(torch.int32), want.view(torch.int32))


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


@pytest.mark.parametrize("x2", [False, True])
@pytest.mark.parametrize("c_in,c_out", [(8, 16), (32, 64), (64, 128)])
def test_conv_epilogue_tile_stats(cuda, x2, c_in, c_out):
    """hc_native_gather_gemm[_x2]_stats: the epilogue's per-tile {sum, centred sum of squares}
    equal float64 statistics of the same fp32 output tiles (ragged last tile excluded rows),
    and hc_native_bn_relu_forward_tiles reproduces the two-pass batch norm (cnn_ops.cpp:455-466)."""
    f, _ = random_pair(32, 3, seed=c_out + x2, n_lo=900, n_hi=2500)
    s = SuperPsh.from_levels(f)
    n = s.total_columns()
    assert n % 128 != 0
    fm = nconv.field_map_native(s, s, ConvSpec(3, 1, 0, c_in, c_out), nconv.TILED)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand((n, c_in), device="cuda", generator=g) * 2 - 1 + 0.3
    w = (torch.rand((c_out, c_in * 27), device="cuda", generator=g) * 2 - 1) * 0.2
    tiles = (n + 127) // 128
    st = torch.full((tiles, c_out, 2), float("nan"), device="cuda")
    y = torch.empty((n, c_out), device="cuda")
    if x2:
        xs = nconv.split(x)
        wp = nconv.pack_weights_x2(w, c_out, c_in, 27, nconv.PACK_FORWARD)
        _lib.check(_lib.lib.hc_native_gather_gemm_x2_stats(_p(fm.data), fm.layout, n, 27, _p(xs), c_in, _p(wp), c_out,
                                                           _p(y), _p(st), None))
        assert torch.equal(y, nconv.gather_gemm_x2(fm, xs, wp, c_out))
    else:
        xb = x.to(torch.bfloat16)
        wp = nconv.pack_weights(w, c_out, c_in, 27, False)
        _lib.check(_lib.lib.hc_native_gather_gemm_stats(_p(fm.data), fm.layout, n, 27, _p(xb), c_in, _p(wp), c_out,
                                                        _p(y), _lib.HC_DTYPE_F32, _p(st), None))
        assert torch.equal(y, nconv.gather_gemm(fm, xb, wp, c_out, torch.float32))
    yd = torch.cat([y.double(), torch.zeros((tiles * 128 - n, c_out), dtype=torch.float64, device="cuda")])
    yd = yd.view(tiles, 128, c_out)
    cnt = torch.clamp(n - torch.arange(tiles, device="cuda") * 128, max=128).double()
    mask = (torch.arange(128, device="cuda")[None, :] < cnt[:, None]).double()[:, :, None]
    s1 = (yd * mask).sum(1)
    m2 = (((yd - (s1 / cnt[:, None])[:, None, :]) ** 2) * mask).sum(1)
    assert _rel(st[..., 0].cpu().numpy(), s1.cpu().numpy()) < 1e-6
    assert _rel(st[..., 1].cpu().numpy(), m2.cpu().numpy()) < 1e-6
    # fold + apply vs the two-pass kernels
    rm1, rv1 = torch.zeros(c_out, device="cuda"), torch.ones(c_out, device="cuda")
    rm2, rv2 = rm1.clone(), rv1.clone()
    inv1, inv2 = torch.empty(c_out, device="cuda"), torch.empty(c_out, device="cuda")
    xh1, xh2 = torch.empty_like(y), torch.empty_like(y)
    o1, o2 = torch.empty_like(y), torch.empty_like(y)
    ws = torch.empty(int(_lib.lib.hc_native_bn_workspace(n, c_out)), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib.hc_native_bn_relu_forward_tiles(_p(st), n, c_out, 0.1, 1e-5, _p(rm1), _p(rv1), _p(inv1), _p(y),
                                                        _p(xh1), _p(o1), _lib.HC_DTYPE_F32, _p(ws), ws.numel(), None))
    _lib.check(_lib.lib.hc_native_bn_relu_forward_dt(_p(y), n, c_out, 1, 0.1, 1e-5, _p(rm2), _p(rv2), _p(inv2), _p(xh2),
                                                     _p(o2), _lib.HC_DTYPE_F32, _p(ws), ws.numel(), None))
    assert _rel(rm1.cpu().numpy(), rm2.cpu().numpy()) < 1e-6
    assert _rel(rv1.cpu().numpy(), rv2.cpu().numpy()) < 1e-6
    assert _rel(inv1.cpu().numpy(), inv2.cpu().numpy()) < 1e-6
    assert _rel(xh1.cpu().numpy(), xh2.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("precision", ["bf16", "f32"])
def test_net_epilogue_stats_equals_two_pass(cuda, precision):
    """The net step with batch-norm statistics from the conv epilogue gives the same loss,
    gradients and running statistics as with the separate two-pass statistics kernels."""
    from paper_1803_11385_b200.psh import PshLevel, VoxelSet, mix_seed
    levels = []
    s = VoxelSet.sphere(32, True)
    cur, li = s, 0
    while True:
        levels.append(SuperPsh.from_levels([PshLevel.build(cur, mix_seed(3, li))] * 4))
        if cur.resolution == 4:
            break
        cur = cur.coarsen()
        li += 1
    labels = torch.tensor([1, 0, 3, 2], device="cuda")
    out = []
    for epi in (True, False):
        net = nnet.NativeHashNet(5, 4, seed=3, dropout=0.0, precision=precision)
        net.epilogue_stats = epi
        nb = nnet.NetBatch.build(levels)
        gen = torch.Generator(device="cuda").manual_seed(1)
        feats = torch.rand((3, levels[0].total_columns()), device="cuda", generator=gen)
        x = net.input_features(feats)
        loss, grads, fc = net.loss_and_gradients(nb, x, labels)
        out.append((float(loss), [g.clone() for g in grads], [b["run_mean"].clone() for b in net.blocks],
                    [b["run_var"].clone() for b in net.blocks]))
    (l1, g1, m1, v1), (l2, g2, m2, v2) = out
    tol = 1e-5 if precision == "f32" else 1e-3
    assert abs(l1 - l2) <= tol * abs(l2)
    for a, b in zip(g1, g2):
        assert _rel(a.cpu().numpy(), b.cpu().numpy()) < tol
    for a, b in zip(m1 + v1, m2 + v2):
        assert _rel(a.cpu().numpy(), b.cpu().numpy()) < 1e-5


def test_native_net_step_f32_matches_reference_net_cfg2(cuda, ref):
    """BASELINE config 2 size (64^3 shells x 32, 5 conv/pool levels, 40 classes): one fp32 training
    step of the native net against the unmodified fp32 reference net on the same tables, weights
    and labels. The reference itself sums in fp32 over up to ~450 k voxels per weight gradient,
    so the bars are loss 1e-5, gradients 1e-4 normwise, running statistics 1e-5 (measured on a B200:
    loss 1.3e-6, gradients <= 2.5e-5, statistics <= 4e-6)."""
    level_max, classes, b = 6, 40, 32
    s = ref.sphere_set(64, True)
    levels, cur = [], s
    while True:
        levels.append(ref.build_psh(cur, 0))
        if cur.resolution == 4:
            break
        cur = ref.coarsen(cur)
    supers = [ref.build_super([lv] * b) for lv in levels]
    labels = (np.arange(b, dtype=np.int32) * 7) % classes
    rn = ref.net_make(level_max, classes, 5)
    rn.set_dropout(0.0)
    head_in = nnet.channels_at_level(2) * 8
    net = nnet.NativeHashNet(level_max, classes, seed=1, dropout=0.0, precision="f32")
    for i in range(rn.nblocks):
        net.set_reference_weights(i, torch.from_numpy(rn.conv(i)).cuda())
    for dst, src in zip((net.fc1_w, net.fc1_b, net.fc2_w, net.fc2_b), rn.fc(classes, head_in)):
        dst.copy_(torch.from_numpy(src))
    loss_r, grads_r, fc_r = rn.loss_and_gradients(supers, labels, classes, head_in)
    nb = nnet.NetBatch.build([SuperPsh.from_host(sp) for sp in supers])
    x = net.input_features(torch.from_numpy(supers[0].data).cuda())
    loss_n, grads_n, fc_n = net.loss_and_gradients(nb, x, torch.from_numpy(labels).long().cuda())
    errs = {"loss": abs(float(loss_n) - loss_r) / abs(loss_r)}
    for i, gr in enumerate(grads_r):
        blk = net.blocks[i]
        gn = grads_n[i].view(blk["cout_p"], blk["cin_p"], 27)[:blk["cout"], :blk["cin"]].reshape(gr.shape)
        errs[f"dw{i}"] = _rel(gn.cpu().numpy(), gr)
        m_r, v_r = rn.bn(i)
        errs[f"mean{i}"] = _rel(blk["run_mean"][:blk["cout"]].cpu().numpy(), m_r)
        errs[f"var{i}"] = _rel(blk["run_var"][:blk["cout"]].cpu().numpy(), v_r)
    for k, (a, r) in enumerate(zip(fc_n, fc_r)):
        errs[f"fc{k}"] = _rel(a.cpu().numpy(), r)
    print(errs)
    assert errs["loss"] < 1e-5, errs
    assert all(v < 1e-4 for k, v in errs.items() if k.startswith(("dw", "fc"))), errs
    assert all(v < 1e-5 for k, v in errs.items() if k.startswith(("mean", "var"))), errs


def test_multi_tensor_sgd_bit_exact(cuda):
    """hc_native_sgd_update_multi (one launch for many tensors) applies net.cpp:339-346's update
    v = momentum*v + lr*(g + wd*w); w -= v with separate fp32 roundings to every tensor, bit for
    bit the per-element numpy float32 restatement (sizes straddle the 256-thread blocks)."""
    rng = np.random.default_rng(0)
    sizes = [1, 255, 256, 257, 5000, 70001]
    ws = [rng.standard_normal(n).astype(np.float32) for n in sizes]
    vs = [rng.standard_normal(n).astype(np.float32) for n in sizes]
    gs = [rng.standard_normal(n).astype(np.float32) for n in sizes]
    lr, mom, wd = np.float32(0.1), np.float32(0.9), np.float32(5e-4)
    tw = [torch.from_numpy(a.copy()).cuda() for a in ws]
    tv = [torch.from_numpy(a.copy()).cuda() for a in vs]
    tg = [torch.from_numpy(a.copy()).cuda() for a in gs]
    k = len(sizes)
    arr = lambda ts: (C.c_void_p * k)(*[t.data_ptr() for t in ts])  # noqa: E731
    _lib.check(_lib.lib.hc_native_sgd_update_multi(arr(tw), arr(tv), arr(tg), (C.c_int64 * k)(*sizes), k,
                                                   float(lr), float(mom), float(wd), None))
    for w, v, g, dw, dv in zip(ws, vs, gs, tw, tv):
        v_new = (mom * v) + (lr * (g + (wd * w)))
        w_new = w - v_new
        assert np.array_equal(dv.cpu().numpy(), v_new) and np.array_equal(dw.cpu().numpy(), w_new)


@pytest.mark.parametrize("classes,b,denom", [(40, 32, 32), (7, 100, 400), (256, 3, 3)])
def test_softmax_xent_matches_double_reference(cuda, classes, b, denom):
    """hc_native_softmax_xent (net.cpp:260-283): loss and scores gradient equal a float64
    log-softmax to 1e-12 / fp32 rounding, for column counts above and below a warp's 32."""
    from paper_1803_11385_b200 import _lib
    from paper_1803_11385_b200._lib import check, lib
    g = torch.Generator(device="cuda").manual_seed(classes + b)
    scores = (torch.randn((classes, b), device="cuda", generator=g) * 8).contiguous()
    labels = torch.randint(0, classes, (b,), device="cuda", generator=g)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    d = torch.empty_like(scores)
    s = torch.cuda.current_stream().cuda_stream
    import ctypes
    check(lib.hc_native_softmax_xent(ctypes.c_void_p(scores.data_ptr()), classes, b,
                                     ctypes.c_void_p(labels.data_ptr()), denom, ctypes.c_void_p(loss.data_ptr()),
                                     ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(s)))
    logp = torch.log_softmax(scores.double().t(), dim=1)
    rows = torch.arange(b, device="cuda")
    want = -logp[rows, labels].sum() / denom
    assert abs(float(loss[0]) - float(want)) <= 1e-12 * max(1.0, abs(float(want)))
    dw = logp.exp()
    dw[rows, labels] -= 1.0
    assert torch.allclose(d.double(), (dw.t() / denom), rtol=0, atol=1e-7 / denom + 1e-12)


def test_dropout_apply_equals_torch_composition(cuda):
    """hc_native_dropout_apply == ((u < keep).float() / keep, x * mask) bit for bit."""
    import ctypes
    from paper_1803_11385_b200._lib import check, lib
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((1000, 32), device="cuda", generator=g)
    u = torch.rand(x.shape, device="cuda", generator=g)
    for keep in (0.5, 0.8, 1.0):
        m, o = torch.empty_like(x), torch.empty_like(x)
        p = lambda t: ctypes.c_void_p(t.data_ptr())
        check(lib.hc_native_dropout_apply(p(u), p(x), x.numel(), keep, p(m), p(o),
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        want_m = (u < keep).float() / keep
        assert torch.equal(m, want_m) and torch.equal(o, x * want_m)
