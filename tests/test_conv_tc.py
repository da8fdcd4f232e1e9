"""Native tcgen05 implicit-GEMM conv: forward (gather-GEMM), weight gradient (MN-major
split-K) and stride-1 input gradient (flipped kernel) against float64 references.

Tolerance contract (SURVEY.md §8c, bf16 path): operands are quantised to bf16
identically on both sides, the reference accumulates in float64, the GPU in fp32 ->
||gpu - ref||_F / ||ref||_F <= 1e-5 (fp32 outputs). The bf16 quantisation error
itself is reported separately against the unquantised fp32 oracle (<= 1e-2)."""
import numpy as np
import pytest
import torch

from helpers import levels_to_arrays, random_pair, shell_pair

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200 import conv as nconv  # noqa: E402
from paper_1803_11385_b200 import ops  # noqa: E402
from paper_1803_11385_b200.ops import ConvSpec  # noqa: E402
from paper_1803_11385_b200.psh import SuperPsh  # noqa: E402

TOL_F32_OUT = 1e-5
TOL_DW = 5e-5


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-300))


def ref_gather_gemm(fmap, x, w_ref, c_out):
    """Y[n,co] = sum_t sum_ci X[fmap[n,t],ci] W[co, ci*taps + t]   (float64)"""
    n, taps = fmap.shape
    c_in = x.shape[1]
    xd = torch.cat([x.double(), torch.zeros((1, c_in), dtype=torch.float64, device=x.device)])
    idx = torch.where(fmap >= 0, fmap.long(), torch.full_like(fmap.long(), x.shape[0]))
    g = xd[idx]  # n, taps, c_in
    w = w_ref.double().view(c_out, c_in, taps)  # co, ci, t
    return torch.einsum("ntc,oct->no", g, w)


def ref_dw(fmap, x, dy):
    n, taps = fmap.shape
    c_in = x.shape[1]
    xd = torch.cat([x.double(), torch.zeros((1, c_in), dtype=torch.float64, device=x.device)])
    idx = torch.where(fmap >= 0, fmap.long(), torch.full_like(fmap.long(), x.shape[0]))
    g = xd[idx]
    return torch.einsum("no,ntc->oct", dy.double(), g).reshape(dy.shape[1], c_in * taps)


def layouts(fmap):
    """The same row-major map in the tap-major and tile-major layouts."""
    n, taps = fmap.shape
    pad = (n + 127) // 128 * 128
    tiled = torch.full((pad, taps), -1, dtype=torch.int32, device=fmap.device)
    tiled[:n] = fmap
    return [nconv.FieldMap(fmap.t().contiguous(), n, taps, nconv.TAP_MAJOR),
            nconv.FieldMap(tiled.view(pad // 128, 128, taps).permute(0, 2, 1).contiguous(), n, taps, nconv.TILED)]


def bf16_round(t):
    return t.to(torch.bfloat16).float()


@pytest.mark.parametrize("c_in,c_out", [(8, 16), (16, 16), (16, 32), (32, 64), (64, 64), (64, 128), (128, 256),
                                        (24, 48), (8, 256), (256, 16)])
@pytest.mark.parametrize("n", [1000, 5003])
def test_gather_gemm_random_maps(cuda, c_in, c_out, n):
    if c_out not in (16, 32, 64, 128, 256):
        pytest.skip("c_out outside the tcgen05 tile set")
    g = torch.Generator(device="cuda").manual_seed(c_in * 1000 + c_out + n)
    n_in = n + 37
    x = bf16_round(torch.rand((n_in, c_in), device="cuda", generator=g) * 2 - 1)
    w = bf16_round(torch.rand((c_out, c_in * 27), device="cuda", generator=g) * 2 - 1)
    fmap = torch.randint(-1, n_in, (n, 27), device="cuda", generator=g, dtype=torch.int32)
    fmap[torch.rand((n, 27), device="cuda", generator=g) < 0.4] = -1
    wp = nconv.pack_weights(w, c_out, c_in, 27, False)
    y = nconv.gather_gemm(fmap, x.to(torch.bfloat16), wp, c_out, torch.float32)
    yr = ref_gather_gemm(fmap, x, w, c_out)
    assert rel(y, yr) <= TOL_F32_OUT
    yb = nconv.gather_gemm(fmap, x.to(torch.bfloat16), wp, c_out, torch.bfloat16)
    assert rel(yb.float(), yr) <= 4e-3
    for fm in layouts(fmap):
        assert torch.equal(nconv.gather_gemm(fm, x.to(torch.bfloat16), wp, c_out, torch.float32), y), fm.layout


@pytest.mark.parametrize("c_in,c_out", [(8, 16), (16, 16), (16, 64), (64, 64), (64, 128), (32, 256), (128, 32),
                                        (320, 256)])
def test_dw_random_maps(cuda, c_in, c_out):
    """(320, 256): 68 m-tiles at 2 per CTA's TMEM -> 34 groups (a plan clamped to 32 groups would
    give groups 3 m-tiles and overrun the 512-column allocation)."""
    g = torch.Generator(device="cuda").manual_seed(7 * c_in + c_out)
    n, n_in = 20011, 19000
    x = bf16_round(torch.rand((n_in, c_in), device="cuda", generator=g) * 2 - 1)
    dy = bf16_round(torch.rand((n, c_out), device="cuda", generator=g) * 2 - 1)
    fmap = torch.randint(-1, n_in, (n, 27), device="cuda", generator=g, dtype=torch.int32)
    dw = nconv.conv_dw(fmap, x.to(torch.bfloat16), dy.to(torch.bfloat16))
    assert rel(dw, ref_dw(fmap, x, dy)) <= TOL_DW
    dw2 = nconv.conv_dw(fmap, x.to(torch.bfloat16), dy.to(torch.bfloat16))
    assert torch.equal(dw, dw2), "dW must be deterministic"
    for fm in layouts(fmap):
        assert torch.equal(nconv.conv_dw(fm, x.to(torch.bfloat16), dy.to(torch.bfloat16)), dw), fm.layout


@pytest.mark.parametrize("c_in,c_out", [(16, 16), (32, 64), (64, 64), (3, 2), (24, 48), (100, 70)])
def test_layer_vs_oracle_on_shell(cuda, restated, c_in, c_out):
    """Whole layer (forward, dW, dX) on a 64^3 shell batch vs the double oracle
    (oracle/hc_oracle.c conv_forward / conv_backward) on bf16-quantised operands; channel
    counts outside the tensor-core tile set (the paper's 3 -> 2, 24 -> 48, 100 -> 70) are
    zero-padded inside the layer."""
    f, _ = shell_pair(64, 2)
    fa = levels_to_arrays(f)
    s = SuperPsh.from_levels(f)
    N = s.total_columns()
    rng = np.random.default_rng(c_in + c_out)
    q = lambda a: torch.from_numpy(a).to(torch.bfloat16).float().numpy()  # noqa: E731
    x = q(rng.uniform(-1, 1, (c_in, N)).astype(np.float32))
    w = q(rng.uniform(-1, 1, (c_out, c_in * 27)).astype(np.float32))
    dy = q(rng.uniform(-1, 1, (c_out, N)).astype(np.float32))
    spec = ConvSpec(3, 1, 0, c_in, c_out)
    f64 = np.float64
    cols64 = restated.hash2col(fa, x.astype(f64), fa, spec, f64)
    y64 = restated.matmul(w.astype(f64), cols64, f64)
    dw64, dx64 = restated.conv_backward(dy.astype(f64), w.astype(f64), cols64, fa, fa, spec, f64)

    layer = nconv.HashConv(s, torch.from_numpy(w).cuda(), spec, out_dtype=torch.float32)
    xv = nconv.to_voxel_major(torch.from_numpy(x).cuda())
    dyv = nconv.to_voxel_major(torch.from_numpy(dy).cuda())
    y = nconv.to_channel_major(layer.forward(xv))
    dw, dxv = layer.backward(dyv, xv, torch.float32)
    dx = nconv.to_channel_major(dxv)
    t = lambda a: torch.from_numpy(a)  # noqa: E731
    assert rel(y.cpu(), t(y64)) <= TOL_F32_OUT
    assert rel(dw.cpu(), t(dw64)) <= TOL_DW
    assert rel(dx.cpu(), t(dx64)) <= TOL_F32_OUT
    # fmap used by the layer equals the reference-layout K0 map and the oracle's
    want = restated.field_map(fa, fa, spec)
    tiled = layer.fmap.data.permute(0, 2, 1).reshape(-1, 27)[:N].cpu().numpy().astype(np.int64)
    assert np.array_equal(tiled, want)
    assert (layer.fmap.data.permute(0, 2, 1).reshape(-1, 27)[N:] == -1).all()
    tap = nconv.field_map_native(s, s, spec, nconv.TAP_MAJOR)
    assert np.array_equal(tap.data.t().cpu().numpy().astype(np.int64), want)


def test_quantisation_error_reported(cuda, restated):
    """bf16 quantisation error of the native path vs the unquantised fp32 oracle."""
    f, _ = random_pair(16, 2, seed=11, n_lo=300, n_hi=800)
    fa = levels_to_arrays(f)
    s = SuperPsh.from_levels(f)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (16, s.total_columns())).astype(np.float32)
    w = rng.uniform(-1, 1, (32, 16 * 27)).astype(np.float32)
    spec = ConvSpec(3, 1, 0, 16, 32)
    y64 = restated.matmul(w.astype(np.float64), restated.hash2col(fa, x.astype(np.float64), fa, spec, np.float64),
                          np.float64)
    layer = nconv.HashConv(s, torch.from_numpy(w).cuda(), spec, out_dtype=torch.float32)
    y = nconv.to_channel_major(layer.forward(nconv.to_voxel_major(torch.from_numpy(x).cuda())))
    err = rel(y.cpu(), torch.from_numpy(y64))
    assert err <= 1e-2, err


def test_layout_round_trip(cuda):
    x = torch.rand((37, 1001), device="cuda")
    v = nconv.to_voxel_major(x)
    assert v.shape == (1001, 37) and v.dtype == torch.bfloat16
    back = nconv.to_channel_major(v)
    assert torch.equal(back, x.to(torch.bfloat16).float())
    assert torch.equal(nconv.to_channel_major(x.t().contiguous()), x)


@pytest.mark.parametrize("c_in,c_out", [(16, 16), (32, 64), (64, 32)])
def test_native_deconv_vs_oracle(cuda, restated, c_in, c_out):
    """Native deconvolution (transposed field map + W^T gather-GEMM; backward on the conv's
    own map) vs the double oracle deconv_forward / deconv_backward (cnn_ops.cpp:408-435) on
    bf16-quantised operands, coarsening spec {2,2,0}."""
    f, cl = shell_pair(32, 2)
    fa, ca = levels_to_arrays(f), levels_to_arrays(cl)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(cl)
    nf, nc = fine.total_columns(), coarse.total_columns()
    rng = np.random.default_rng(c_in * 7 + c_out)
    q = lambda a: torch.from_numpy(a).to(torch.bfloat16).float().numpy()  # noqa: E731
    spec = ConvSpec(2, 2, 0, c_in, c_out)
    w = q(rng.uniform(-1, 1, (c_out, c_in * 8)).astype(np.float32))
    dc = q(rng.uniform(-1, 1, (c_out, nc)).astype(np.float32))
    fg = q(rng.uniform(-1, 1, (c_in, nf)).astype(np.float32))
    f64 = np.float64
    y64 = restated.deconv_forward(ca, dc.astype(f64), fa, w.astype(f64), spec, f64)
    dw64, dd64 = restated.deconv_backward(fg.astype(f64), w.astype(f64), dc.astype(f64), ca, fa, spec, f64)
    layer = nconv.HashDeconv(coarse, fine, torch.from_numpy(w).cuda(), spec, out_dtype=torch.float32)
    dcv = nconv.to_voxel_major(torch.from_numpy(dc).cuda())
    y = nconv.to_channel_major(layer.forward(dcv))
    dw, ddv = layer.backward(nconv.to_voxel_major(torch.from_numpy(fg).cuda()), dcv, torch.float32)
    t = lambda a: torch.from_numpy(a)  # noqa: E731
    assert rel(y.cpu(), t(y64)) <= TOL_F32_OUT
    assert rel(dw.cpu(), t(dw64)) <= TOL_DW
    assert rel(nconv.to_channel_major(ddv).cpu(), t(dd64)) <= TOL_F32_OUT


@pytest.mark.parametrize("n", [1, 127, 128, 129])
def test_native_tiny_and_ragged_batches(cuda, n):
    """Single voxel, one partial tile, exactly one tile, one voxel past a tile: forward, dW and
    dX match float64 (the tile-major map pads with -1; dW partials of idle splits are zero)."""
    g = torch.Generator(device="cuda").manual_seed(n)
    c_in, c_out, n_in = 16, 32, n + 5
    x = bf16_round(torch.rand((n_in, c_in), device="cuda", generator=g) * 2 - 1)
    dy = bf16_round(torch.rand((n, c_out), device="cuda", generator=g) * 2 - 1)
    w = bf16_round(torch.rand((c_out, c_in * 27), device="cuda", generator=g) * 2 - 1)
    fmap = torch.randint(-1, n_in, (n, 27), device="cuda", generator=g, dtype=torch.int32)
    wp = nconv.pack_weights(w, c_out, c_in, 27, False)
    assert rel(nconv.gather_gemm(fmap, x.to(torch.bfloat16), wp, c_out, torch.float32),
               ref_gather_gemm(fmap, x, w, c_out)) <= TOL_F32_OUT
    assert rel(nconv.conv_dw(fmap, x.to(torch.bfloat16), dy.to(torch.bfloat16)), ref_dw(fmap, x, dy)) <= TOL_DW


def test_native_empty_batch(cuda):
    x = torch.zeros((4, 16), dtype=torch.bfloat16, device="cuda")
    fmap = torch.zeros((0, 27), dtype=torch.int32, device="cuda")
    wp = nconv.pack_weights(torch.zeros((32, 16 * 27), device="cuda"), 32, 16, 27, False)
    assert nconv.gather_gemm(fmap, x, wp, 32).shape == (0, 32)
    dw = nconv.conv_dw(fmap, x, torch.zeros((0, 32), dtype=torch.bfloat16, device="cuda"))
    assert dw.shape == (32, 16 * 27) and float(dw.abs().sum()) == 0.0


def test_native_argument_errors(cuda):
    x = torch.zeros((4, 12), dtype=torch.bfloat16, device="cuda")  # C_in not a multiple of 8
    fmap = torch.zeros((4, 27), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match="multiple of 8"):
        nconv.gather_gemm(fmap, x, torch.zeros((16, 384), dtype=torch.bfloat16, device="cuda"), 16)
    x = torch.zeros((4, 16), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="16, 32, 64, 128 or 256"):
        nconv.gather_gemm(fmap, x, torch.zeros((24, 448), dtype=torch.bfloat16, device="cuda"), 24)


# ---------------------------------------------------------------- full size: the bench workload
@pytest.fixture(scope="module")
def bench_shell(cuda):
    """BASELINE config 4's per-GPU shard, the exact `bench.py` workload: 8 x 256^3 shells."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    return SuperPsh.from_levels([bench.shell_levels(256)[0]] * 8)


def test_full_size_native_layer_properties(bench_shell):
    """Size-independent properties of the fused kernels at N = 1,826,368, C 64 -> 64:
    (1) identity at the centre tap reproduces the input exactly; (2) the input gradient
    (flipped-kernel gather-GEMM) is the adjoint of the forward, <W*x, dy> = <x, W^T*dy>;
    (3) the weight gradient is the same bilinear form, <dW(x, dy), W> = <dy, W*x>. The fp32
    accumulation bound is scaled by the absolute-value forms (|W|*|x| etc.)."""
    s = bench_shell
    n, C = s.total_columns(), 64
    assert n == 8 * 228296
    fm = nconv.field_map_native(s, s, ConvSpec(3, 1, 0, C, C), nconv.TILED)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = (torch.rand((n, C), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    eye = torch.zeros((C, C * 27), device="cuda")
    eye.view(C, C, 27)[torch.arange(C), torch.arange(C), 13] = 1.0
    y = nconv.gather_gemm(fm, x, nconv.pack_weights(eye, C, C, 27, False), C, torch.float32)
    assert torch.equal(y, x.float())

    w = bf16_round(torch.rand((C, C * 27), device="cuda", generator=g) * 2 - 1)
    dy = (torch.rand((n, C), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    y = nconv.gather_gemm(fm, x, nconv.pack_weights(w, C, C, 27, False), C, torch.float32)
    dx = nconv.gather_gemm(fm, dy, nconv.pack_weights(w, C, C, 27, True), C, torch.float32)
    fwd_form = (y.double() * dy.double()).sum()
    adj_form = (x.double() * dx.double()).sum()
    ya = nconv.gather_gemm(fm, x.abs(), nconv.pack_weights(w.abs(), C, C, 27, False), C, torch.float32)
    scale = float((ya.double() * dy.double().abs()).sum())
    assert abs(float(fwd_form - adj_form)) <= 1e-5 * scale, (float(fwd_form), float(adj_form), scale)

    dw = nconv.conv_dw(fm, x, dy)
    dw_form = (dw.double() * w.double()).sum()
    assert abs(float(dw_form - fwd_form)) <= 1e-5 * scale, (float(dw_form), float(fwd_form), scale)


def test_dw_plan_rejects_shapes_beyond_tmem(cuda):
    """A (taps x C_in) extent whose m-tile groups cannot keep their accumulators in TMEM is an
    invalid argument (the workspace query returns 0), never a silent TMEM overrun."""
    from paper_1803_11385_b200._lib import lib
    assert lib.hc_native_dw_workspace(1000, 27, 2048, 256) == 0
    assert lib.hc_native_dw_workspace(1000, 27, 320, 256) > 0
    x = torch.zeros((64, 2048), dtype=torch.bfloat16, device="cuda")
    dy = torch.zeros((64, 256), dtype=torch.bfloat16, device="cuda")
    fmap = torch.zeros((64, 27), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match="dW supports at most"):
        nconv.conv_dw(fmap, x, dy)


@pytest.mark.parametrize("precision", ["bf16", "f32"])
@pytest.mark.parametrize("kernel,stride,pad", [(2, 2, 0), (3, 2, 0), (3, 2, 1)])
def test_strided_layer_vs_oracle(cuda, restated, precision, kernel, stride, pad):
    """Strided native layer (fine -> next-coarser structure): forward over the strided field map,
    dW by the split-K kernel on it, dX by the gather-GEMM over the TRANSPOSED map (cnn_ops.cpp:
    217-232 col2hash without a column matrix) vs the double oracle; bf16 on quantised operands,
    f32 on unquantised fp32 inputs (split precision), both within 1e-5 (dW 5e-5 at bf16)."""
    from helpers import random_pair
    f, c = random_pair(32, 3, seed=kernel * 10 + pad, n_lo=900, n_hi=2500)
    fa, ca = levels_to_arrays(f), levels_to_arrays(c)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    nf, nc = fine.total_columns(), coarse.total_columns()
    c_in, c_out = 32, 64
    rng = np.random.default_rng(kernel + pad)
    q = (lambda a: torch.from_numpy(a).to(torch.bfloat16).float().numpy()) if precision == "bf16" else (lambda a: a)
    x = q(rng.uniform(-1, 1, (c_in, nf)).astype(np.float32))
    taps = kernel ** 3
    w = q(rng.uniform(-1, 1, (c_out, c_in * taps)).astype(np.float32))
    dy = q(rng.uniform(-1, 1, (c_out, nc)).astype(np.float32))
    spec = ConvSpec(kernel, stride, pad, c_in, c_out)
    f64 = np.float64
    cols64 = restated.hash2col(fa, x.astype(f64), ca, spec, f64)
    y64 = restated.matmul(w.astype(f64), cols64, f64)
    dw64, dx64 = restated.conv_backward(dy.astype(f64), w.astype(f64), cols64, fa, ca, spec, f64)
    layer = nconv.HashConv(fine, torch.from_numpy(w).cuda(), spec, out_dtype=torch.float32, precision=precision,
                           output=coarse)
    if precision == "f32":
        xv, dyv = torch.from_numpy(x).cuda().t().contiguous(), torch.from_numpy(dy).cuda().t().contiguous()
    else:
        xv, dyv = nconv.to_voxel_major(torch.from_numpy(x).cuda()), nconv.to_voxel_major(torch.from_numpy(dy).cuda())
    y = layer.forward(xv).float().t().cpu().numpy()
    dw, dxv = layer.backward(dyv, xv, torch.float32)
    dx = dxv.float().t().cpu().numpy()
    assert y.shape == (c_out, nc) and dx.shape == (c_in, nf)
    assert rel(torch.from_numpy(y), torch.from_numpy(y64)) <= TOL_F32_OUT
    assert rel(dw.cpu(), torch.from_numpy(dw64)) <= (TOL_DW if precision == "bf16" else 1e-5)
    assert rel(torch.from_numpy(dx), torch.from_numpy(dx64)) <= TOL_F32_OUT
