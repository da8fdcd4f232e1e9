"""Split-precision fused conv (hc_native_*_x2): the reference's fp32 conv_forward /
conv_backward (cnn_ops.cpp:206-232) on the tcgen05 bf16 path, fp32 operands carried as
bf16 hi/lo planes.

Tolerance contract: on UNQUANTISED fp32 inputs the GPU result is
within ||gpu - ref64||_F / ||ref64||_F <= 1e-5 of the float64 instantiation of the same
sparse op — forward, weight gradient and input gradient alike. (The representation error
of the split is <= 2^-17 relative per operand; measured ~4e-6 normwise at every size up to
the 256^3 x 8 bench workload, dW with 8192-voxel accumulation chains.)"""
import numpy as np
import pytest
import torch

from helpers import levels_to_arrays, random_pair, shell_pair

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200 import conv as nconv  # noqa: E402
from paper_1803_11385_b200.ops import ConvSpec  # noqa: E402
from paper_1803_11385_b200.psh import SuperPsh  # noqa: E402

TOL = 1e-5


def rel(a, b):
    a, b = torch.as_tensor(a).double(), torch.as_tensor(b).double()
    return float((a.cpu() - b.cpu()).norm() / b.cpu().norm().clamp_min(1e-300))


def ref64(fmap_rows, x, w, dy, c_in, c_out):
    """float64 forward / dW / dX of the gather-GEMM over a row-major field map (-1 = empty):
    Y[n] = sum_t X[map(n,t)] W_t^T, dW_t = dY^T X[map(.,t)], dX = scatter of dY W_t."""
    n, taps = fmap_rows.shape
    x64 = torch.cat([x.double(), torch.zeros((1, c_in), dtype=torch.float64, device=x.device)])
    dy64 = dy.double()
    w64 = w.double().view(c_out, c_in, taps)
    y = torch.zeros((n, c_out), dtype=torch.float64, device=x.device)
    dw = torch.zeros((c_out, c_in, taps), dtype=torch.float64, device=x.device)
    dx = torch.zeros((x.shape[0] + 1, c_in), dtype=torch.float64, device=x.device)
    for t in range(taps):
        col = fmap_rows[:, t].long()
        idx = torch.where(col >= 0, col, torch.full_like(col, x.shape[0]))
        g = x64[idx]
        y += g @ w64[:, :, t].T
        dw[:, :, t] = dy64.T @ g
        dx.index_add_(0, idx, dy64 @ w64[:, :, t])
    return y, dw.reshape(c_out, c_in * taps), dx[:-1]


def _rand(shape, g):
    return torch.rand(shape, device="cuda", generator=g) * 2 - 1


@pytest.mark.parametrize("c_in,c_out", [(8, 16), (16, 16), (32, 64), (64, 64), (64, 128), (128, 32), (128, 128),
                                        (24, 32), (40, 16)])
def test_x2_random_maps(cuda, c_in, c_out):
    """Forward and weight gradient on random maps with 40% empty cells, unquantised inputs."""
    g = torch.Generator(device="cuda").manual_seed(c_in * 100 + c_out)
    n = 20011
    x, dy = _rand((n, c_in), g), _rand((n, c_out), g)
    w = _rand((c_out, c_in * 27), g)
    fm = torch.randint(-1, n, (n, 27), device="cuda", generator=g, dtype=torch.int32)
    fm[torch.rand((n, 27), device="cuda", generator=g) < 0.4] = -1
    y64, dw64, _ = ref64(fm, x, w, dy, c_in, c_out)
    xs, dys = nconv.split(x), nconv.split(dy)
    y = nconv.gather_gemm_x2(fm, xs, nconv.pack_weights_x2(w, c_out, c_in, 27), c_out)
    dw = nconv.conv_dw_x2(fm, xs, dys)
    assert rel(y, y64) <= TOL
    assert rel(dw, dw64) <= TOL
    assert torch.equal(nconv.conv_dw_x2(fm, xs, dys), dw), "dW must be deterministic"


def test_split_planes(cuda):
    """hi = rn(v), lo = rn(v - hi); both layouts give the same rows; |v - hi - lo| <= 2^-17 |v|."""
    g = torch.Generator(device="cuda").manual_seed(3)
    x = _rand((1001, 40), g) * 1e3
    s = nconv.split(x)
    assert s.shape == (1001, 80) and s.dtype == torch.bfloat16
    hi, lo = s[:, :40].float(), s[:, 40:].float()
    assert torch.equal(hi, x.to(torch.bfloat16).float())
    assert torch.equal(lo, (x - hi).to(torch.bfloat16).float())
    assert float(((x - hi - lo).abs() / x.abs().clamp_min(1e-30)).max()) <= 2.0 ** -17
    assert torch.equal(nconv.split(x.t().contiguous(), channel_major=True), s)


@pytest.mark.parametrize("c_in,c_out", [(64, 64), (16, 32), (3, 2), (128, 128)])
def test_x2_layer_vs_double_oracle_on_shell(cuda, restated, c_in, c_out):
    """The whole layer (forward, dW, dX) on a 64^3 x 2 shell batch vs the double oracle's
    conv_forward / conv_backward (oracle/hc_oracle.c, cnn_ops.cpp:206-232) on the SAME
    unquantised fp32 inputs; 3 -> 2 exercises the channel padding."""
    f, _ = shell_pair(64, 2)
    fa = levels_to_arrays(f)
    s = SuperPsh.from_levels(f)
    N = s.total_columns()
    rng = np.random.default_rng(c_in * 7 + c_out)
    x = rng.uniform(-1, 1, (c_in, N)).astype(np.float32)
    w = rng.uniform(-1, 1, (c_out, c_in * 27)).astype(np.float32)
    dy = rng.uniform(-1, 1, (c_out, N)).astype(np.float32)
    spec = ConvSpec(3, 1, 0, c_in, c_out)
    f64 = np.float64
    cols64 = restated.hash2col(fa, x.astype(f64), fa, spec, f64)
    y64 = restated.matmul(w.astype(f64), cols64, f64)
    dw64, dx64 = restated.conv_backward(dy.astype(f64), w.astype(f64), cols64, fa, fa, spec, f64)

    layer = nconv.HashConv(s, torch.from_numpy(w).cuda(), spec, precision="f32")
    xv = torch.from_numpy(x).cuda().t().contiguous()
    y = layer.forward(xv)
    dw, dxv = layer.backward(torch.from_numpy(dy).cuda().t().contiguous(), xv)
    assert y.dtype == torch.float32 and dxv.dtype == torch.float32
    assert rel(y.t(), y64) <= TOL
    assert rel(dw, dw64) <= TOL
    assert rel(dxv.t(), dx64) <= TOL


@pytest.mark.parametrize("n", [1, 127, 128, 129])
def test_x2_tiny_and_ragged(cuda, n):
    g = torch.Generator(device="cuda").manual_seed(n)
    c_in, c_out, n_in = 16, 32, n + 5
    x, dy, w = _rand((n_in, c_in), g), _rand((n, c_out), g), _rand((c_out, c_in * 27), g)
    fm = torch.randint(-1, n_in, (n, 27), device="cuda", generator=g, dtype=torch.int32)
    y64, dw64, _ = ref64(fm, x, w, dy, c_in, c_out)
    y = nconv.gather_gemm_x2(fm, nconv.split(x), nconv.pack_weights_x2(w, c_out, c_in, 27), c_out)
    # dY rows beyond the map's n: the dW's dY operand has exactly n rows
    dw = nconv.conv_dw_x2(fm, nconv.split(x), nconv.split(dy))
    assert rel(y, y64) <= TOL
    assert rel(dw, dw64) <= TOL


def test_x2_empty_and_errors(cuda):
    xs = torch.zeros((4, 32), dtype=torch.bfloat16, device="cuda")
    fm = torch.zeros((0, 27), dtype=torch.int32, device="cuda")
    wp = nconv.pack_weights_x2(torch.zeros((32, 16 * 27), device="cuda"), 32, 16, 27)
    assert nconv.gather_gemm_x2(fm, xs, wp, 32).shape == (0, 32)
    dw = nconv.conv_dw_x2(fm, xs, torch.zeros((0, 64), dtype=torch.bfloat16, device="cuda"))
    assert dw.shape == (32, 16 * 27) and float(dw.abs().sum()) == 0.0
    fm = torch.zeros((4, 27), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match="at most 128"):
        nconv.gather_gemm_x2(fm, xs, torch.zeros((512, 896), dtype=torch.bfloat16, device="cuda"), 256)
    with pytest.raises(ValueError, match="multiple of 4"):
        nconv.split(torch.zeros((4, 6), device="cuda"))


# ---------------------------------------------------------------- full size: the bench workload
@pytest.fixture(scope="module")
def bench_shell(cuda):
    """BASELINE config 4's per-GPU shard, the exact `bench.py` workload: 8 x 256^3 shells."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    return SuperPsh.from_levels([bench.shell_levels(256)[0]] * 8)


def test_x2_full_size_vs_float64(bench_shell):
    """N = 1,826,368 voxels, C 64 -> 64 (the bench workload, fp32 headline): forward, dW
    (reduction over 1.8 M voxels) and dX against float64 computed on the device."""
    s = bench_shell
    n, C = s.total_columns(), 64
    spec = ConvSpec(3, 1, 0, C, C)
    g = torch.Generator(device="cuda").manual_seed(11)
    x, dy, w = _rand((n, C), g), _rand((n, C), g), _rand((C, C * 27), g)
    layer = nconv.HashConv(s, w, spec, precision="f32")
    y = layer.forward(x)
    dw, dx = layer.backward(dy, x)
    rows = nconv.field_map_native(s, s, spec, nconv.ROW_MAJOR).data
    y64, dw64, dx64 = ref64(rows, x, w, dy, C, C)
    assert rel(y, y64) <= TOL
    assert rel(dw, dw64) <= TOL
    assert rel(dx, dx64) <= TOL
