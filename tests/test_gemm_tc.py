"""Reference-layout contraction on tcgen05 (csrc/gemm_tc.cu): matmul / matmul_trans_a /
matmul_trans_b (gemm.cpp:14-69) through the C ABI in each math mode, against the float64
product of the same fp32 operands. FAST = 3xTF32 (TMA-eligible shapes) or FFMA tiles
(others), held to the reference-layout FAST bar of 1e-5 normwise; TF32 = one tf32 pass,
held to 2e-3. Shapes cover K tails (K % 32 != 0), column and row tails, multi-tile rows
(ra > 128), the split-K path (long K, few tiles) and unaligned shapes (FFMA fallback)."""
import numpy as np
import pytest
import torch

from helpers import rel_fro

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200 import ops  # noqa: E402

FAST_TOL, TF32_TOL = 1e-5, 2e-3

# (ra, k, cb): conv fwd Y = W cols (ra = C_out, k = 27 C_in, cb = voxels) and friends
NN = [(16, 216, 3680), (64, 1728, 20000), (7, 36, 132), (200, 100, 1000), (64, 27 * 8, 999), (5, 33, 77)]
# matmul_trans_b (dW = dY cols^T): (ra = C_out, k = voxels, rb = 27 C_in)
NT = [(16, 3680, 216), (64, 100000, 1728), (32, 4100, 36), (8, 2000, 100), (3, 901, 27)]
# matmul_trans_a (dcols = W^T dY): (ra = C_out, k = 27 C_in, cb = voxels)
TN = [(16, 216, 3680), (64, 1728, 10000), (64, 300, 132), (9, 40, 1001)]


def _run(fn, a, b, mode):
    with ops.math_mode(mode):
        c = fn(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    return c.cpu().numpy()


def _rand(rng, *shape):
    return rng.uniform(-1, 1, shape).astype(np.float32)


@pytest.mark.parametrize("mode,tol", [("fast", FAST_TOL), ("tf32", TF32_TOL)])
@pytest.mark.parametrize("ra,k,cb", NN)
def test_matmul(cuda, mode, tol, ra, k, cb):
    rng = np.random.default_rng(ra * 7 + k + cb)
    a, b = _rand(rng, ra, k), _rand(rng, k, cb)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    assert rel_fro(_run(ops.matmul, a, b, mode), ref) <= tol


@pytest.mark.parametrize("mode,tol", [("fast", FAST_TOL), ("tf32", TF32_TOL)])
@pytest.mark.parametrize("ra,k,rb", NT)
def test_matmul_trans_b(cuda, mode, tol, ra, k, rb):
    rng = np.random.default_rng(ra * 5 + k + rb)
    a, b = _rand(rng, ra, k), _rand(rng, rb, k)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    assert rel_fro(_run(ops.matmul_trans_b, a, b, mode), ref) <= tol


@pytest.mark.parametrize("mode,tol", [("fast", FAST_TOL), ("tf32", TF32_TOL)])
@pytest.mark.parametrize("ra,k,cb", TN)
def test_matmul_trans_a(cuda, mode, tol, ra, k, cb):
    rng = np.random.default_rng(ra * 3 + k + cb)
    a, b = _rand(rng, ra, k), _rand(rng, ra, cb)
    ref = a.astype(np.float64).T @ b.astype(np.float64)
    assert rel_fro(_run(ops.matmul_trans_a, a, b, mode), ref) <= tol


def test_split_k_is_deterministic(cuda):
    rng = np.random.default_rng(3)
    a, b = _rand(rng, 64, 200000), _rand(rng, 1728, 200000)
    c1 = _run(ops.matmul_trans_b, a, b, "fast")
    c2 = _run(ops.matmul_trans_b, a, b, "fast")
    assert np.array_equal(c1, c2)


def test_tf32_mode_is_tensor_core(cuda):
    """tf32 differs from the fp32 FAST product on a TMA-eligible shape (i.e. the tf32
    tensor path ran) but is identical to it on an unaligned one (both take FFMA)."""
    rng = np.random.default_rng(4)
    a, b = _rand(rng, 64, 256), _rand(rng, 256, 1024)
    assert not np.array_equal(_run(ops.matmul, a, b, "tf32"), _run(ops.matmul, a, b, "fast"))
    a, b = _rand(rng, 64, 255), _rand(rng, 255, 1023)
    assert np.array_equal(_run(ops.matmul, a, b, "tf32"), _run(ops.matmul, a, b, "fast"))


def test_tensor_core_truncates_tf32_operands(cuda):
    """gemm_tc.cu's 3xTF32 split uses the raw fp32 tile as its hi part, which is valid only
    because the tensor core truncates fp32 operands to tf32 (low 13 bits ignored): pin that."""
    rng = np.random.default_rng(5)
    a, b = _rand(rng, 64, 256), _rand(rng, 256, 1024)

    def trunc(x):
        return (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)

    assert np.array_equal(_run(ops.matmul, a, b, "tf32"), _run(ops.matmul, trunc(a), trunc(b), "tf32"))
