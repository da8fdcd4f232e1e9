"""The rest of cnn_ops.hpp on the GPU (csrc/ops_layer.cu): batch norm, scale, ReLU and
inverted dropout, fp32 and fp64, against the unmodified reference (oracle/_ref).

Bars: ReLU, scale forward and dropout (its mask is the reference's mt19937_64 stream) are
bit-exact. Batch norm and scale backward reduce per channel in double (a fixed tree order
here, sequential in the reference): fp32 results are compared for equality — the double
sums differ only in their last bits, far below the float rounding step — and fp64 results
within 1e-12 relative."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200 import ops  # noqa: E402

DT = [np.float32, np.float64]


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _same(got, want, dtype, tol=1e-12):
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else got
    if np.dtype(dtype) == np.float32:
        assert np.array_equal(got, want), _rel(got, want)
    else:
        assert _rel(got, want) <= tol


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("c,n", [(3, 53), (16, 4099), (64, 100000), (5, 1)])
def test_batch_norm_matches_reference(cuda, ref, dtype, c, n):
    rng = np.random.default_rng(c * 7 + n)
    x = (rng.standard_normal((c, n)) * 3 + 1.5).astype(dtype)
    rm, rv = rng.uniform(-1, 1, c).astype(dtype), rng.uniform(0.5, 2, c).astype(dtype)
    for training in (True, False):
        y_r, rm_r, rv_r, inv_r = ref.bn_forward(x, rm, rv, 1e-5, 0.1, training, dtype)
        st = ops.BatchNormStats(c, dtype=dtype)
        st.running_mean[:], st.running_var[:] = rm, rv
        cache = ops.BatchNormCache()
        y = ops.batch_norm_forward(x, st, training, cache)
        _same(y, y_r, dtype)
        _same(cache.inv_std, inv_r, dtype)
        _same(st.running_mean, rm_r, dtype)
        _same(st.running_var, rv_r, dtype)
        if training:
            dy = rng.standard_normal((c, n)).astype(dtype)
            _same(ops.batch_norm_backward(dy, cache), ref.bn_backward(dy, y_r, inv_r, dtype), dtype)


@pytest.mark.parametrize("dtype", DT)
def test_scale_and_relu_match_reference(cuda, ref, dtype):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((7, 3001)).astype(dtype)
    x[0, :4] = [0.0, -0.0, 1e-30, -1e-30]
    g, b = rng.standard_normal(7).astype(dtype), rng.standard_normal(7).astype(dtype)
    assert np.array_equal(ops.scale_forward(x, g, b), ref.scale_forward(x, g, b, dtype))
    dy = rng.standard_normal(x.shape).astype(dtype)
    got = ops.scale_backward(dy, x, g)
    dg_r, db_r, dx_r = ref.scale_backward(dy, x, g, dtype)
    assert np.array_equal(got.input, dx_r)
    _same(got.gamma, dg_r, dtype)
    _same(got.beta, db_r, dtype)
    y_r, dx_r = ref.relu(x, dy, dtype)
    y = ops.relu_forward(x)
    assert np.array_equal(y.view(np.uint8), y_r.view(np.uint8))  # bitwise: +0 for -0 inputs
    assert np.array_equal(ops.relu_backward(dy, y), dx_r)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("shape,ratio,seed", [((4, 1000), 0.5, 7), ((1, 1), 0.3, 1), ((128, 97), 0.25, 2 ** 63 + 5),
                                              ((3, 313), 0.9, 0), ((640, 32), 0.5, 12345)])
def test_dropout_mask_is_the_reference_stream(cuda, ref, dtype, shape, ratio, seed):
    rng = np.random.default_rng(int(seed % 1000))
    x = rng.standard_normal(shape).astype(dtype)
    dy = rng.standard_normal(shape).astype(dtype)
    y_r, keep_r, dx_r = ref.dropout(x, ratio, seed, True, dy, dtype)
    mask = ops.DropoutMask()
    y = ops.dropout_forward(x, ratio, seed, True, mask)
    assert np.array_equal(mask.keep, keep_r)
    assert np.array_equal(y, y_r)
    assert np.array_equal(ops.dropout_backward(dy, mask, ratio), dx_r)


def test_dropout_identity_modes_and_errors(cuda, ref):
    x = np.arange(12, dtype=np.float32).reshape(3, 4)
    for training, ratio in ((False, 0.5), (True, 0.0)):
        mask = ops.DropoutMask()
        assert np.array_equal(ops.dropout_forward(x, ratio, 3, training, mask), x)
        assert (mask.keep == 1).all()
    with pytest.raises(ValueError, match=r"dropout ratio must be in \[0,1\)"):
        ops.dropout_forward(x, 1.0, 3, True)
    with pytest.raises(ValueError, match="batch_norm: empty input"):
        ops.batch_norm_forward(np.zeros((2, 0), np.float32), ops.BatchNormStats(2), True)
    with pytest.raises(ValueError, match="batch_norm: stats channel mismatch"):
        ops.batch_norm_forward(np.zeros((2, 5), np.float32), ops.BatchNormStats(3), True)
    with pytest.raises(ValueError, match="relu_backward: shape mismatch"):
        ops.relu_backward(np.zeros((2, 5), np.float32), np.zeros((2, 4), np.float32))
