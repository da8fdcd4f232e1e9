"""fp64 reference-layout operators (the reference's double instantiation, cnn_ops.cpp:652-653,
gemm.cpp:117-118) through the C ABI's *_f64 entry points: bit-identical to the unmodified
reference's double results on the golden instances (tests/golden: conv64 / dw64 / dx64 are
oracle/_ref outputs) and to the C oracle's double instantiation on random batches (every
operator, strided and stride-1 specs). ops.py picks the precision from the inputs' dtype,
like the reference templates."""
import numpy as np
import pytest
import torch

from helpers import golden_instances, levels_to_arrays, load_instance, random_pair

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200 import ops  # noqa: E402
from paper_1803_11385_b200.ops import ConvSpec  # noqa: E402
from paper_1803_11385_b200.psh import SuperPsh  # noqa: E402

F64 = np.float64


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else t


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("path", golden_instances(), ids=lambda p: p.split("/")[-1])
def test_golden_double_instantiation_bit_exact(cuda, path):
    z, fa, ca = load_instance(path)
    fine, coarse = SuperPsh.from_host(fa), SuperPsh.from_host(ca)
    spec = ConvSpec(*(int(x) for x in z["spec"]))
    out_s = fine if spec.stride == 1 else coarse
    data, w, dout = (_dev(z[k].astype(F64)) for k in ("data", "w", "dout"))
    out = ops.conv_forward(fine, data, out_s, w, spec)
    assert out.dtype == torch.float64
    assert np.array_equal(_np(out), z["conv64"])
    cols = ops.hash2col(fine, data, out_s, spec)
    g = ops.conv_backward(dout, w, cols, fine, out_s, spec)
    assert np.array_equal(_np(g.weights), z["dw64"]) and np.array_equal(_np(g.input), z["dx64"])


@pytest.mark.parametrize("spec", [(3, 1, 0), (2, 2, 0), (3, 2, 0), (2, 2, 1), (5, 1, 0)])
def test_random_batches_f64_vs_oracle(cuda, restated, spec):
    f, c = random_pair(16, 3, seed=(hash(spec) & 0xFFFF) + 7, n_lo=150, n_hi=500)
    fa, ca = levels_to_arrays(f), levels_to_arrays(c)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    sp = ConvSpec(*spec, 4, 6)
    out_s, out_a = (fine, fa) if sp.stride == 1 else (coarse, ca)
    rng = np.random.default_rng(11)
    fd = sp.kernel ** 3
    data = rng.uniform(-1, 1, (4, fa.total_columns()))
    w = rng.uniform(-1, 1, (6, 4 * fd))
    dout = rng.uniform(-1, 1, (6, out_a.total_columns()))
    ocols = restated.hash2col(fa, data, out_a, sp, F64)
    cols = ops.hash2col(fine, _dev(data), out_s, sp)
    assert cols.dtype == torch.float64 and np.array_equal(_np(cols), ocols)
    assert np.array_equal(_np(ops.conv_forward(fine, _dev(data), out_s, _dev(w), sp)),
                          restated.matmul(w, ocols, F64))
    g = ops.conv_backward(_dev(dout), _dev(w), cols, fine, out_s, sp)
    odw, odx = restated.conv_backward(dout, w, ocols, fa, out_a, sp, F64)
    assert np.array_equal(_np(g.weights), odw) and np.array_equal(_np(g.input), odx)
    y = rng.uniform(-1, 1, ocols.shape)
    assert np.array_equal(_np(ops.col2hash(_dev(y), fine, out_s, sp)), restated.col2hash(y, fa, out_a, sp, F64))
    if sp.stride > 1:
        psp = ConvSpec(sp.kernel, sp.stride, sp.pad, 4, 4)
        q = rng.integers(-3, 4, (4, fa.total_columns())).astype(F64)  # ties: first-hit seed, strict '>'
        mp = ops.max_pool(fine, _dev(q), coarse, psp)
        om, osw = restated.max_pool(fa, q, ca, psp, F64)
        assert np.array_equal(_np(mp.output), om) and np.array_equal(_np(mp.switches), osw)
        assert np.array_equal(_np(ops.max_unpool(mp.output, mp.switches, fine, coarse, psp)),
                              restated.max_unpool(om, osw, fa, ca, psp, F64))
        assert np.array_equal(_np(ops.avg_pool(fine, _dev(data), coarse, psp)),
                              restated.avg_pool(fa, data, ca, psp, F64))
        cv = rng.uniform(-1, 1, (4, ca.total_columns()))
        assert np.array_equal(_np(ops.avg_unpool(_dev(cv), fine, coarse, psp)),
                              restated.avg_unpool(cv, fa, ca, psp, F64))
        # deconvolution (coarse C_out=6 -> fine C_in=4) and its backward
        dw_ = rng.uniform(-1, 1, (6, 4 * fd))
        din = rng.uniform(-1, 1, (6, ca.total_columns()))
        assert np.array_equal(_np(ops.deconv_forward(coarse, _dev(din), fine, _dev(dw_), sp)),
                              restated.deconv_forward(ca, din, fa, dw_, sp, F64))
        fg = rng.uniform(-1, 1, (4, fa.total_columns()))
        b = ops.deconv_backward(_dev(fg), _dev(dw_), _dev(din), coarse, fine, sp)
        rdw, rdx = restated.deconv_backward(fg, dw_, din, ca, fa, sp, F64)
        assert np.array_equal(_np(b.weights), rdw) and np.array_equal(_np(b.input), rdx)


def test_gemms_f64_bit_exact(cuda, restated):
    rng = np.random.default_rng(8)
    a, b = rng.uniform(-1, 1, (7, 300)), rng.uniform(-1, 1, (300, 129))
    a[a < -0.8] = 0.0  # the reference skips zero a-entries (gemm.cpp:21)
    assert np.array_equal(_np(ops.matmul(_dev(a), _dev(b))), restated.matmul(a, b, F64))
    c = rng.uniform(-1, 1, (7, 129))
    assert np.array_equal(_np(ops.matmul_trans_a(_dev(a), _dev(c))), restated.matmul_trans_a(a, c, F64))
    d = rng.uniform(-1, 1, (11, 300))
    assert np.array_equal(_np(ops.matmul_trans_b(_dev(a), _dev(d))), restated.matmul_trans_b(a, d, F64))


def test_mixed_inputs_follow_the_first_floating_input(cuda):
    """Like the reference templates: T comes from the inputs; a float32 call stays fp32."""
    x32 = torch.rand((3, 40), device="cuda")
    y32 = torch.rand((40, 5), device="cuda")
    assert ops.matmul(x32, y32).dtype == torch.float32
    assert ops.matmul(x32.double(), y32).dtype == torch.float64
