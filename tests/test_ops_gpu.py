"""GPU parity of the reference-layout operators (C ABI through ops.py) against the
reference's golden fixtures, the CPU oracle (oracle/hc_oracle.c) and the reference's
own known-answer tests (tests/test_cnn_ops.cpp). EXACT math is bit-identical; FAST
math is checked against the double instantiation with a normwise bound."""
import numpy as np
import pytest
import torch

from helpers import GOLDEN, golden_instances, levels_to_arrays, load_instance, random_pair, rel_fro, sha, shell_pair

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200 import ops  # noqa: E402
from paper_1803_11385_b200.ops import ConvSpec  # noqa: E402
from paper_1803_11385_b200.psh import PshLevel, SuperPsh, VoxelSet  # noqa: E402

FAST_TOL = 1e-5  # ||gpu - ref64||_F / ||ref64||_F for fp32


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else t


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ---------------------------------------------------------------- golden instances
@pytest.mark.parametrize("path", golden_instances(), ids=lambda p: p.split("/")[-1])
def test_golden_instance_bit_exact(cuda, path):
    z, fa, ca = load_instance(path)
    fine, coarse = SuperPsh.from_host(fa), SuperPsh.from_host(ca)
    spec = ConvSpec(*(int(x) for x in z["spec"]))
    dc_spec = ConvSpec(*(int(x) for x in z["dc_spec"]))
    pool = ConvSpec(*(int(x) for x in z["pool_spec"]))
    out_s = fine if spec.stride == 1 else coarse
    data, w, dout = _dev(z["data"]), _dev(z["w"]), _dev(z["dout"])
    cols = ops.hash2col(fine, data, out_s, spec)
    assert sha(_np(cols)) == str(z["cols_sha"])
    assert np.array_equal(_np(ops.conv_forward(fine, data, out_s, w, spec)), z["conv_out"])
    g = ops.conv_backward(dout, w, cols, fine, out_s, spec)
    assert np.array_equal(_np(g.weights), z["dw"])
    assert np.array_equal(_np(g.input), z["dx"])
    mp = ops.max_pool(fine, data, coarse, pool)
    assert np.array_equal(_np(mp.output), z["mp"]) and np.array_equal(_np(mp.switches), z["sw"])
    assert np.array_equal(_np(ops.avg_pool(fine, data, coarse, pool)), z["ap"])
    assert np.array_equal(_np(ops.max_unpool(mp.output, mp.switches, fine, coarse, pool)), z["max_restored"])
    assert np.array_equal(_np(ops.avg_unpool(_dev(z["coarse_vals"]), fine, coarse, pool)), z["avg_restored"])
    assert np.array_equal(_np(ops.deconv_forward(coarse, _dev(z["dc_in"]), fine, _dev(z["dc_w"]), dc_spec)),
                          z["dc_out"])
    b = ops.deconv_backward(data, _dev(z["dc_w"]), _dev(z["dc_in"]), coarse, fine, dc_spec)
    assert np.array_equal(_np(b.weights), z["dcb_dw"]) and np.array_equal(_np(b.input), z["dcb_dx"])
    assert np.array_equal(_np(ops.col2hash(_dev(z["y"]), fine, out_s, spec)), z["c2h"])


@pytest.mark.parametrize("path", golden_instances()[:6], ids=lambda p: p.split("/")[-1])
def test_golden_instance_fast_math_tolerance(cuda, path):
    z, fa, ca = load_instance(path)
    fine, coarse = SuperPsh.from_host(fa), SuperPsh.from_host(ca)
    spec = ConvSpec(*(int(x) for x in z["spec"]))
    out_s = fine if spec.stride == 1 else coarse
    with ops.math_mode("fast"):
        data, w, dout = _dev(z["data"]), _dev(z["w"]), _dev(z["dout"])
        out = ops.conv_forward(fine, data, out_s, w, spec)
        cols = ops.hash2col(fine, data, out_s, spec)
        g = ops.conv_backward(dout, w, cols, fine, out_s, spec)
    assert rel_fro(_np(out), z["conv64"]) <= FAST_TOL
    assert rel_fro(_np(g.weights), z["dw64"]) <= FAST_TOL
    assert rel_fro(_np(g.input), z["dx64"]) <= FAST_TOL


def test_shell32_config1_digests(cuda):
    """BASELINE config 1: 32^3 shell, 3x3x3 conv C 8->16 fwd/bwd + max-pool (+unpool)."""
    from oracle.oracle import Ref, have_ref
    z = np.load(f"{GOLDEN}/shell32.npz")
    f, c = shell_pair(32, 1)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    assert fine.total_columns() == 3680 and coarse.total_columns() == 896
    if not have_ref():
        pytest.skip("seeded inputs come from the reference RNG (oracle/_ref)")
    ref = Ref()
    data = _dev(ref.random_matrix(8, 3680, 5))
    w = _dev(ref.random_matrix(16, 8 * 27, 6))
    dout = _dev(ref.random_matrix(16, 3680, 7))
    spec, pool = ConvSpec(3, 1, 0, 8, 16), ConvSpec(2, 2, 0, 8, 8)
    cols = ops.hash2col(fine, data, fine, spec)
    assert sha(_np(cols)) == str(z["cols"])
    assert sha(_np(ops.conv_forward(fine, data, fine, w, spec))) == str(z["conv_out"])
    g = ops.conv_backward(dout, w, cols, fine, fine, spec)
    assert sha(_np(g.weights)) == str(z["dw"]) and sha(_np(g.input)) == str(z["dx"])
    mp = ops.max_pool(fine, data, coarse, pool)
    assert sha(_np(mp.output)) == str(z["mp"]) and sha(_np(mp.switches)) == str(z["sw"])
    assert sha(_np(ops.max_unpool(mp.output, mp.switches, fine, coarse, pool))) == str(z["unpool"])


# ---------------------------------------------------------------- oracle parity, larger
@pytest.mark.parametrize("spec", [(3, 1, 0), (2, 2, 0), (3, 2, 0), (2, 2, 1), (1, 1, 0), (5, 1, 0), (4, 2, 1)])
def test_random_batches_vs_oracle(cuda, restated, spec):
    f, c = random_pair(16, 3, seed=hash(spec) & 0xFFFF, n_lo=150, n_hi=600)
    fa, ca = levels_to_arrays(f), levels_to_arrays(c)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    sp = ConvSpec(*spec, 5, 7)
    out_s, out_a = (fine, fa) if sp.stride == 1 else (coarse, ca)
    rng = np.random.default_rng(1)
    fd = sp.kernel ** 3
    data = rng.uniform(-1, 1, (5, fa.total_columns())).astype(np.float32)
    w = rng.uniform(-1, 1, (7, 5 * fd)).astype(np.float32)
    dout = rng.uniform(-1, 1, (7, out_a.total_columns())).astype(np.float32)
    fm = _np(ops.field_map(fine, out_s, sp))
    assert np.array_equal(fm.astype(np.int64), restated.field_map(fa, out_a, sp))
    cols = ops.hash2col(fine, _dev(data), out_s, sp)
    ocols = restated.hash2col(fa, data, out_a, sp)
    assert np.array_equal(_np(cols), ocols)
    assert np.array_equal(_np(ops.conv_forward(fine, _dev(data), out_s, _dev(w), sp)), restated.matmul(w, ocols))
    g = ops.conv_backward(_dev(dout), _dev(w), cols, fine, out_s, sp)
    odw, odx = restated.conv_backward(dout, w, ocols, fa, out_a, sp)
    assert np.array_equal(_np(g.weights), odw) and np.array_equal(_np(g.input), odx)
    if sp.stride > 1:
        psp = ConvSpec(sp.kernel, sp.stride, sp.pad, 5, 5)
        mp = ops.max_pool(fine, _dev(data), coarse, psp)
        om, osw = restated.max_pool(fa, data, ca, psp)
        assert np.array_equal(_np(mp.output), om) and np.array_equal(_np(mp.switches), osw)
        assert np.array_equal(_np(ops.max_unpool(mp.output, mp.switches, fine, coarse, psp)),
                              restated.max_unpool(om, osw, fa, ca, psp))
        assert np.array_equal(_np(ops.avg_pool(fine, _dev(data), coarse, psp)), restated.avg_pool(fa, data, ca, psp))
        cv = rng.uniform(-1, 1, (5, ca.total_columns())).astype(np.float32)
        assert np.array_equal(_np(ops.avg_unpool(_dev(cv), fine, coarse, psp)), restated.avg_unpool(cv, fa, ca, psp))


def test_shell64_batch4_vs_oracle(cuda, restated):
    f, c = shell_pair(64, 4)
    fa, ca = levels_to_arrays(f), levels_to_arrays(c)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    sp = ConvSpec(3, 1, 0, 16, 16)
    rng = np.random.default_rng(2)
    N = fa.total_columns()
    data = rng.uniform(-1, 1, (16, N)).astype(np.float32)
    cols = ops.hash2col(fine, _dev(data), fine, sp)
    ocols = restated.hash2col(fa, data, fa, sp)
    assert np.array_equal(_np(cols), ocols)
    y = rng.uniform(-1, 1, ocols.shape).astype(np.float32)
    assert np.array_equal(_np(ops.col2hash(_dev(y), fine, fine, sp)), restated.col2hash(y, fa, fa, sp))
    psp = ConvSpec(2, 2, 0, 16, 16)
    mp = ops.max_pool(fine, _dev(data), coarse, psp)
    om, osw = restated.max_pool(fa, data, ca, psp)
    assert np.array_equal(_np(mp.output), om) and np.array_equal(_np(mp.switches), osw)
    assert np.array_equal(_np(ops.max_unpool(mp.output, mp.switches, fine, coarse, psp)),
                          restated.max_unpool(om, osw, fa, ca, psp))


@pytest.mark.parametrize("C,pad", [(7, 0), (16, 0), (5, 1)])
def test_staged_pool_vs_oracle(cuda, restated, C, pad):
    """2^3 pooling through k_pool_staged (ops_ref.cu): 128^3 shells (blocks stage their
    child spans through shared memory) mixed with a sparse random set of the same
    resolution (blocks spanning many (model, z) pairs take the direct gathers). An odd
    column count (N % 4 != 0) makes every plane's span start at a different 16-byte
    alignment shift, and the last plane's copies meet the array end."""
    fs, cs = shell_pair(128, 1)
    fr, cr = random_pair(128, 1, seed=11, n_lo=30001, n_hi=30001)
    f, c = [fs[0], fr[0], fs[0]], [cs[0], cr[0], cs[0]]
    fa, ca = levels_to_arrays(f), levels_to_arrays(c)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    assert fa.total_columns() % 4 != 0
    psp = ConvSpec(2, 2, pad, C, C)  # pad 1: every field straddles two coarse-z child planes differently
    rng = np.random.default_rng(C)
    data = rng.integers(-4, 5, (C, fa.total_columns())).astype(np.float32)  # many ties: strict '>' order
    mp = ops.max_pool(fine, _dev(data), coarse, psp)
    om, osw = restated.max_pool(fa, data, ca, psp)
    assert np.array_equal(_np(mp.output), om) and np.array_equal(_np(mp.switches), osw)
    assert np.array_equal(_np(ops.avg_pool(fine, _dev(data), coarse, psp)), restated.avg_pool(fa, data, ca, psp))
    # the adjoint direction through k_unpool_staged (coarse spans per (model, coarse z))
    assert np.array_equal(_np(ops.max_unpool(mp.output, mp.switches, fine, coarse, psp)),
                          restated.max_unpool(om, osw, fa, ca, psp))
    cv = rng.uniform(-1, 1, (C, ca.total_columns())).astype(np.float32)
    cv[:, ::7] = -0.0  # 0 (+) -0.0 -> +0.0 as in the reference
    assert np.array_equal(_np(ops.avg_unpool(_dev(cv), fine, coarse, psp)).view(np.uint32),
                          restated.avg_unpool(cv, fa, ca, psp).view(np.uint32))


def test_staged_pool_captures_into_a_graph(cuda):
    """k_pool_staged (2^3 max / avg pooling) replays from a CUDA graph with the same results."""
    f, c = shell_pair(64, 2)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    sp = ConvSpec(2, 2, 0, 16, 16)
    x = torch.randn((16, fine.total_columns()), device="cuda")
    want = ops.max_pool(fine, x, coarse, sp)
    want_avg = ops.avg_pool(fine, x, coarse, sp)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ops.max_pool(fine, x, coarse, sp)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        got = ops.max_pool(fine, x, coarse, sp)
        got_avg = ops.avg_pool(fine, x, coarse, sp)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(got.output, want.output) and torch.equal(got.switches, want.switches)
    assert torch.equal(got_avg, want_avg)


def test_locate_matches_oracle(cuda, restated):
    f, _ = random_pair(16, 2, seed=5)
    fa = levels_to_arrays(f)
    s = SuperPsh.from_levels(f)
    rng = np.random.default_rng(0)
    q = np.concatenate([rng.integers(1, 3, (4000, 1)), rng.integers(0, 16, (4000, 3))], axis=1).astype(np.int32)
    got = _np(ops.locate(s, _dev(q)))
    want = np.array([restated.locate(fa, int(r[0]), r[1:]) for r in q])
    assert np.array_equal(got, want)
    back = s.download()
    for k in ("hash", "offsets", "tags", "model_of_slot", "hash_acc", "offset_acc", "data_acc"):
        assert np.array_equal(getattr(back, k), getattr(fa, k).astype(getattr(back, k).dtype))


# ---------------------------------------------------------------- known-answer tests (test_cnn_ops.cpp)
def _single(p, res, value=2.5):
    lvl = PshLevel.build(VoxelSet.make(3, res, [p], [[value]]))
    return SuperPsh.from_levels([lvl]), torch.tensor([[value]], device="cuda")


def test_kat_isolated_voxel_center_row(cuda):  # test_cnn_ops.cpp:53-62
    s, d = _single((4, 4, 4), 8)
    cols = _np(ops.hash2col(s, d, s, ConvSpec(3, 1, 0, 1, 1)))
    assert cols.shape == (27, 1)
    assert all(cols[r, 0] == (2.5 if r == 13 else 0.0) for r in range(27))


def test_kat_stride2_field_gathers_cube(cuda):  # test_cnn_ops.cpp:64-97
    coords = [(x, y, z) for z in (2, 3) for y in (2, 3) for x in (2, 3)] + [(0, 0, 0), (5, 5, 5)]
    vals = [100 + i for i in range(8)] + [7, 9]
    fs = VoxelSet.make(3, 8, coords, [vals])
    fine = SuperPsh.from_levels([PshLevel.build(fs)])
    coarse = SuperPsh.from_levels([PshLevel.build(VoxelSet.make(3, 4, [(1, 1, 1)], [[0.0]]))])
    fc, ff = fs.arrays()
    cols = _np(ops.hash2col(fine, _dev(ff), coarse, ConvSpec(2, 2, 0, 1, 1)))
    assert cols.shape == (8, 1)
    for row in range(8):
        p = (2 + (row & 1), 2 + ((row >> 1) & 1), 2 + (row >> 2))
        idx = [tuple(c) for c in fc].index(p)
        assert cols[row, 0] == ff[0, idx]


def test_kat_col2hash_two_voxels(cuda):  # test_cnn_ops.cpp:140-156
    s = SuperPsh.from_levels([PshLevel.build(VoxelSet.make(3, 8, [(3, 3, 3), (4, 3, 3)], [[1.0, 1.0]]))])
    dcols = np.zeros((27, 2), np.float32)
    dcols[13, 0], dcols[14, 0], dcols[12, 1], dcols[13, 1] = 10, 20, 40, 80
    g = _np(ops.col2hash(_dev(dcols), s, s, ConvSpec(3, 1, 0, 1, 1)))
    assert g[0, 0] == 50.0 and g[0, 1] == 100.0


def test_kat_delta_kernel_and_all_ones(cuda):  # test_cnn_ops.cpp:196-216
    f, _ = random_pair(16, 2, seed=43)
    s = SuperPsh.from_levels(f)
    data = levels_to_arrays(f).data
    w = np.zeros((3, 81), np.float32)
    for ch in range(3):
        w[ch, ch * 27 + 13] = 1.0
    assert np.array_equal(_np(ops.conv_forward(s, _dev(data), s, _dev(w), ConvSpec(3, 1, 0, 3, 3))), data)
    s1, d1 = _single((4, 4, 4), 8, 1.75)
    out = _np(ops.conv_forward(s1, d1, s1, torch.ones((1, 27), device="cuda"), ConvSpec(3, 1, 0, 1, 1)))
    assert out[0, 0] == np.float32(1.75)


def test_kat_dw_center_tap_only(cuda):  # test_cnn_ops.cpp:248-262
    s, d = _single((4, 4, 4), 8, 3.0)
    sp = ConvSpec(3, 1, 0, 1, 2)
    w = torch.rand((2, 27), device="cuda")
    cols = ops.hash2col(s, d, s, sp)
    dout = torch.tensor([[5.0], [-2.0]], device="cuda")
    dw = _np(ops.conv_backward(dout, w, cols, s, s, sp).weights)
    for r, v in enumerate((5.0, -2.0)):
        for k in range(27):
            assert dw[r, k] == (v * 3.0 if k == 13 else 0.0)


def test_kat_zero_output_grad(cuda):  # test_cnn_ops.cpp:236-246
    f, _ = random_pair(16, 1, seed=51)
    s = SuperPsh.from_levels(f)
    sp = ConvSpec(3, 1, 0, 3, 4)
    d = _dev(levels_to_arrays(f).data)
    cols = ops.hash2col(s, d, s, sp)
    g = ops.conv_backward(torch.zeros((4, s.total_columns()), device="cuda"), torch.rand((4, 81), device="cuda"),
                          cols, s, s, sp)
    assert not _np(g.weights).any() and not _np(g.input).any()


def test_kat_pools_over_block_1_to_8(cuda):  # test_cnn_ops.cpp:308-344
    coords = [(x, y, z) for z in (4, 5) for y in (4, 5) for x in (4, 5)]
    fs = VoxelSet.make(3, 8, coords, [list(range(1, 9))])
    fine = SuperPsh.from_levels([PshLevel.build(fs)])
    coarse = SuperPsh.from_levels([PshLevel.build(fs.coarsen())])
    sp = ConvSpec(2, 2, 0, 1, 1)
    d = _dev(fs.arrays()[1])
    mp = ops.max_pool(fine, d, coarse, sp)
    assert _np(mp.output)[0, 0] == 8.0 and _np(mp.switches)[0, 0] == 7
    assert _np(ops.avg_pool(fine, d, coarse, sp))[0, 0] == np.float32(36.0 / 8.0)
    one = VoxelSet.make(3, 8, [(4, 4, 4)], [[-3.5]])
    f1, c1 = SuperPsh.from_levels([PshLevel.build(one)]), SuperPsh.from_levels([PshLevel.build(one.coarsen())])
    m1 = ops.max_pool(f1, torch.tensor([[-3.5]], device="cuda"), c1, sp)
    assert _np(m1.output)[0, 0] == -3.5 and _np(m1.switches)[0, 0] == 0


def test_kat_unpools(cuda):  # test_cnn_ops.cpp:373-400, 446-468
    one = VoxelSet.make(3, 8, [(5, 2, 7)], [[4.25]])
    f1, c1 = SuperPsh.from_levels([PshLevel.build(one)]), SuperPsh.from_levels([PshLevel.build(one.coarsen())])
    sp = ConvSpec(2, 2, 0, 1, 1)
    d = torch.tensor([[4.25]], device="cuda")
    mp = ops.max_pool(f1, d, c1, sp)
    assert np.array_equal(_np(ops.max_unpool(mp.output, mp.switches, f1, c1, sp)), np.array([[4.25]], np.float32))
    cube = VoxelSet.make(3, 8, [(x, y, z) for z in (0, 1) for y in (0, 1) for x in (0, 1)], [[0.0] * 8])
    fc, cc = SuperPsh.from_levels([PshLevel.build(cube)]), SuperPsh.from_levels([PshLevel.build(cube.coarsen())])
    out = _np(ops.avg_unpool(torch.tensor([[8.0]], device="cuda"), fc, cc, sp))
    assert np.allclose(out, 1.0)
    cube2 = VoxelSet.make(3, 8, [(x, y, z) for z in (2, 3) for y in (2, 3) for x in (2, 3)], [[0.0] * 8])
    f2, c2 = SuperPsh.from_levels([PshLevel.build(cube2)]), SuperPsh.from_levels([PshLevel.build(cube2.coarsen())])
    dc = _np(ops.deconv_forward(c2, torch.tensor([[6.5]], device="cuda"), f2, torch.ones((1, 8), device="cuda"), sp))
    assert np.array_equal(dc, np.full((1, 8), 6.5, np.float32))


def test_errors_mirror_reference_messages(cuda):
    f, c = random_pair(16, 1, seed=97)
    f2, _ = random_pair(16, 2, seed=98)
    fine, coarse, two = SuperPsh.from_levels(f), SuperPsh.from_levels(c), SuperPsh.from_levels(f2)
    d = _dev(levels_to_arrays(f).data)
    sp = ConvSpec(2, 2, 0, 3, 3)
    mp = ops.max_pool(fine, d, coarse, sp)
    sw = mp.switches.clone()
    sw[0, 0] = 8  # F^3 == 8 is out of range (test_cnn_ops.cpp:436-444)
    with pytest.raises(ValueError, match="unpool: switch index out of range"):
        ops.max_unpool(mp.output, sw, fine, coarse, sp)
    with pytest.raises(ValueError, match="batch size mismatch"):
        ops.hash2col(fine, d, two, ConvSpec(3, 1, 0, 3, 3))
    with pytest.raises(ValueError, match="stride-1 fields need an odd kernel size"):
        ops.hash2col(fine, d, fine, ConvSpec(2, 1, 0, 3, 3))
    with pytest.raises(ValueError, match="stride-1 ops keep the level fixed"):
        ops.hash2col(fine, d, coarse, ConvSpec(3, 1, 0, 3, 3))
    with pytest.raises(ValueError, match="input resolution must be output resolution \\* stride"):
        ops.hash2col(fine, d, fine, ConvSpec(2, 2, 0, 3, 3))
    with pytest.raises(ValueError, match="bad conv spec"):
        ops.hash2col(fine, d, fine, ConvSpec(0, 1, 0, 3, 3))
    with pytest.raises(ValueError, match="hash2col: input data shape mismatch"):
        ops.hash2col(fine, d[:2], fine, ConvSpec(3, 1, 0, 3, 3))
    with pytest.raises(ValueError, match="pooling requires stride >= 2"):
        ops.max_pool(fine, d, fine, ConvSpec(3, 1, 0, 3, 3))
    with pytest.raises(ValueError, match="conv_forward: weight shape mismatch"):
        ops.conv_forward(fine, d, fine, torch.ones((4, 80), device="cuda"), ConvSpec(3, 1, 0, 3, 4))
    with pytest.raises(ValueError, match="col2hash: column gradient shape mismatch"):
        ops.col2hash(torch.ones((80, fine.total_columns()), device="cuda"), fine, fine, ConvSpec(3, 1, 0, 3, 3))


# ---------------------------------------------------------------- full-size properties (256^3, b=8)
@pytest.fixture(scope="module")
def shell256(cuda):
    f, c = shell_pair(256, 8)
    return SuperPsh.from_levels(f), SuperPsh.from_levels(c)


def test_full_size_pool_unpool_idempotence(shell256):
    """pool(unpool(pool(x))) == pool(x) at BASELINE config 4 size (test_cnn_ops.cpp:402-410).
    The property needs non-negative inputs (unpool zero-fills the other children), which
    is what the net feeds max-pool: post-ReLU activations (net.cpp:207-213)."""
    fine, coarse = shell256
    assert fine.total_columns() == 8 * 228296
    sp = ConvSpec(2, 2, 0, 16, 16)
    x = torch.rand((16, fine.total_columns()), device="cuda") + 1e-3
    once = ops.max_pool(fine, x, coarse, sp)
    back = ops.max_unpool(once.output, once.switches, fine, coarse, sp)
    twice = ops.max_pool(fine, back, coarse, sp)
    assert torch.equal(twice.output, once.output)
    assert torch.equal(twice.switches, once.switches)
    # the restored field holds exactly one non-zero per (channel, coarse voxel)
    assert int((back != 0).sum()) == int((once.switches >= 0).sum())


def test_full_size_delta_kernel_and_adjoint(shell256):
    fine, _ = shell256
    C = 4
    sp = ConvSpec(3, 1, 0, C, C)
    x = torch.rand((C, fine.total_columns()), device="cuda") * 2 - 1
    w = torch.zeros((C, C * 27), device="cuda")
    for ch in range(C):
        w[ch, ch * 27 + 13] = 1.0
    assert torch.equal(ops.conv_forward(fine, x, fine, w, sp), x)
    cols = ops.hash2col(fine, x, fine, sp)
    g = torch.Generator(device="cuda").manual_seed(13)
    y = torch.rand(cols.shape, device="cuda", generator=g) * 2 - 1
    lhs = torch.dot(cols.double().flatten(), y.double().flatten())
    rhs = torch.dot(x.double().flatten(), ops.col2hash(y, fine, fine, sp).double().flatten())
    # col2hash rounds its fp32 sums (<= 27 terms each): bound the difference by the dot
    # product's condition, sum |cols * y| (7.4M random-sign terms cancel to |lhs| ~ 40, so a
    # bound relative to |lhs| would only measure the cancellation, not the operator).
    scale = float(torch.dot(cols.double().abs().flatten(), y.double().abs().flatten()))
    assert abs(float(lhs - rhs)) <= 1e-6 * scale


def test_full_size_field_map_symmetry(shell256):
    """Stride-1 neighbourhoods are symmetric: map[o, t] = g  <=>  map[g, 26 - t] = o."""
    fine, _ = shell256
    m = ops.field_map(fine, fine, ConvSpec(3, 1, 0, 1, 1)).long()
    n = m.shape[0]
    o = torch.arange(n, device="cuda").unsqueeze(1).expand(n, 27)
    t = torch.arange(27, device="cuda").unsqueeze(0).expand(n, 27)
    hit = m >= 0
    back = m.clamp(min=0)[hit], (26 - t)[hit]
    assert torch.equal(m[back[0], back[1]], o[hit])
    assert torch.equal(m[:, 13], torch.arange(n, device="cuda"))  # centre tap is the voxel itself


# ---------------------------------------------------------------- dense-oracle equivalence
def test_hash_conv_equals_dense_conv3d(cuda):
    """test_cnn_ops.cpp:99-117 in spirit, independent of every oracle in this repo: on random
    sparse sets the hash convolution equals a dense 3-D cross-correlation (zero padding) of the
    densified grid at the occupied voxels — fp64 through the reference-layout path (<= 1e-12)
    and bf16-quantised operands through the native tcgen05 path (fp32 accumulation, <= 1e-5)."""
    import torch.nn.functional as F
    from paper_1803_11385_b200 import conv as nconv
    res, cin, cout = 16, 8, 16
    rng = np.random.default_rng(21)
    levels, coords_all = [], []
    for k in range(2):
        flat = rng.choice(res ** 3, size=300 + 150 * k, replace=False)
        c = np.stack([flat % res, (flat // res) % res, flat // (res * res)], 1).astype(np.int32)
        levels.append(PshLevel.build(VoxelSet.make(3, res, c, np.zeros((1, len(c)), np.float32)), 5 + k))
        coords_all.append(c)
    s = SuperPsh.from_levels(levels)
    n = s.total_columns()
    x = rng.uniform(-1, 1, (cin, n))
    w = rng.uniform(-1, 1, (cout, cin * 27))
    spec = ConvSpec(3, 1, 0, cin, cout)
    y_hash = _np(ops.conv_forward(s, _dev(x), s, _dev(w), spec))  # fp64 path
    xb = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    wb = torch.from_numpy(w).to(torch.bfloat16).double().numpy()
    fm = nconv.field_map_native(s, s, spec)
    y_nat = nconv.gather_gemm(fm, _dev(xb.T.copy()).to(torch.bfloat16), nconv.pack_weights(_dev(wb).float(), cout, cin, 27),
                              cout, torch.float32).double().cpu().numpy().T
    for k, c in enumerate(coords_all):
        q = np.concatenate([np.full((len(c), 1), k + 1), c], 1).astype(np.int32)
        cols = _np(ops.locate(s, _dev(q))).astype(np.int64)
        assert (cols >= 0).all()
        for xs, ws, got, tol in ((x, w, y_hash, 1e-12), (xb, wb, y_nat, 1e-5)):
            grid = torch.zeros((1, cin, res, res, res), dtype=torch.float64)
            grid[0, :, c[:, 2], c[:, 1], c[:, 0]] = torch.from_numpy(xs[:, cols])
            dense = F.conv3d(grid, torch.from_numpy(ws).view(cout, cin, 3, 3, 3), padding=1)[0]
            want = dense[:, c[:, 2], c[:, 1], c[:, 0]].numpy()
            err = np.linalg.norm(got[:, cols] - want) / np.linalg.norm(want)
            assert err <= tol, (k, tol, err)


# ---------------------------------------------------------------- 2-D structures (dim = 2)
def _random_pair_2d(res, models, seed, n_lo=60, n_hi=200):
    from paper_1803_11385_b200.psh import mix_seed
    rng = np.random.default_rng(seed)
    fine, coarse = [], []
    for k in range(models):
        n = int(rng.integers(n_lo, n_hi + 1))
        flat = rng.choice(res * res, size=n, replace=False)
        coords = np.zeros((n, 3), np.int32)
        coords[:, 0], coords[:, 1] = flat % res, flat // res
        s = VoxelSet.make(2, res, coords, rng.uniform(-1, 1, (3, n)).astype(np.float32))
        fine.append(PshLevel.build(s, mix_seed(seed, 20 + k)))
        coarse.append(PshLevel.build(s.coarsen(), mix_seed(seed, 20 + k)))
    return fine, coarse


@pytest.mark.parametrize("spec", [(3, 1, 0), (2, 2, 0), (3, 2, 0), (5, 1, 0)])
def test_2d_structures_vs_oracle(cuda, restated, spec):
    """The reference's operators take dim-2 structures too (F^2 fields, psh.hpp:21-35):
    every reference-layout operator on random 2-D batches, bit-exact vs the oracle."""
    f, c = _random_pair_2d(32, 3, seed=hash(spec) & 0xFFF)
    fa, ca = levels_to_arrays(f), levels_to_arrays(c)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    assert fine.dim == 2
    sp = ConvSpec(*spec, 4, 6)
    out_s, out_a = (fine, fa) if sp.stride == 1 else (coarse, ca)
    rng = np.random.default_rng(5)
    fd = sp.kernel ** 2
    data = rng.uniform(-1, 1, (4, fa.total_columns())).astype(np.float32)
    w = rng.uniform(-1, 1, (6, 4 * fd)).astype(np.float32)
    dout = rng.uniform(-1, 1, (6, out_a.total_columns())).astype(np.float32)
    assert np.array_equal(_np(ops.field_map(fine, out_s, sp)).astype(np.int64), restated.field_map(fa, out_a, sp))
    ocols = restated.hash2col(fa, data, out_a, sp)
    cols = ops.hash2col(fine, _dev(data), out_s, sp)
    assert np.array_equal(_np(cols), ocols)
    assert np.array_equal(_np(ops.conv_forward(fine, _dev(data), out_s, _dev(w), sp)), restated.matmul(w, ocols))
    g = ops.conv_backward(_dev(dout), _dev(w), cols, fine, out_s, sp)
    odw, odx = restated.conv_backward(dout, w, ocols, fa, out_a, sp)
    assert np.array_equal(_np(g.weights), odw) and np.array_equal(_np(g.input), odx)
    if sp.stride > 1:
        psp = ConvSpec(sp.kernel, sp.stride, sp.pad, 4, 4)
        mp = ops.max_pool(fine, _dev(data), coarse, psp)
        om, osw = restated.max_pool(fa, data, ca, psp)
        assert np.array_equal(_np(mp.output), om) and np.array_equal(_np(mp.switches), osw)
        assert np.array_equal(_np(ops.max_unpool(mp.output, mp.switches, fine, coarse, psp)),
                              restated.max_unpool(om, osw, fa, ca, psp))
        assert np.array_equal(_np(ops.avg_pool(fine, _dev(data), coarse, psp)), restated.avg_pool(fa, data, ca, psp))


def test_2d_native_conv_vs_double(cuda):
    """The fused tcgen05 path on a 2-D batch (9 taps): forward, input gradient and weight
    gradient against float64 on the same bf16-quantised operands."""
    from paper_1803_11385_b200 import conv as nconv
    f, _ = _random_pair_2d(64, 4, seed=9, n_lo=400, n_hi=900)
    s = SuperPsh.from_levels(f)
    n, cin, cout = s.total_columns(), 32, 64
    spec = ConvSpec(3, 1, 0, cin, cout)
    fm = nconv.field_map_native(s, s, spec)
    rm = ops.field_map(s, s, spec)  # row-major int32 [n][9]
    assert rm.shape == (n, 9)
    g = torch.Generator(device="cuda").manual_seed(4)
    x = (torch.rand((n, cin), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = (torch.rand((cout, cin * 9), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16).float()
    dy = (torch.rand((n, cout), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    xd = torch.cat([x.double(), torch.zeros((1, cin), dtype=torch.float64, device="cuda")])
    idx = torch.where(rm >= 0, rm.long(), torch.full_like(rm.long(), n))
    want = torch.einsum("ntc,oct->no", xd[idx], w.double().view(cout, cin, 9))
    y = nconv.gather_gemm(fm, x, nconv.pack_weights(w, cout, cin, 9), cout, torch.float32)
    assert float((y.double() - want).norm() / want.norm()) <= 1e-5
    dw = nconv.conv_dw(fm, x, dy)
    dw_want = torch.einsum("no,ntc->oct", dy.double(), xd[idx]).reshape(cout, cin * 9)
    assert float((dw.double() - dw_want).norm() / dw_want.norm()) <= 5e-5


def test_full_size_int64_index_paths(shell256):
    """C = 64 at BASELINE config 4 size: the column matrix has 27 * 64 * 1,826,368 = 3.2e9
    elements (> 2^31), so hash2col's and the contraction's 64-bit index math is exercised.
    The centre-tap identity kernel must reproduce the input exactly (EXACT math: the zero
    weights are skipped like gemm.cpp:21) and to fp32 accuracy through 3xTF32 over the
    materialised column matrix (FAST matmul). FAST conv_forward itself routes to the fused
    split-precision conv (hc_fused_route_count), whose identity error is the hi/lo split's
    representation bound, |y - x| <= 2^-17 |x| elementwise."""
    fine, _ = shell256
    C = 64
    n = fine.total_columns()
    assert 27 * C * n > 2 ** 31
    sp = ConvSpec(3, 1, 0, C, C)
    g = torch.Generator(device="cuda").manual_seed(17)
    x = torch.rand((C, n), device="cuda", generator=g) * 2 - 1
    w = torch.zeros((C, C * 27), device="cuda")
    w.view(C, C, 27)[torch.arange(C), torch.arange(C), 13] = 1.0
    assert torch.equal(ops.conv_forward(fine, x, fine, w, sp), x)
    from paper_1803_11385_b200._lib import lib
    with ops.math_mode("fast"):
        cols = ops.hash2col(fine, x, fine, sp)
        y = ops.matmul(w, cols)  # 3xTF32 over the 3.2e9-element column matrix
        del cols
        routed = lib.hc_fused_route_count()
        yf = ops.conv_forward(fine, x, fine, w, sp)
        assert lib.hc_fused_route_count() == routed + 1
    assert float((y - x).abs().max()) <= 1e-6
    assert bool(((yf - x).abs() <= 2.0 ** -17 * x.abs()).all())


def test_split_super_round_trip(cuda):
    """psh_batch.cpp:80-102 split_super: the device super-PSH splits back into the levels it
    was built from (tables and data rows), and rebuilding from the split levels reproduces
    the super-PSH's arrays."""
    f, _ = random_pair(16, 3, seed=41)
    s = SuperPsh.from_levels(f)
    data = torch.rand((3, s.total_columns()), device="cuda")
    parts = s.split(data)
    assert len(parts) == 3
    acc = s.download().data_acc
    for k, (orig, got) in enumerate(zip(f, parts)):
        assert (got.dim, got.resolution, got.n, got.hash_dim, got.offset_dim) == \
            (orig.dim, orig.resolution, orig.n, orig.hash_dim, orig.offset_dim)
        ho, oo, to, _ = orig.arrays()
        hg, og, tg, dg = got.arrays()
        assert np.array_equal(ho, hg) and np.array_equal(oo, og) and np.array_equal(to, tg)
        assert np.array_equal(dg, _np(data[:, int(acc[k]):int(acc[k + 1])]))
    a, b = s.download(), SuperPsh.from_levels(parts).download()
    for name in ("hash", "offsets", "tags", "model_of_slot", "hash_acc", "offset_acc", "data_acc", "hash_dims",
                 "offset_dims"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name


def test_unpool_switch_check_is_stream_ordered(cuda):
    """The switch range check never synchronises (ops_ref.cu max_unpool): asynchronous calls
    record the failure for hc_deferred_status (cnn_ops.cpp:326-332's message), a valid call
    records nothing, and max_unpool captures into a CUDA graph."""
    f, c = random_pair(16, 1, seed=97)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    d = _dev(levels_to_arrays(f).data)
    sp = ConvSpec(2, 2, 0, 3, 3)
    mp = ops.max_pool(fine, d, coarse, sp)
    good = ops.max_unpool(mp.output, mp.switches, fine, coarse, sp, check_now=False)
    torch.cuda.synchronize()
    ops.check_deferred()  # nothing recorded
    bad = mp.switches.clone()
    bad[1, 2] = -7
    ops.max_unpool(mp.output, bad, fine, coarse, sp, check_now=False)  # returns without raising
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="unpool: switch index out of range"):
        ops.check_deferred()
    ops.check_deferred()  # the flag is cleared by the report
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ops.max_unpool(mp.output, mp.switches, fine, coarse, sp, check_now=False)  # warm-up
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = ops.max_unpool(mp.output, mp.switches, fine, coarse, sp, check_now=False)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, good)
    ops.check_deferred()


@pytest.mark.parametrize("shift", [0, 1, 3])
def test_unpool_switch_check_every_position(cuda, shift):
    """The vectorised range scan (k_check_switches) sees a bad switch in the unaligned head,
    the 16-byte body and the tail, for every out-of-range kind, and passes -1 and fd - 1."""
    f, c = random_pair(16, 2, seed=98)
    fine, coarse = SuperPsh.from_levels(f), SuperPsh.from_levels(c)
    sp = ConvSpec(2, 2, 0, 5, 5)
    d = torch.rand((5, fine.total_columns()), device="cuda")
    mp = ops.max_pool(fine, d, coarse, sp)
    n = mp.switches.numel()
    buf = torch.empty(n + shift, dtype=torch.int32, device="cuda")
    sw = buf[shift:].view_as(mp.switches)
    sw.copy_(mp.switches)
    sw.view(-1)[0], sw.view(-1)[-1] = -1, 7  # range edges are valid
    ops.max_unpool(mp.output, sw, fine, coarse, sp, check_now=False)
    torch.cuda.synchronize()
    ops.check_deferred()
    for pos in [0, 1, 2, 3, 4, n // 2, n - 5, n - 2, n - 1]:
        for badv in [8, -2, 2 ** 31 - 1, -2 ** 31]:
            sw.copy_(mp.switches)
            sw.view(-1)[pos] = badv
            ops.max_unpool(mp.output, sw, fine, coarse, sp, check_now=False)
            torch.cuda.synchronize()
            with pytest.raises(ValueError, match="unpool: switch index out of range"):
                ops.check_deferred()


def _tiled_to_rows(tiled, n, taps):
    t = tiled.data.view(-1, taps, 128).permute(0, 2, 1).reshape(-1, taps)
    return t[:n]


@pytest.mark.gpu
def _zyx_sorted_levels(res, models, seed, n_lo, n_hi):
    """Random sets whose columns are (z, y, x)-sorted like the shells'."""
    from paper_1803_11385_b200.psh import PshLevel, VoxelSet, mix_seed
    rng = np.random.default_rng(seed)
    out = []
    for k in range(models):
        n = int(rng.integers(n_lo, n_hi + 1))
        flat = np.sort(rng.choice(res ** 3, size=n, replace=False))
        coords = np.stack([flat % res, (flat // res) % res, flat // (res * res)], axis=1).astype(np.int32)
        out.append(PshLevel.build(VoxelSet.make(3, res, coords, np.zeros((1, n), np.float32)), mix_seed(seed, k)))
    return out


@pytest.mark.parametrize("case", ["random_dense", "random_sparse", "shell32x3", "edges", "sorted_dense",
                                  "sorted_sparse", "sorted_edges", "shell_two_handles"])
def test_tiled_field_map_matches_rows(cuda, restated, case):
    """The tile-major 3x3x3 map the fused conv consumes (k_field_map_tiled) equals the row-major
    map (k_field_map) and the oracle's field_map (cnn_ops.cpp:100-119) entry for entry, on
    dense random sets (x-runs across warp boundaries), sparse sets, a batched shell and a set
    whose voxels all lie on the domain faces; the last tile's padding is -1. Also on
    (z, y, x)-sorted random sets and faces (x-runs adjacent in column order, identical models
    back to back) and with separate input / output handles of one level."""
    from paper_1803_11385_b200 import conv as nconv
    s_out = None
    if case == "sorted_dense":
        f = _zyx_sorted_levels(16, 3, 41, 1500, 3000)
    elif case == "sorted_sparse":
        f = _zyx_sorted_levels(64, 4, 42, 200, 900)
    elif case == "sorted_edges":
        res = 8
        g = np.stack(np.meshgrid(np.arange(res), np.arange(res), np.arange(res), indexing="ij"), -1).reshape(-1, 3)
        g = g[(g == 0).any(1) | (g == res - 1).any(1)]
        g = g[np.lexsort((g[:, 0], g[:, 1], g[:, 2]))].astype(np.int32)
        from paper_1803_11385_b200.psh import PshLevel, VoxelSet, mix_seed
        s0 = VoxelSet.make(3, res, g, np.zeros((1, len(g)), np.float32))
        f = [PshLevel.build(s0, mix_seed(6, 1))] * 3
    elif case == "shell_two_handles":
        f, _ = shell_pair(32, 2)
        s_out = SuperPsh.from_levels(f)
    elif case == "random_dense":
        f, _ = random_pair(16, 3, seed=31, n_lo=1500, n_hi=3000)  # long x-runs, warp-boundary runs
    elif case == "random_sparse":
        f, _ = random_pair(64, 4, seed=32, n_lo=200, n_hi=900)
    elif case == "shell32x3":
        f, _ = shell_pair(32, 3)
    else:  # every voxel on the domain faces: the x-1 / x+1 columns leave the grid
        from paper_1803_11385_b200.psh import PshLevel, VoxelSet, mix_seed
        res = 8
        g = np.stack(np.meshgrid(np.arange(res), np.arange(res), np.arange(res), indexing="ij"), -1).reshape(-1, 3)
        g = g[(g == 0).any(1) | (g == res - 1).any(1)].astype(np.int32)
        s0 = VoxelSet.make(3, res, g, np.zeros((1, len(g)), np.float32))
        f = [PshLevel.build(s0, mix_seed(5, 1)), PshLevel.build(s0, mix_seed(5, 2))]
    s = SuperPsh.from_levels(f)
    so = s_out if s_out is not None else s
    n = s.total_columns()
    spec = ConvSpec(3, 1, 0, 1, 1)
    tm = nconv.field_map_native(s, so, spec, nconv.TILED)
    rows = _tiled_to_rows(tm, n, 27)
    rm = ops.field_map(s, so, spec)
    assert torch.equal(rows, rm)
    pad = tm.data.view(-1, 27, 128)[-1, :, (n % 128 or 128):]
    assert bool((pad == -1).all())
    fa = levels_to_arrays(f)
    assert np.array_equal(_np(rows).astype(np.int64), restated.field_map(fa, fa, spec))
