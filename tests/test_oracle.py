"""Pin the CPU oracle (oracle/hc_oracle.c) against the reference's golden fixtures
and, where the reference library is built, against the reference itself."""
import numpy as np
import pytest

from helpers import GOLDEN, golden_instances, load_instance, sha


@pytest.mark.parametrize("path", golden_instances(), ids=lambda p: p.split("/")[-1])
def test_restatement_matches_golden(restated, path):
    z, fine, coarse = load_instance(path)
    spec = tuple(int(x) for x in z["spec"])
    dc_spec = tuple(int(x) for x in z["dc_spec"])
    pool = tuple(int(x) for x in z["pool_spec"])
    out_s = fine if spec[1] == 1 else coarse
    R = restated
    cols = R.hash2col(fine, z["data"], out_s, spec)
    assert sha(cols) == str(z["cols_sha"])
    conv = R.matmul(z["w"], cols)
    assert np.array_equal(conv, z["conv_out"])
    dw, dx = R.conv_backward(z["dout"], z["w"], cols, fine, out_s, spec)
    assert np.array_equal(dw, z["dw"]) and np.array_equal(dx, z["dx"])
    mp, sw = R.max_pool(fine, z["data"], coarse, pool)
    assert np.array_equal(mp, z["mp"]) and np.array_equal(sw, z["sw"])
    assert np.array_equal(R.avg_pool(fine, z["data"], coarse, pool), z["ap"])
    assert np.array_equal(R.max_unpool(mp, sw, fine, coarse, pool), z["max_restored"])
    assert np.array_equal(R.avg_unpool(z["coarse_vals"], fine, coarse, pool), z["avg_restored"])
    assert np.array_equal(R.deconv_forward(coarse, z["dc_in"], fine, z["dc_w"], dc_spec), z["dc_out"])
    bdw, bdx = R.deconv_backward(z["data"], z["dc_w"], z["dc_in"], coarse, fine, dc_spec)
    assert np.array_equal(bdw, z["dcb_dw"]) and np.array_equal(bdx, z["dcb_dx"])
    assert np.array_equal(R.col2hash(z["y"], fine, out_s, spec), z["c2h"])
    # double instantiation
    f64 = np.float64
    cols64 = R.hash2col(fine, z["data"].astype(f64), out_s, spec, f64)
    assert np.array_equal(R.matmul(z["w"].astype(f64), cols64, f64), z["conv64"])
    dw64, dx64 = R.conv_backward(z["dout"].astype(f64), z["w"].astype(f64), cols64, fine, out_s, spec, f64)
    assert np.array_equal(dw64, z["dw64"]) and np.array_equal(dx64, z["dx64"])


def test_restated_locate_fig2(restated):
    """test_psh_core.cpp:23-75 worked example: (3,1) -> slot (1,0) -> data index 3."""
    from helpers import Arrays
    z = np.load(f"{GOLDEN}/fig2.npz")
    n, m, r, slot, idx = (int(x) for x in z["meta"])
    assert (n, m, r, slot, idx) == (8, 3, 2, 1, 3)
    assert list(z["hash"]) == [0, 3, 2, 7, 5, -1, 4, 1, 6]  # test_psh_core.cpp:71
    s = Arrays(dim=2, resolution=8, batch=1, hash=z["hash"], offsets=z["offsets"], tags=z["tags"],
               model_of_slot=np.ones(9, np.int32), hash_acc=np.array([0, 9]), offset_acc=np.array([0, 4]),
               data_acc=np.array([0, 8]), hash_dims=np.array([3], np.int32), offset_dims=np.array([2], np.int32))
    for i, p in enumerate(z["pixels"]):
        assert restated.locate(s, 1, p) == i
    occupied = {tuple(p) for p in z["pixels"][:, :2]}
    for y in range(5):
        for x in range(7):
            if (x, y) not in occupied:
                assert restated.locate(s, 1, (x, y, 0)) == -1


def _random_instance(ref, trial):
    inst = ref.make_instance(trial)
    return inst["fine"], inst["coarse"], inst["spec"]


@pytest.mark.parametrize("trial", range(12, 36))
def test_restatement_matches_reference_library(ref, restated, trial):
    """Bit-exact against the compiled reference on instances beyond the golden set."""
    fine, coarse, spec = _random_instance(ref, trial)
    out_s = fine if spec[1] == 1 else coarse
    c_in, c_out = spec[3], spec[4]
    fd = spec[0] ** 3
    data = ref.random_matrix(c_in, fine.total_columns(), trial + 1)
    w = ref.random_matrix(c_out, c_in * fd, trial + 2)
    dout = ref.random_matrix(c_out, out_s.total_columns(), trial + 3)
    cols = ref.hash2col(fine, data, out_s, spec)
    assert np.array_equal(restated.hash2col(fine, data, out_s, spec), cols)
    assert np.array_equal(restated.matmul(w, cols), ref.matmul(w, cols))
    a = ref.conv_backward(dout, w, cols, fine, out_s, spec)
    b = restated.conv_backward(dout, w, cols, fine, out_s, spec)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    pool = (2, 2, 0, c_in, c_in)
    mp = ref.max_pool(fine, data, coarse, pool)
    mq = restated.max_pool(fine, data, coarse, pool)
    assert np.array_equal(mp[0], mq[0]) and np.array_equal(mp[1], mq[1])
    assert np.array_equal(ref.max_unpool(*mp, fine, coarse, pool), restated.max_unpool(*mq, fine, coarse, pool))
    fm = restated.field_map(fine, out_s, spec)
    # field map equals reference locate on every tap (spot check 64 columns)
    cols_info = {}
    for slot in range(out_s.total_slots()):
        idx = out_s.hash[slot]
        if idx >= 0:
            v = out_s.model_of_slot[slot]
            cols_info[int(out_s.data_acc[v - 1] + idx)] = (v, out_s.tags[3 * slot:3 * slot + 3])
    F, S, P = spec[0], spec[1], spec[2]
    for col in list(cols_info)[:64]:
        v, p = cols_info[col]
        base = [int(c) - (F - 1) // 2 if S == 1 else int(c) * S - P for c in p]
        row = 0
        for dz in range(F):
            for dy in range(F):
                for dx in range(F):
                    q = (base[0] + dx, base[1] + dy, base[2] + dz)
                    inside = all(0 <= c < fine.resolution for c in q)
                    want = fine.locate(v, q) if inside else -1
                    assert fm[col, row] == want
                    row += 1
