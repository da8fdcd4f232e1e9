"""Host-side producers of the framework (C++ in libhcb200.so): sphere shells,
coarsen, the greedy PSH builder and the .psh container — checked byte-for-byte
against the reference (golden fixtures and, where built, the reference library)."""
import numpy as np
import pytest

from helpers import GOLDEN, sha
from paper_1803_11385_b200.psh import PshLevel, VoxelSet, mix_seed, read_psh_file, write_psh_file


def test_fig2_injected_offsets_reproduce_reference_tables():
    """test_psh_core.cpp:23-75 / acceptance.cpp:71-107."""
    z = np.load(f"{GOLDEN}/fig2.npz")
    s = VoxelSet.make(2, 8, z["pixels"], z["features"])
    p = PshLevel.build(s, 0, z["offsets"], 2)
    h, o, t, d = p.arrays()
    assert (p.n, p.hash_dim, p.offset_dim) == (8, 3, 2)
    assert list(h) == [0, 3, 2, 7, 5, -1, 4, 1, 6]
    assert np.array_equal(h, z["hash"]) and np.array_equal(t, z["tags"])


def test_shell32_tables_identical_to_reference():
    z = np.load(f"{GOLDEN}/shell32.npz")
    s = VoxelSet.sphere(32, True)
    assert s.count() == int(z["n"][0]) == 3680  # SURVEY §0 probe
    assert s.coarsen().count() == int(z["n"][1]) == 896
    h, o, t, d = PshLevel.build(s, mix_seed(1, 0)).arrays()
    assert sha(h) == str(z["hash_sha"])


@pytest.mark.parametrize("res", [16, 32])
def test_builder_matches_reference_library(ref, res):
    for seed in range(4):
        rs = ref.random_set(res, 60 + 40 * seed, 500 + seed)
        vs = VoxelSet.make(3, res, rs.coords, rs.features)
        for pair in ((vs, rs), (vs.coarsen(), ref.coarsen(rs))):
            ours, theirs = PshLevel.build(pair[0], seed), ref.build_psh(pair[1], seed)
            h, o, t, _ = ours.arrays()
            assert (ours.hash_dim, ours.offset_dim) == (theirs.hash_dim, theirs.offset_dim)
            assert np.array_equal(h, theirs.hash) and np.array_equal(o, theirs.offsets)
            assert np.array_equal(t, theirs.tags)
            assert theirs.validate(pair[1]) == 0


def test_shell64_matches_reference_library(ref):
    rs, vs = ref.sphere_set(64), VoxelSet.sphere(64)
    c, f = vs.arrays()
    assert np.array_equal(c, rs.coords) and np.array_equal(f, rs.features)
    h, o, t, _ = PshLevel.build(vs, 7).arrays()
    theirs = ref.build_psh(rs, 7)
    assert np.array_equal(h, theirs.hash) and np.array_equal(o, theirs.offsets) and np.array_equal(t, theirs.tags)


def test_psh_file_round_trip(tmp_path, ref):
    s = VoxelSet.sphere(16)
    levels = [PshLevel.build(s, 1), PshLevel.build(s.coarsen(), 2)]
    path = str(tmp_path / "a.psh")
    write_psh_file(path, levels)
    back = read_psh_file(path)
    for a, b in zip(levels, back):
        for x, y in zip(a.arrays(), b.arrays()):
            assert np.array_equal(x, y)
    # the reference reader accepts our container and vice versa (psh_io.cpp:45-90)
    theirs = ref.read_psh_file(path)
    assert np.array_equal(theirs[0].hash, levels[0].arrays()[0])
    path2 = str(tmp_path / "b.psh")
    ref.write_psh_file(path2, theirs)
    assert open(path, "rb").read() == open(path2, "rb").read()


def test_voxel_set_errors_mirror_reference():
    with pytest.raises(ValueError, match="resolution must be a power of two"):
        VoxelSet.make(3, 12, [[0, 0, 0]], [[1.0]])
    with pytest.raises(ValueError, match="duplicate voxel coordinate"):
        VoxelSet.make(3, 8, [[1, 1, 1], [1, 1, 1]], [[1.0, 2.0]])
    with pytest.raises(ValueError, match="voxel coordinate out of range"):
        VoxelSet.make(3, 8, [[8, 0, 0]], [[1.0]])
    with pytest.raises(ValueError, match="coarsen requires resolution >= 8"):
        VoxelSet.make(3, 4, [[0, 0, 0]], [[1.0]]).coarsen()
    with pytest.raises(RuntimeError, match="not a .psh container"):
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".psh") as f:
            f.write(b"nope")
            f.flush()
            read_psh_file(f.name)


def test_mix_seed_matches_reference():
    from oracle.oracle import mix_seed as py_mix
    for s, i in [(0, 0), (1, 5), (2**63 + 7, 123456)]:
        assert mix_seed(s, i) == py_mix(s, i)
