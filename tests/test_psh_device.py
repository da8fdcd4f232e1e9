"""GPU perfect-spatial-hash construction (csrc/psh_build.cu).

The device builder keeps the reference's sizing and lookup semantics (psh.cpp:170-227)
but searches offsets in parallel, so its tables are a different perfect hash of the same
set. Checked here: perfection (every voxel in exactly one slot, under its own tag; every
other slot redundant, psh_core invariants of test_psh_core.cpp), identical m_bar, and
identical lookups — the K0 field map and hash2col through the GPU-built tables equal those
through the reference-identical host builder's tables, bit for bit."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1803_11385_b200 import ops  # noqa: E402
from paper_1803_11385_b200.ops import ConvSpec  # noqa: E402
from paper_1803_11385_b200.psh import PshLevel, SuperPsh, VoxelSet  # noqa: E402


def _flat(v, e, dim):  # types.hpp:57-61, x fastest
    return v[:, 0] + e * (v[:, 1] + (e * v[:, 2] if dim == 3 else 0))


def _check_perfect(level: PshLevel, coords: np.ndarray):
    h, o, t, _ = level.arrays()
    dim, m, r, n = level.dim, level.hash_dim, level.offset_dim, level.n
    p = coords.astype(np.int64)[:, :dim]
    cell = _flat(p % r, r, dim)
    off = o.reshape(-1, dim)[cell].astype(np.int64)
    slot = _flat((p % m + off) % m, m, dim)
    assert np.array_equal(h[slot], np.arange(n)), "voxel i must sit in its own slot"
    assert np.array_equal(t.reshape(-1, dim)[slot], p.astype(np.uint16)), "tags = coordinates"
    free = np.ones(h.size, bool)
    free[slot] = False
    assert (h[free] == -1).all() and (t.reshape(-1, dim)[free] == 0xFFFF).all(), "other slots redundant"


@pytest.mark.parametrize("res,n,dim", [(16, 300, 3), (32, 3000, 3), (64, 20000, 3), (64, 1500, 2), (128, 9000, 2)])
def test_device_psh_is_perfect(cuda, res, n, dim):
    rng = np.random.default_rng(res + n + dim)
    flat = rng.choice(res ** dim, size=n, replace=False)
    coords = np.zeros((n, 3), np.int32)
    coords[:, 0], coords[:, 1] = flat % res, (flat // res) % res
    if dim == 3:
        coords[:, 2] = flat // (res * res)
    s = VoxelSet.make(dim, res, coords, np.zeros((1, n), np.float32))  # n x 3, z = 0 for dim 2
    cpu, gpu = PshLevel.build(s, 5), PshLevel.build_device(s, 5)
    assert gpu.hash_dim == cpu.hash_dim and gpu.n == cpu.n
    sc, _ = s.arrays()
    _check_perfect(gpu, sc)


@pytest.mark.parametrize("res", [32, 128])
def test_device_psh_lookups_equal_reference_tables(cuda, res):
    s = VoxelSet.sphere(res, True)
    cpu, gpu = PshLevel.build(s, 1), PshLevel.build_device(s, 1)
    sc, _ = s.arrays()
    _check_perfect(gpu, sc)
    a, b = SuperPsh.from_levels([cpu] * 2), SuperPsh.from_levels([gpu] * 2)
    spec = ConvSpec(3, 1, 0, 4, 4)
    assert torch.equal(ops.field_map(a, a, spec), ops.field_map(b, b, spec))
    x = torch.rand((4, a.total_columns()), device="cuda")
    assert torch.equal(ops.hash2col(a, x, a, spec), ops.hash2col(b, x, b, spec))
