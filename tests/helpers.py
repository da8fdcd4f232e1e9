"""Shared test helpers: golden-fixture loading and seeded instance builders."""
from __future__ import annotations

import glob
import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_KEYS = ("hash", "offsets", "tags", "model_of_slot", "hash_acc", "offset_acc", "data_acc", "hash_dims",
         "offset_dims")


class Arrays:
    """SuperPsh-like bag of host arrays (accepted by oracle.Restated, oracle.Ref.super_from
    and paper_1803_11385_b200.psh.SuperPsh.from_host)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    def total_columns(self) -> int:
        return int(self.data_acc[self.batch])

    def total_slots(self) -> int:
        return int(self.hash_acc[self.batch])


def super_from_npz(z, prefix: str) -> Arrays:
    dim, res, batch = (int(x) for x in z[f"{prefix}_meta"])
    return Arrays(dim=dim, resolution=res, batch=batch, data=None, **{k: z[f"{prefix}_{k}"] for k in _KEYS})


def golden_instances():
    return sorted(glob.glob(os.path.join(GOLDEN, "inst_*.npz")))


def load_instance(path: str):
    z = np.load(path)
    return z, super_from_npz(z, "fine"), super_from_npz(z, "coarse")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def levels_to_arrays(levels) -> Arrays:
    """Concatenate product PshLevels on the host exactly like psh_batch.cpp:8-54."""
    dim, res = levels[0].dim, levels[0].resolution
    hs, os_, ts, mos, ds = [], [], [], [], []
    hacc, oacc, dacc, hd, od = [0], [0], [0], [], []
    for k, l in enumerate(levels):
        h, o, t, d = l.arrays()
        hs.append(h)
        os_.append(o)
        ts.append(t)
        ds.append(d)
        mos.append(np.full(h.size, k + 1, np.int32))
        hacc.append(hacc[-1] + h.size)
        oacc.append(oacc[-1] + l.offset_cells())
        dacc.append(dacc[-1] + l.n)
        hd.append(l.hash_dim)
        od.append(l.offset_dim)
    return Arrays(dim=dim, resolution=res, batch=len(levels), hash=np.concatenate(hs), offsets=np.concatenate(os_),
                  tags=np.concatenate(ts), model_of_slot=np.concatenate(mos), hash_acc=np.array(hacc, np.int64),
                  offset_acc=np.array(oacc, np.int64), data_acc=np.array(dacc, np.int64),
                  hash_dims=np.array(hd, np.int32), offset_dims=np.array(od, np.int32),
                  data=np.concatenate(ds, axis=1))


def random_pair(res: int, models: int, seed: int, n_lo: int = 50, n_hi: int = 250):
    """A fine/coarse batch built with the product's own host builder (byte-identical
    to the reference builder), like test_cnn_ops.cpp:27-43 make_fixture."""
    from paper_1803_11385_b200.psh import PshLevel, VoxelSet, mix_seed
    rng = np.random.default_rng(seed)
    fine, coarse = [], []
    for k in range(models):
        n = int(rng.integers(n_lo, n_hi + 1))
        flat = rng.choice(res ** 3, size=n, replace=False)
        coords = np.stack([flat % res, (flat // res) % res, flat // (res * res)], axis=1).astype(np.int32)
        feats = rng.uniform(-1, 1, size=(3, n)).astype(np.float32)
        s = VoxelSet.make(3, res, coords, feats)
        fine.append(PshLevel.build(s, mix_seed(seed, 20 + k)))
        coarse.append(PshLevel.build(s.coarsen(), mix_seed(seed, 20 + k)))
    return fine, coarse


def shell_pair(res: int, batch: int):
    """Synthetic shell (bench.cpp:33-77) pyramid level 0/1, replicated `batch` times."""
    from paper_1803_11385_b200.psh import PshLevel, VoxelSet, mix_seed
    s = VoxelSet.sphere(res, True)
    f = PshLevel.build(s, mix_seed(1, 0))
    c = PshLevel.build(s.coarsen(), mix_seed(1, 1))
    return [f] * batch, [c] * batch


def rel_fro(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
