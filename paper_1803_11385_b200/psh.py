"""Hashed storage: voxel sets, PSH levels (host, C++) and the device super-PSH.

Mirrors the reference's L1/L2 surface (voxel.hpp, psh.hpp, psh_io.hpp,
psh_batch.hpp, net.hpp:build_pyramid/build_batch) over the C ABI. Tables are
produced by the library's own C++ builder (byte-identical to the reference's
for the same set and seed) and concatenated straight into device memory.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def mix_seed(seed: int, item: int) -> int:
    """rng.hpp:53-58 (splitmix64 finaliser)."""
    return int(lib.hc_mix_seed(seed & (2**64 - 1), item & (2**64 - 1)))


class VoxelSet:
    """voxel.hpp:16-25 SparseVoxelSet (host), canonical (z,y,x) order."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        info = np.zeros(4, np.int64)
        check(lib.hc_voxel_set_info(self._h, _ptr(info)))
        self.dim, self.resolution, self.n, self.channels = (int(x) for x in info)

    @classmethod
    def sphere(cls, resolution: int, shell: bool = True) -> "VoxelSet":
        """bench.cpp:33-77 sphere_voxels."""
        h = C.c_void_p()
        check(lib.hc_sphere_voxels(resolution, int(shell), C.byref(h)))
        return cls(h)

    @classmethod
    def make(cls, dim: int, resolution: int, coords, features) -> "VoxelSet":
        """voxel.cpp:76-110 make_sparse_set; coords n x 3 (x,y,z), features C x n."""
        coords = np.ascontiguousarray(coords, np.int32).reshape(-1, 3)
        features = np.ascontiguousarray(features, np.float32).reshape(-1, coords.shape[0])
        h = C.c_void_p()
        check(lib.hc_voxel_set_make(dim, resolution, coords.shape[0], _ptr(coords), features.shape[0],
                                    _ptr(features), C.byref(h)))
        return cls(h)

    def coarsen(self) -> "VoxelSet":
        """voxel.cpp:218-268 coarsen."""
        h = C.c_void_p()
        check(lib.hc_coarsen(self._h, C.byref(h)))
        return VoxelSet(h)

    def count(self) -> int:
        return self.n

    def arrays(self):
        coords = np.zeros((self.n, 3), np.int32)
        feats = np.zeros((self.channels, self.n), np.float32)
        check(lib.hc_voxel_set_copy(self._h, _ptr(coords), _ptr(feats)))
        return coords, feats

    def __del__(self):
        if getattr(self, "_h", None):
            lib.hc_voxel_set_free(self._h)
            self._h = None


class PshLevel:
    """psh.hpp:21-35 PshLevel (host): H, Phi, T and the data array."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        info = np.zeros(6, np.int64)
        check(lib.hc_psh_level_info(self._h, _ptr(info)))
        self.dim, self.resolution, self.n, self.hash_dim, self.offset_dim, self.channels = (int(x) for x in info)

    @classmethod
    def build(cls, s: VoxelSet, seed: int = 0, injected=None, injected_dim: int = 0) -> "PshLevel":
        """psh.cpp:179-227 build_psh."""
        inj = None if injected is None else np.ascontiguousarray(injected, np.uint8)
        h = C.c_void_p()
        check(lib.hc_build_psh(s._h, seed, _ptr(inj), 0 if inj is None else inj.size, injected_dim, C.byref(h)))
        return cls(h)

    @classmethod
    def build_device(cls, s: VoxelSet, seed: int = 0) -> "PshLevel":
        """build_psh on the GPU (hc_build_psh_device): same sizing and lookups, tables found
        by a parallel search (a different valid PSH of the same set)."""
        h = C.c_void_p()
        check(lib.hc_build_psh_device(s._h, seed, C.byref(h)))
        return cls(h)

    def hash_slots(self) -> int:
        return self.hash_dim ** self.dim

    def offset_cells(self) -> int:
        return self.offset_dim ** self.dim

    def arrays(self):
        """(hash i32[m^d], offsets u8[r^d * d], tags u16[m^d * d], data f32[C x n])"""
        M, R = self.hash_slots(), self.offset_cells()
        h = np.empty(M, np.int32)
        o = np.empty(R * self.dim, np.uint8)
        t = np.empty(M * self.dim, np.uint16)
        d = np.empty((self.channels, self.n), np.float32)
        check(lib.hc_psh_level_copy(self._h, _ptr(h), _ptr(o), _ptr(t), _ptr(d)))
        return h, o, t, d

    def __del__(self):
        if getattr(self, "_h", None):
            lib.hc_psh_level_free(self._h)
            self._h = None


def write_psh_file(path: str, levels: Sequence[PshLevel]) -> None:
    """psh_io.cpp:92 write_psh_file."""
    arr = (C.c_void_p * len(levels))(*[l._h.value for l in levels])
    check(lib.hc_write_psh_file(path.encode(), arr, len(levels)))


def read_psh_file(path: str) -> List[PshLevel]:
    """psh_io.cpp:98 read_psh_file."""
    arr = (C.c_void_p * 32)()
    n = C.c_int32()
    check(lib.hc_read_psh_file(path.encode(), arr, 32, C.byref(n)))
    return [PshLevel(arr[i]) for i in range(n.value)]


def build_pyramid(finest: VoxelSet, seed: int = 1) -> List[PshLevel]:
    """net.cpp:19-32 build_pyramid: build_psh + coarsen down to resolution 4,
    level seeds mix_seed(seed, level_index)."""
    levels, cur, i = [], finest, 0
    while True:
        levels.append(PshLevel.build(cur, mix_seed(seed, i)))
        if cur.resolution == 4:
            break
        cur = cur.coarsen()
        i += 1
    return levels


@dataclass
class SuperHost:
    """psh_batch.hpp:15-38 SuperPsh arrays on the host."""

    dim: int
    resolution: int
    batch: int
    hash: np.ndarray
    offsets: np.ndarray
    tags: np.ndarray
    model_of_slot: np.ndarray
    hash_acc: np.ndarray
    offset_acc: np.ndarray
    data_acc: np.ndarray
    hash_dims: np.ndarray
    offset_dims: np.ndarray
    data: Optional[np.ndarray] = None

    def total_columns(self) -> int:
        return int(self.data_acc[self.batch])

    def total_slots(self) -> int:
        return int(self.hash_acc[self.batch])


class SuperPsh:
    """Device-resident super-PSH (opaque hc_psh*). Replaces `const SuperPsh&` at the
    operator boundary; build it from PSH levels (device-side build_super) or from
    host arrays of an existing SuperPsh."""

    def __init__(self, handle, data=None):
        self._h = handle
        info = np.zeros(6, np.int64)
        check(lib.hc_psh_info(self._h, _ptr(info)))
        self.dim, self.resolution, self.batch, self.M, self.R, self.N = (int(x) for x in info)
        self.data = data  # optional D* (C x N) kept by the caller

    @staticmethod
    def _stream(stream):
        if stream is not None:
            return C.c_void_p(stream)
        try:
            import torch
            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return None

    @classmethod
    def from_levels(cls, levels: Sequence[PshLevel], stream=None) -> "SuperPsh":
        """psh_batch.cpp:8-54 build_super, concatenating straight into device memory."""
        arr = (C.c_void_p * len(levels))(*[l._h.value for l in levels])
        h = C.c_void_p()
        check(lib.hc_psh_upload_levels(arr, len(levels), C.byref(h), cls._stream(stream)))
        return cls(h)

    @classmethod
    def from_host(cls, s, stream=None) -> "SuperPsh":
        """Upload any object with the SuperPsh attributes (e.g. a reference SuperPsh)."""
        keep = dict(
            hash=np.ascontiguousarray(s.hash, np.int32), offsets=np.ascontiguousarray(s.offsets, np.uint8),
            tags=np.ascontiguousarray(s.tags, np.uint16),
            mos=None if getattr(s, "model_of_slot", None) is None else np.ascontiguousarray(s.model_of_slot, np.int32),
            hacc=np.ascontiguousarray(s.hash_acc, np.int64), oacc=np.ascontiguousarray(s.offset_acc, np.int64),
            dacc=np.ascontiguousarray(s.data_acc, np.int64), hd=np.ascontiguousarray(s.hash_dims, np.int32),
            od=np.ascontiguousarray(s.offset_dims, np.int32))
        v = _lib.SuperHostC(int(s.dim), int(s.resolution), int(s.batch), 0, _ptr(keep["hash"]),
                            _ptr(keep["offsets"]), _ptr(keep["tags"]), _ptr(keep["mos"]), _ptr(keep["hacc"]),
                            _ptr(keep["oacc"]), _ptr(keep["dacc"]), _ptr(keep["hd"]), _ptr(keep["od"]))
        h = C.c_void_p()
        check(lib.hc_psh_upload(C.byref(v), C.byref(h), cls._stream(stream)))
        return cls(h, getattr(s, "data", None))

    def total_columns(self) -> int:
        return self.N

    def total_slots(self) -> int:
        return self.M

    def download(self) -> SuperHost:
        b = self.batch
        out = SuperHost(self.dim, self.resolution, b, np.empty(self.M, np.int32),
                        np.empty(self.R * self.dim, np.uint8), np.empty(self.M * self.dim, np.uint16),
                        np.empty(self.M, np.int32), np.empty(b + 1, np.int64), np.empty(b + 1, np.int64),
                        np.empty(b + 1, np.int64), np.empty(b, np.int32), np.empty(b, np.int32))
        check(lib.hc_psh_download(self._h, *(_ptr(getattr(out, k)) for k in (
            "hash", "offsets", "tags", "model_of_slot", "hash_acc", "offset_acc", "data_acc", "hash_dims",
            "offset_dims"))))
        return out

    def split(self, data=None) -> List[PshLevel]:
        """psh_batch.cpp:80-102 split_super: one host PshLevel per model. `data`: optional
        device tensor (C x N fp32) whose columns become the levels' data arrays."""
        out = (C.c_void_p * max(self.batch, 1))()
        count = C.c_int32()
        ch, ptr = 0, None
        if data is not None:
            data = data.float().contiguous()
            ch, ptr = int(data.shape[0]), C.c_void_p(data.data_ptr())
        check(lib.hc_split_super(self._h, ptr, ch, out, self.batch, C.byref(count)))
        return [PshLevel(C.c_void_p(out[i])) for i in range(count.value)]

    def columns_ptr(self) -> int:
        """Device pointer of the int4 {x,y,z,model} column table."""
        p = C.c_void_p()
        check(lib.hc_psh_columns(self._h, C.byref(p)))
        return p.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib.hc_psh_free(self._h)
            self._h = None


def build_batch_levels(pyramids: Sequence[Sequence[PshLevel]], level: int) -> List[PshLevel]:
    """net.cpp:40-53 build_batch, one level: the level-`level` PshLevel of every model."""
    return [p[level] for p in pyramids]
