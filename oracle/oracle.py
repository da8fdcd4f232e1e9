"""TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 hot path.

Two ctypes front-ends:

* ``Restated`` — our plain-C restatement of the reference algorithm
  (oracle/hc_oracle.c, built into oracle/_build/libhc_oracle.so). This is the
  parity checker used by tests/, __graft_entry__.smoke() and bench.py's
  cpu_baseline leg. Each C function cites the reference file:line it follows.
* ``Ref`` — the unmodified reference library (/root/reference/proj/src,
  compiled by oracle/Makefile into oracle/_ref/libhcref.so) behind the flat shim
  oracle/ref_shim.cpp. Used to pin the restatement, to produce the golden
  fixtures in tests/golden/, and as the reference CPU baseline.

The product package (paper_1803_11385_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libhcref.so")
RESTATED_SO = os.path.join(HERE, "_build", "libhc_oracle.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class SuperArrays:
    """Host arrays of one super-PSH (psh_batch.hpp:15-38). ``data`` is C x N float32."""

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


class _HcoSuper(C.Structure):
    _fields_ = [("dim", C.c_int32), ("resolution", C.c_int32), ("batch", C.c_int32),
                ("reserved", C.c_int32),
                ("hash", C.c_void_p), ("offsets", C.c_void_p), ("tags", C.c_void_p),
                ("model_of_slot", C.c_void_p), ("hash_acc", C.c_void_p),
                ("offset_acc", C.c_void_p), ("data_acc", C.c_void_p),
                ("hash_dims", C.c_void_p), ("offset_dims", C.c_void_p)]


class _HcoSpec(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32),
                ("in_channels", C.c_int32), ("out_channels", C.c_int32)]


def _norm_super(s) -> SuperArrays:
    """Accept any object carrying the SuperPsh attributes; coerce dtypes."""
    return SuperArrays(
        dim=int(s.dim), resolution=int(s.resolution), batch=int(s.batch),
        hash=np.ascontiguousarray(s.hash, np.int32),
        offsets=np.ascontiguousarray(s.offsets, np.uint8),
        tags=np.ascontiguousarray(s.tags, np.uint16),
        model_of_slot=np.ascontiguousarray(s.model_of_slot, np.int32),
        hash_acc=np.ascontiguousarray(s.hash_acc, np.int64),
        offset_acc=np.ascontiguousarray(s.offset_acc, np.int64),
        data_acc=np.ascontiguousarray(s.data_acc, np.int64),
        hash_dims=np.ascontiguousarray(s.hash_dims, np.int32),
        offset_dims=np.ascontiguousarray(s.offset_dims, np.int32),
        data=None if getattr(s, "data", None) is None else np.ascontiguousarray(s.data, np.float32))


def _spec5(spec) -> tuple:
    if isinstance(spec, (tuple, list)):
        return tuple(int(x) for x in spec)
    return (int(spec.kernel), int(spec.stride), int(spec.pad), int(spec.in_channels),
            int(spec.out_channels))


def mix_seed(seed: int, item: int) -> int:
    """rng.hpp:53-58 splitmix64 finaliser (pure Python)."""
    m = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (item + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def field_volume(spec, dim: int = 3) -> int:
    return _spec5(spec)[0] ** dim


# =============================================================== restatement
class Restated:
    """ctypes front-end of oracle/_build/libhc_oracle.so (the parity checker)."""

    def __init__(self, path: str = RESTATED_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle restatement`")
        self.lib = C.CDLL(path)
        L = self.lib
        L.hco_locate.restype = C.c_int64
        L.hco_locate.argtypes = [C.POINTER(_HcoSuper), C.c_int32, C.c_int32, C.c_int32, C.c_int32]

    def _view(self, s):
        s = _norm_super(s)
        v = _HcoSuper(s.dim, s.resolution, s.batch, 0, _ptr(s.hash), _ptr(s.offsets), _ptr(s.tags),
                      _ptr(s.model_of_slot), _ptr(s.hash_acc), _ptr(s.offset_acc),
                      _ptr(s.data_acc), _ptr(s.hash_dims), _ptr(s.offset_dims))
        v._keep = s  # keep arrays alive
        return v

    @staticmethod
    def _spec(spec):
        return _HcoSpec(*_spec5(spec))

    def locate(self, s, model: int, p) -> int:
        v = self._view(s)
        return int(self.lib.hco_locate(C.byref(v), model, int(p[0]), int(p[1]), int(p[2])))

    def field_map(self, inp, out, spec) -> np.ndarray:
        vi, vo = self._view(inp), self._view(out)
        fd = field_volume(spec, vi.dim)
        m = np.empty((vo._keep.total_columns(), fd), np.int64)
        rc = self.lib.hco_field_map(C.byref(vi), C.byref(vo), self._spec(spec), _ptr(m))
        if rc:
            raise ValueError("field_map: bad structure pair / spec")
        return m

    def _t(self, dtype):
        return ("f32", np.float32) if np.dtype(dtype) == np.float32 else ("f64", np.float64)

    def hash2col(self, inp, data, out, spec, dtype=np.float32):
        suf, T = self._t(dtype)
        vi, vo = self._view(inp), self._view(out)
        k, s, p, cin, cout = _spec5(spec)
        data = np.ascontiguousarray(data, T)
        res = np.empty((cin * k ** vi.dim, vo._keep.total_columns()), T)
        rc = getattr(self.lib, f"hco_hash2col_{suf}")(C.byref(vi), _ptr(data), C.byref(vo),
                                                      self._spec(spec), _ptr(res))
        if rc:
            raise ValueError("hash2col: invalid arguments")
        return res

    def col2hash(self, g, inp, out, spec, dtype=np.float32):
        suf, T = self._t(dtype)
        vi, vo = self._view(inp), self._view(out)
        k, s, p, cin, cout = _spec5(spec)
        g = np.ascontiguousarray(g, T)
        res = np.empty((cin, vi._keep.total_columns()), T)
        rc = getattr(self.lib, f"hco_col2hash_{suf}")(_ptr(g), C.byref(vi), C.byref(vo),
                                                      self._spec(spec), _ptr(res))
        if rc:
            raise ValueError("col2hash: invalid arguments")
        return res

    def max_pool(self, inp, data, out, spec, dtype=np.float32):
        suf, T = self._t(dtype)
        vi, vo = self._view(inp), self._view(out)
        cin = _spec5(spec)[3]
        n = vo._keep.total_columns()
        res = np.empty((cin, n), T)
        sw = np.empty((cin, n), np.int32)
        rc = getattr(self.lib, f"hco_max_pool_{suf}")(C.byref(vi), _ptr(np.ascontiguousarray(data, T)),
                                                      C.byref(vo), self._spec(spec), _ptr(res), _ptr(sw))
        if rc:
            raise ValueError("max_pool: invalid arguments")
        return res, sw

    def avg_pool(self, inp, data, out, spec, dtype=np.float32):
        suf, T = self._t(dtype)
        vi, vo = self._view(inp), self._view(out)
        cin = _spec5(spec)[3]
        res = np.empty((cin, vo._keep.total_columns()), T)
        rc = getattr(self.lib, f"hco_avg_pool_{suf}")(C.byref(vi), _ptr(np.ascontiguousarray(data, T)),
                                                      C.byref(vo), self._spec(spec), _ptr(res))
        if rc:
            raise ValueError("avg_pool: invalid arguments")
        return res

    def max_unpool(self, coarse, switches, fine, cs, spec, dtype=np.float32):
        suf, T = self._t(dtype)
        vf, vc = self._view(fine), self._view(cs)
        cin = _spec5(spec)[3]
        res = np.empty((cin, vf._keep.total_columns()), T)
        rc = getattr(self.lib, f"hco_max_unpool_{suf}")(
            _ptr(np.ascontiguousarray(coarse, T)), _ptr(np.ascontiguousarray(switches, np.int32)),
            C.byref(vf), C.byref(vc), self._spec(spec), _ptr(res))
        if rc == -2:
            raise ValueError("unpool: switch index out of range")
        if rc:
            raise ValueError("max_unpool: invalid arguments")
        return res

    def avg_unpool(self, coarse, fine, cs, spec, dtype=np.float32):
        suf, T = self._t(dtype)
        vf, vc = self._view(fine), self._view(cs)
        cin = _spec5(spec)[3]
        res = np.empty((cin, vf._keep.total_columns()), T)
        rc = getattr(self.lib, f"hco_avg_unpool_{suf}")(
            _ptr(np.ascontiguousarray(coarse, T)), C.byref(vf), C.byref(vc), self._spec(spec), _ptr(res))
        if rc:
            raise ValueError("avg_unpool: invalid arguments")
        return res

    def _gemm(self, name, a, b, dtype, shape_fn):
        suf, T = self._t(dtype)
        a = np.ascontiguousarray(a, T)
        b = np.ascontiguousarray(b, T)
        out_shape, args = shape_fn(a, b)
        c = np.empty(out_shape, T)
        fn = getattr(self.lib, f"hco_{name}_{suf}")
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64]
        fn(_ptr(a), _ptr(b), _ptr(c), *args)
        return c

    def matmul(self, a, b, dtype=np.float32):  # gemm.cpp:30
        return self._gemm("matmul", a, b, dtype,
                          lambda a, b: ((a.shape[0], b.shape[1]), (a.shape[0], a.shape[1], b.shape[1])))

    def matmul_trans_a(self, a, b, dtype=np.float32):  # gemm.cpp:37
        return self._gemm("matmul_trans_a", a, b, dtype,
                          lambda a, b: ((a.shape[1], b.shape[1]), (a.shape[0], a.shape[1], b.shape[1])))

    def matmul_trans_b(self, a, b, dtype=np.float32):  # gemm.cpp:54
        return self._gemm("matmul_trans_b", a, b, dtype,
                          lambda a, b: ((a.shape[0], b.shape[0]), (a.shape[0], a.shape[1], b.shape[0])))

    # compositions, exactly as cnn_ops.cpp composes them
    def conv_forward(self, inp, data, out, w, spec, dtype=np.float32):  # cnn_ops.cpp:206-215
        return self.matmul(w, self.hash2col(inp, data, out, spec, dtype), dtype)

    def conv_backward(self, dout, w, cols, inp, out, spec, dtype=np.float32):  # cnn_ops.cpp:217-232
        dw = self.matmul_trans_b(dout, cols, dtype)
        dcols = self.matmul_trans_a(w, dout, dtype)
        return dw, self.col2hash(dcols, inp, out, spec, dtype)

    def deconv_forward(self, coarse, cdata, fine, w, spec, dtype=np.float32):  # cnn_ops.cpp:408-419
        return self.col2hash(self.matmul_trans_a(w, cdata, dtype), fine, coarse, spec, dtype)

    def deconv_backward(self, fgrad, w, cdata, coarse, fine, spec, dtype=np.float32):  # :421-435
        dcols = self.hash2col(fine, fgrad, coarse, spec, dtype)
        return self.matmul_trans_b(cdata, dcols, dtype), self.matmul(w, dcols, dtype)


# =============================================================== reference
class RefError(Exception):
    pass


class Ref:
    """ctypes front-end of the unmodified reference (oracle/_ref/libhcref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)
        L = self.lib
        for name in ("hcref_set_sphere", "hcref_set_random", "hcref_set_make", "hcref_set_coarsen",
                     "hcref_psh_build", "hcref_super_build", "hcref_super_from_arrays"):
            getattr(L, name).restype = C.c_void_p
        L.hcref_set_random.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_int, C.c_int]
        L.hcref_set_make.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
        L.hcref_set_coarsen.argtypes = [C.c_void_p]
        L.hcref_set_info.argtypes = [C.c_void_p, C.c_void_p]
        L.hcref_set_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.hcref_set_free.argtypes = [C.c_void_p]
        L.hcref_psh_build.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int64, C.c_int]
        L.hcref_psh_info.argtypes = [C.c_void_p, C.c_void_p]
        L.hcref_psh_copy.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        L.hcref_psh_validate.argtypes = [C.c_void_p, C.c_void_p]
        L.hcref_psh_query.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.hcref_psh_query.restype = C.c_int64
        L.hcref_psh_hash_slot.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.hcref_psh_hash_slot.restype = C.c_int64
        L.hcref_psh_free.argtypes = [C.c_void_p]
        L.hcref_psh_write_file.argtypes = [C.c_char_p, C.c_void_p, C.c_int]
        L.hcref_psh_read_file.argtypes = [C.c_char_p, C.c_void_p, C.c_int]
        L.hcref_super_build.argtypes = [C.c_void_p, C.c_int]
        L.hcref_super_from_arrays.argtypes = [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 9 + [C.c_int, C.c_void_p]
        L.hcref_super_info.argtypes = [C.c_void_p, C.c_void_p]
        L.hcref_super_copy.argtypes = [C.c_void_p] * 11
        L.hcref_super_free.argtypes = [C.c_void_p]
        L.hcref_locate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.hcref_locate.restype = C.c_int64
        L.hcref_random_matrix_f32.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_float, C.c_float, C.c_void_p]
        L.hcref_random_matrix_f64.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_double, C.c_double, C.c_void_p]
        L.hcref_set_threads.argtypes = [C.c_int]

    # ---------------------------------------------------------------- errors
    def _check(self, rc: int):
        if rc == 0:
            return
        buf = C.create_string_buffer(512)
        self.lib.hcref_last_error(buf, 512)
        msg = buf.value.decode()
        if rc == 1:
            raise ValueError(msg)  # std::invalid_argument
        raise RuntimeError(msg)  # std::runtime_error

    def _handle(self, h):
        if not h:
            self._check(2)
        return h

    def set_threads(self, n: int):
        self.lib.hcref_set_threads(int(n))

    def max_threads(self) -> int:
        return int(self.lib.hcref_max_threads())

    # ---------------------------------------------------------------- voxel sets
    def _set_arrays(self, h):
        info = np.zeros(4, np.int64)
        self.lib.hcref_set_info(h, _ptr(info))
        n, ch = int(info[2]), int(info[3])
        coords = np.zeros((n, 3), np.int32)
        feats = np.zeros((ch, n), np.float32)
        self.lib.hcref_set_copy(h, _ptr(coords), _ptr(feats))
        return RefSet(self, h, int(info[0]), int(info[1]), coords, feats)

    def sphere_set(self, res: int, shell: bool = True) -> "RefSet":
        return self._set_arrays(self._handle(self.lib.hcref_set_sphere(res, int(shell))))

    def random_set(self, res: int, n: int, seed: int, channels: int = 3, unit_normals: bool = True):
        return self._set_arrays(self._handle(self.lib.hcref_set_random(res, n, seed, channels, int(unit_normals))))

    def make_set(self, dim: int, res: int, coords, features) -> "RefSet":
        coords = np.ascontiguousarray(coords, np.int32).reshape(-1, 3)
        features = np.ascontiguousarray(features, np.float32)
        h = self.lib.hcref_set_make(dim, res, coords.shape[0], _ptr(coords), features.shape[0], _ptr(features))
        return self._set_arrays(self._handle(h))

    def coarsen(self, s: "RefSet") -> "RefSet":
        return self._set_arrays(self._handle(self.lib.hcref_set_coarsen(s.h)))

    # ---------------------------------------------------------------- PSH
    def build_psh(self, s: "RefSet", seed: int = 0, injected=None, injected_dim: int = 0) -> "RefPsh":
        inj = None if injected is None else np.ascontiguousarray(injected, np.uint8)
        h = self.lib.hcref_psh_build(s.h, seed, _ptr(inj), 0 if inj is None else inj.size, injected_dim)
        return RefPsh(self, self._handle(h))

    def build_super(self, levels: Sequence["RefPsh"]) -> "RefSuper":
        arr = (C.c_void_p * len(levels))(*[l.h for l in levels])
        return RefSuper(self, self._handle(self.lib.hcref_super_build(arr, len(levels))))

    def super_from(self, s) -> "RefSuper":
        """Wrap any SuperPsh-like arrays (e.g. built by the product's builder)."""
        s = _norm_super(s)
        ch = 0 if s.data is None else s.data.shape[0]
        h = self.lib.hcref_super_from_arrays(
            s.dim, s.resolution, s.batch, _ptr(s.hash), _ptr(s.offsets), _ptr(s.tags),
            _ptr(s.model_of_slot), _ptr(s.hash_acc), _ptr(s.offset_acc), _ptr(s.data_acc),
            _ptr(s.hash_dims), _ptr(s.offset_dims), ch, _ptr(s.data))
        return RefSuper(self, self._handle(h))

    def write_psh_file(self, path: str, levels: Sequence["RefPsh"]):
        arr = (C.c_void_p * len(levels))(*[l.h for l in levels])
        self._check(self.lib.hcref_psh_write_file(path.encode(), arr, len(levels)))

    def read_psh_file(self, path: str):
        arr = (C.c_void_p * 32)()
        n = self.lib.hcref_psh_read_file(path.encode(), arr, 32)
        if n < 0:
            self._check(2)
        return [RefPsh(self, arr[i]) for i in range(n)]

    def rng_draws(self, seed: int, bounds) -> list:
        """Sequential Rng(seed).uniform_int(lo, hi) draws (rng.hpp:28-37)."""
        lo = np.array([b[0] for b in bounds], np.int64)
        hi = np.array([b[1] for b in bounds], np.int64)
        out = np.zeros(len(bounds), np.int64)
        self.lib.hcref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        self.lib.hcref_rng_draws(seed, len(bounds), _ptr(lo), _ptr(hi), _ptr(out))
        return [int(x) for x in out]

    def make_instance(self, trial: int):
        """tests/acceptance.cpp:174-203 make_instance, through the reference library.
        Returns dict(sets, fine, coarse, spec, c_in, c_out, seed)."""
        seed = 90000 + trial * 17
        res = (8, 16, 32)[trial % 3]
        models = 1 + trial % 3
        # the Rng stream draws c_in, c_out, then n per model (bounds known up front)
        nhi = 400 if res == 32 else 150
        draws = self.rng_draws(seed, [(1, 8), (1, 8)] + [(20, nhi)] * models)
        c_in, c_out = draws[0], draws[1]
        spec = [(3, 1, 0), (2, 2, 0), (3, 2, 0), (2, 2, 1)][trial % 4] + (c_in, c_out)
        sets, fl, cl = [], [], []
        for k in range(models):
            s = self.random_set(res, draws[2 + k], mix_seed(seed, 10 + k))
            fl.append(self.build_psh(s, mix_seed(seed, 20 + k)))
            cl.append(self.build_psh(self.coarsen(s), mix_seed(seed, 20 + k)))
            sets.append(s)
        return dict(sets=sets, fine=self.build_super(fl), coarse=self.build_super(cl), spec=spec, c_in=c_in,
                    c_out=c_out, seed=seed)

    def random_matrix(self, rows: int, cols: int, seed: int, lo=-1.0, hi=1.0, dtype=np.float32):
        out = np.empty((rows, cols), dtype)
        if np.dtype(dtype) == np.float32:
            self.lib.hcref_random_matrix_f32(rows, cols, seed, lo, hi, _ptr(out))
        else:
            self.lib.hcref_random_matrix_f64(rows, cols, seed, lo, hi, _ptr(out))
        return out

    # ---------------------------------------------------------------- net (net.cpp)
    def net_make(self, level_max: int, classes: int, seed: int, input_channels: int = 3) -> "RefNet":
        """net.cpp:135-180 make_graph<float>."""
        L = self.lib
        L.hcref_net_make.restype = C.c_void_p
        L.hcref_net_make.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int]
        return RefNet(self, self._handle(L.hcref_net_make(level_max, classes, seed, input_channels)))

    # ---------------------------------------------------------------- ops
    @staticmethod
    def _suf(dtype):
        return ("f32", np.float32) if np.dtype(dtype) == np.float32 else ("f64", np.float64)

    @staticmethod
    def _sp(spec):
        return (C.c_int * 5)(*_spec5(spec))

    def hash2col(self, inp, data, out, spec, dtype=np.float32):
        suf, T = self._suf(dtype)
        data = np.ascontiguousarray(data, T)
        k, s, p, cin, _ = _spec5(spec)
        res = np.empty((cin * k ** inp.dim, out.total_columns()), T)
        fn = getattr(self.lib, f"hcref_hash2col_{suf}")
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(fn(inp.h, _ptr(data), data.shape[0], data.shape[1], out.h, self._sp(spec), _ptr(res)))
        return res

    def serial_hash2col(self, inp, data, out, spec):
        data = np.ascontiguousarray(data, np.float32)
        k, s, p, cin, _ = _spec5(spec)
        res = np.empty((cin * k ** inp.dim, out.total_columns()), np.float32)
        fn = self.lib.hcref_serial_hash2col
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(fn(inp.h, _ptr(data), data.shape[0], data.shape[1], out.h, self._sp(spec), _ptr(res)))
        return res

    def col2hash(self, g, inp, out, spec, dtype=np.float32, serial=False):
        suf, T = self._suf(dtype)
        g = np.ascontiguousarray(g, T)
        cin = _spec5(spec)[3]
        res = np.empty((cin, inp.total_columns()), T)
        fn = self.lib.hcref_serial_col2hash if serial else getattr(self.lib, f"hcref_col2hash_{suf}")
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(fn(_ptr(g), g.shape[0], g.shape[1], inp.h, out.h, self._sp(spec), _ptr(res)))
        return res

    def conv_forward(self, inp, data, out, w, spec, dtype=np.float32):
        suf, T = self._suf(dtype)
        data = np.ascontiguousarray(data, T)
        w = np.ascontiguousarray(w, T)
        res = np.empty((_spec5(spec)[4], out.total_columns()), T)
        fn = getattr(self.lib, f"hcref_conv_forward_{suf}")
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                       C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        self._check(fn(inp.h, _ptr(data), data.shape[0], data.shape[1], out.h, _ptr(w), w.shape[0],
                       w.shape[1], self._sp(spec), _ptr(res)))
        return res

    def conv_backward(self, dout, w, cols, inp, out, spec, dtype=np.float32):
        suf, T = self._suf(dtype)
        dout, w, cols = (np.ascontiguousarray(x, T) for x in (dout, w, cols))
        dw = np.empty((dout.shape[0], cols.shape[0]), T)
        dx = np.empty((_spec5(spec)[3], inp.total_columns()), T)
        fn = getattr(self.lib, f"hcref_conv_backward_{suf}")
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_int64] * 3 + [C.c_void_p] * 5
        self._check(fn(_ptr(dout), *dout.shape, _ptr(w), *w.shape, _ptr(cols), *cols.shape,
                       inp.h, out.h, self._sp(spec), _ptr(dw), _ptr(dx)))
        return dw, dx

    def max_pool(self, inp, data, out, spec, dtype=np.float32, serial=False):
        suf, T = self._suf(dtype)
        data = np.ascontiguousarray(data, T)
        cin = _spec5(spec)[3]
        res = np.empty((cin, out.total_columns()), T)
        sw = np.empty((cin, out.total_columns()), np.int32)
        fn = self.lib.hcref_serial_max_pool if serial else getattr(self.lib, f"hcref_max_pool_{suf}")
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64] + [C.c_void_p] * 4
        self._check(fn(inp.h, _ptr(data), data.shape[0], data.shape[1], out.h, self._sp(spec), _ptr(res), _ptr(sw)))
        return res, sw

    def avg_pool(self, inp, data, out, spec, dtype=np.float32):
        suf, T = self._suf(dtype)
        data = np.ascontiguousarray(data, T)
        res = np.empty((_spec5(spec)[3], out.total_columns()), T)
        fn = getattr(self.lib, f"hcref_avg_pool_{suf}")
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64] + [C.c_void_p] * 3
        self._check(fn(inp.h, _ptr(data), data.shape[0], data.shape[1], out.h, self._sp(spec), _ptr(res)))
        return res

    def max_unpool(self, coarse, switches, fine, cs, spec, dtype=np.float32):
        suf, T = self._suf(dtype)
        coarse = np.ascontiguousarray(coarse, T)
        switches = np.ascontiguousarray(switches, np.int32)
        res = np.empty((_spec5(spec)[3], fine.total_columns()), T)
        fn = getattr(self.lib, f"hcref_max_unpool_{suf}")
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int64] + [C.c_void_p] * 4
        self._check(fn(_ptr(coarse), *coarse.shape, _ptr(switches), *switches.shape, fine.h, cs.h,
                       self._sp(spec), _ptr(res)))
        return res

    def avg_unpool(self, coarse, fine, cs, spec, dtype=np.float32):
        suf, T = self._suf(dtype)
        coarse = np.ascontiguousarray(coarse, T)
        res = np.empty((_spec5(spec)[3], fine.total_columns()), T)
        fn = getattr(self.lib, f"hcref_avg_unpool_{suf}")
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_int64] + [C.c_void_p] * 4
        self._check(fn(_ptr(coarse), *coarse.shape, fine.h, cs.h, self._sp(spec), _ptr(res)))
        return res

    def deconv_forward(self, coarse, cdata, fine, w, spec, dtype=np.float32):
        suf, T = self._suf(dtype)
        cdata, w = np.ascontiguousarray(cdata, T), np.ascontiguousarray(w, T)
        res = np.empty((_spec5(spec)[3], fine.total_columns()), T)
        fn = getattr(self.lib, f"hcref_deconv_forward_{suf}")
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                       C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        self._check(fn(coarse.h, _ptr(cdata), *cdata.shape, fine.h, _ptr(w), *w.shape, self._sp(spec), _ptr(res)))
        return res

    def deconv_backward(self, fgrad, w, cdata, coarse, fine, spec, dtype=np.float32):
        suf, T = self._suf(dtype)
        fgrad, w, cdata = (np.ascontiguousarray(x, T) for x in (fgrad, w, cdata))
        dw = np.empty(w.shape, T)
        dx = np.empty(cdata.shape, T)
        fn = getattr(self.lib, f"hcref_deconv_backward_{suf}")
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_int64] * 3 + [C.c_void_p] * 5
        self._check(fn(_ptr(fgrad), *fgrad.shape, _ptr(w), *w.shape, _ptr(cdata), *cdata.shape,
                       coarse.h, fine.h, self._sp(spec), _ptr(dw), _ptr(dx)))
        return dw, dx

    def _gemm(self, name, a, b, out_shape, dtype):
        suf, T = self._suf(dtype)
        a, b = np.ascontiguousarray(a, T), np.ascontiguousarray(b, T)
        c = np.empty(out_shape(a, b), T)
        fn = getattr(self.lib, f"hcref_{name}_{suf}")
        fn.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        self._check(fn(_ptr(a), *a.shape, _ptr(b), *b.shape, _ptr(c)))
        return c

    def matmul(self, a, b, dtype=np.float32):
        return self._gemm("matmul", a, b, lambda a, b: (a.shape[0], b.shape[1]), dtype)

    def matmul_trans_a(self, a, b, dtype=np.float32):
        return self._gemm("matmul_trans_a", a, b, lambda a, b: (a.shape[1], b.shape[1]), dtype)

    def matmul_trans_b(self, a, b, dtype=np.float32):
        return self._gemm("matmul_trans_b", a, b, lambda a, b: (a.shape[0], b.shape[0]), dtype)

    # ---- cnn_ops.cpp:437-608 (batch norm, scale, relu, dropout)
    def _layer_fn(self, name, dtype, argtypes):
        suf, T = self._suf(dtype)
        fn = getattr(self.lib, f"hcref_{name}_{suf}")
        fn.argtypes = argtypes
        return fn, T

    def bn_forward(self, x, running_mean, running_var, eps, momentum, training, dtype=np.float32):
        """-> y, running_mean', running_var', inv_std"""
        S = C.c_float if np.dtype(dtype) == np.float32 else C.c_double
        fn, T = self._layer_fn("bn_forward", dtype, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, S, S,
                                                     C.c_int, C.c_void_p, C.c_void_p])
        x = np.ascontiguousarray(x, T)
        rm, rv = np.array(running_mean, T), np.array(running_var, T)
        y, inv = np.empty_like(x), np.zeros(x.shape[0], T)
        self._check(fn(_ptr(x), *x.shape, _ptr(rm), _ptr(rv), eps, momentum, int(training), _ptr(y), _ptr(inv)))
        return y, rm, rv, inv

    def bn_backward(self, dy, normalized, inv_std, dtype=np.float32):
        fn, T = self._layer_fn("bn_backward", dtype, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                                      C.c_void_p])
        dy, xh, inv = (np.ascontiguousarray(a, T) for a in (dy, normalized, inv_std))
        dx = np.empty_like(dy)
        self._check(fn(_ptr(dy), *dy.shape, _ptr(xh), _ptr(inv), _ptr(dx)))
        return dx

    def scale_forward(self, x, gamma, beta, dtype=np.float32):
        fn, T = self._layer_fn("scale_forward", dtype, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                                        C.c_void_p])
        x, g, b = (np.ascontiguousarray(a, T) for a in (x, gamma, beta))
        y = np.empty_like(x)
        self._check(fn(_ptr(x), *x.shape, _ptr(g), _ptr(b), _ptr(y)))
        return y

    def scale_backward(self, dy, x, gamma, dtype=np.float32):
        fn, T = self._layer_fn("scale_backward", dtype, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                                         C.c_void_p, C.c_void_p, C.c_void_p])
        dy, x, g = (np.ascontiguousarray(a, T) for a in (dy, x, gamma))
        dg, db, dx = np.empty(dy.shape[0], T), np.empty(dy.shape[0], T), np.empty_like(dy)
        self._check(fn(_ptr(dy), _ptr(x), *dy.shape, _ptr(g), _ptr(dg), _ptr(db), _ptr(dx)))
        return dg, db, dx

    def relu(self, x, dy, dtype=np.float32):
        """-> relu_forward(x), relu_backward(dy, relu_forward(x))"""
        fn, T = self._layer_fn("relu", dtype, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                               C.c_void_p])
        x, dy = np.ascontiguousarray(x, T), np.ascontiguousarray(dy, T)
        y, dx = np.empty_like(x), np.empty_like(x)
        self._check(fn(_ptr(x), *x.shape, _ptr(dy), _ptr(y), _ptr(dx)))
        return y, dx

    def dropout(self, x, ratio, seed, training, dy, dtype=np.float32):
        """-> y, keep mask (uint8), dropout_backward(dy, mask, ratio)"""
        S = C.c_float if np.dtype(dtype) == np.float32 else C.c_double
        fn, T = self._layer_fn("dropout", dtype, [C.c_void_p, C.c_int64, C.c_int64, S, C.c_uint64, C.c_int,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p])
        x, dy = np.ascontiguousarray(x, T), np.ascontiguousarray(dy, T)
        y, keep, dx = np.empty_like(x), np.empty(x.size, np.uint8), np.empty_like(x)
        self._check(fn(_ptr(x), *x.shape, ratio, seed, int(training), _ptr(dy), _ptr(y), _ptr(keep), _ptr(dx)))
        return y, keep, dx


class RefSet:
    def __init__(self, ref: Ref, h, dim, res, coords, features):
        self.ref, self.h, self.dim, self.resolution = ref, h, dim, res
        self.coords, self.features = coords, features

    def count(self) -> int:
        return self.coords.shape[0]

    def __del__(self):
        try:
            self.ref.lib.hcref_set_free(self.h)
        except Exception:
            pass


class RefPsh:
    def __init__(self, ref: Ref, h):
        self.ref, self.h = ref, h
        info = np.zeros(6, np.int64)
        ref.lib.hcref_psh_info(h, _ptr(info))
        self.dim, self.resolution, self.n, self.hash_dim, self.offset_dim, self.channels = (int(x) for x in info)
        M = self.hash_dim ** self.dim
        R = self.offset_dim ** self.dim
        self.hash = np.empty(M, np.int32)
        self.offsets = np.empty(R * self.dim, np.uint8)
        self.tags = np.empty(M * self.dim, np.uint16)
        self.data = np.empty((self.channels, self.n), np.float32)
        ref.lib.hcref_psh_copy(h, _ptr(self.hash), _ptr(self.offsets), _ptr(self.tags), _ptr(self.data))

    def validate(self, s: RefSet) -> int:
        return int(self.ref.lib.hcref_psh_validate(self.h, s.h))

    def query(self, p) -> int:
        return int(self.ref.lib.hcref_psh_query(self.h, int(p[0]), int(p[1]), int(p[2]) if len(p) > 2 else 0))

    def hash_slot(self, p) -> int:
        return int(self.ref.lib.hcref_psh_hash_slot(self.h, int(p[0]), int(p[1]), int(p[2]) if len(p) > 2 else 0))

    def __del__(self):
        try:
            self.ref.lib.hcref_psh_free(self.h)
        except Exception:
            pass


class RefNet:
    """Reference LayerGraph<float> (net.hpp:40-60) behind the shim: weights out, one
    net_loss_and_gradients call (net.cpp:260-323, training mode) at a time."""

    def __init__(self, ref: "Ref", h):
        self.ref, self.h = ref, h
        L = ref.lib
        L.hcref_net_blocks.argtypes = [C.c_void_p]
        L.hcref_net_conv_shape.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.hcref_net_get_conv.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.hcref_net_get_bn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.hcref_net_get_fc.argtypes = [C.c_void_p] * 5
        L.hcref_net_set_dropout.argtypes = [C.c_void_p, C.c_float]
        L.hcref_net_loss_grads.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.hcref_net_free.argtypes = [C.c_void_p]
        self.nblocks = int(L.hcref_net_blocks(h))
        self.shapes = []
        for i in range(self.nblocks):
            rc = np.zeros(2, np.int64)
            L.hcref_net_conv_shape(h, i, _ptr(rc))
            self.shapes.append((int(rc[0]), int(rc[1])))

    def conv(self, i: int) -> np.ndarray:
        w = np.empty(self.shapes[i], np.float32)
        self.ref.lib.hcref_net_get_conv(self.h, i, _ptr(w))
        return w

    def bn(self, i: int):
        c = self.shapes[i][0]
        m, v = np.empty(c, np.float32), np.empty(c, np.float32)
        self.ref.lib.hcref_net_get_bn(self.h, i, _ptr(m), _ptr(v))
        return m, v

    def fc(self, classes: int, head_in: int):
        w1, b1 = np.empty((128, head_in), np.float32), np.empty(128, np.float32)
        w2, b2 = np.empty((classes, 128), np.float32), np.empty(classes, np.float32)
        self.ref.lib.hcref_net_get_fc(self.h, _ptr(w1), _ptr(b1), _ptr(w2), _ptr(b2))
        return w1, b1, w2, b2

    def set_dropout(self, ratio: float):
        self.ref.lib.hcref_net_set_dropout(self.h, ratio)

    def loss_and_gradients(self, levels, labels, classes: int, head_in: int):
        arr = (C.c_void_p * len(levels))(*[lv.h for lv in levels])
        labels = np.ascontiguousarray(labels, np.int32)
        loss = np.zeros(1, np.float32)
        cg = np.empty(sum(r * c for r, c in self.shapes), np.float32)
        w1, b1 = np.empty((128, head_in), np.float32), np.empty(128, np.float32)
        w2, b2 = np.empty((classes, 128), np.float32), np.empty(classes, np.float32)
        self.ref._check(self.ref.lib.hcref_net_loss_grads(self.h, arr, len(levels), _ptr(labels), labels.size,
                                                          _ptr(loss), _ptr(cg), _ptr(w1), _ptr(b1), _ptr(w2),
                                                          _ptr(b2)))
        grads, o = [], 0
        for r, c in self.shapes:
            grads.append(cg[o:o + r * c].reshape(r, c))
            o += r * c
        return float(loss[0]), grads, (w1, b1, w2, b2)

    def forward(self, levels, classes: int, training: bool = False) -> np.ndarray:
        """net.cpp:181-258 net_forward: scores (classes x b); inference by default."""
        L = self.ref.lib
        L.hcref_net_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        arr = (C.c_void_p * len(levels))(*[lv.h for lv in levels])
        b = int(levels[-1].batch)
        scores = np.empty((classes, b), np.float32)
        self.ref._check(L.hcref_net_forward(self.h, arr, len(levels), int(training), _ptr(scores)))
        return scores

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.hcref_net_free(self.h)
            self.h = None


class RefSuper(SuperArrays):
    """Reference-built SuperPsh: handle + a host copy of its arrays."""

    def __init__(self, ref: Ref, h):
        info = np.zeros(7, np.int64)
        ref.lib.hcref_super_info(h, _ptr(info))
        dim, res, b, M, R, N, ch = (int(x) for x in info)
        arrays = dict(
            hash=np.empty(M, np.int32), offsets=np.empty(R * dim, np.uint8),
            tags=np.empty(M * dim, np.uint16), model_of_slot=np.empty(M, np.int32),
            hash_acc=np.empty(b + 1, np.int64), offset_acc=np.empty(b + 1, np.int64),
            data_acc=np.empty(b + 1, np.int64), hash_dims=np.empty(b, np.int32),
            offset_dims=np.empty(b, np.int32), data=np.empty((ch, N), np.float32))
        ref.lib.hcref_super_copy(h, *(_ptr(arrays[k]) for k in (
            "hash", "offsets", "tags", "model_of_slot", "hash_acc", "offset_acc", "data_acc",
            "hash_dims", "offset_dims", "data")))
        super().__init__(dim=dim, resolution=res, batch=b, **arrays)
        self.ref, self.h = ref, h

    def locate(self, model: int, p) -> int:
        return int(self.ref.lib.hcref_locate(self.h, model, int(p[0]), int(p[1]), int(p[2])))

    def __del__(self):
        try:
            self.ref.lib.hcref_super_free(self.h)
        except Exception:
            pass


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def have_restated() -> bool:
    return os.path.exists(RESTATED_SO)
