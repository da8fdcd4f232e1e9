"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libhcref.so, i.e. /root/reference):

    make -C oracle ref && python tests/golden/make_golden.py

Fixtures (committed; the GPU box has no /root/reference):

* ``inst_XXX.npz`` — acceptance criterion-3 instances (tests/acceptance.cpp:174-203
  make_instance + the input seeds of criterion3, acceptance.cpp:209-232): super-PSH
  tables, inputs, and every reference output (fp32 results of the float
  instantiation; conv outputs/gradients also from the double instantiation).
  Large column matrices are stored as sha256 digests.
* ``fig2.npz`` — the worked 2-D example (test_psh_core.cpp:23-75,
  acceptance.cpp:71-107): reference-built tables with the injected offsets.
* ``shell32.npz`` — config 1 (32^3 shell, C 8->16): digests of the reference's
  hash2col / conv / dW / dX / max_pool / max_unpool outputs on seeded inputs.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Ref, mix_seed  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TRIALS = range(12)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def super_arrays(prefix: str, s) -> dict:
    d = {}
    for k in ("hash", "offsets", "tags", "model_of_slot", "hash_acc", "offset_acc", "data_acc", "hash_dims",
              "offset_dims"):
        d[f"{prefix}_{k}"] = getattr(s, k)
    d[f"{prefix}_meta"] = np.array([s.dim, s.resolution, s.batch], np.int64)
    return d


def instance(ref: Ref, trial: int) -> dict:
    inst = ref.make_instance(trial)
    fine, coarse, spec = inst["fine"], inst["coarse"], inst["spec"]
    c_in, c_out = inst["c_in"], inst["c_out"]
    out_s = fine if spec[1] == 1 else coarse
    fd = spec[0] ** 3
    seed = 91000 + trial * 13
    data = ref.random_matrix(c_in, fine.total_columns(), seed + 1)
    w = ref.random_matrix(c_out, c_in * fd, seed + 2)
    dout = ref.random_matrix(c_out, out_s.total_columns(), seed + 3)
    coarse_vals = ref.random_matrix(c_in, coarse.total_columns(), seed + 4)
    dc_spec = (2, 2, 0, c_in, c_out) if spec[1] == 1 else spec
    dc_fd = dc_spec[0] ** 3
    dc_w = ref.random_matrix(c_out, c_in * dc_fd, seed + 5)
    dc_in = ref.random_matrix(c_out, coarse.total_columns(), seed + 6)
    y = ref.random_matrix(c_in * fd, out_s.total_columns(), seed + 8)
    pool_spec = (2, 2, 0, c_in, c_in)

    cols = ref.hash2col(fine, data, out_s, spec)
    conv_out = ref.matmul(w, cols)
    dw, dx = ref.conv_backward(dout, w, cols, fine, out_s, spec)
    mp, sw = ref.max_pool(fine, data, coarse, pool_spec)
    ap = ref.avg_pool(fine, data, coarse, pool_spec)
    max_restored = ref.max_unpool(mp, sw, fine, coarse, pool_spec)
    avg_restored = ref.avg_unpool(coarse_vals, fine, coarse, pool_spec)
    dc_out = ref.deconv_forward(coarse, dc_in, fine, dc_w, dc_spec)
    dcb_dw, dcb_dx = ref.deconv_backward(data, dc_w, dc_in, coarse, fine, dc_spec)
    c2h = ref.col2hash(y, fine, out_s, spec)
    # double instantiation of the same ops on the same (fp32-valued) inputs
    f64 = np.float64
    cols64 = ref.hash2col(fine, data.astype(f64), out_s, spec, f64)
    conv64 = ref.matmul(w.astype(f64), cols64, f64)
    dw64, dx64 = ref.conv_backward(dout.astype(f64), w.astype(f64), cols64, fine, out_s, spec, f64)

    d = dict(spec=np.array(spec, np.int64), dc_spec=np.array(dc_spec, np.int64),
             pool_spec=np.array(pool_spec, np.int64),
             data=data, w=w, dout=dout, coarse_vals=coarse_vals, dc_w=dc_w, dc_in=dc_in, y=y,
             cols_sha=np.array(sha(cols)), conv_out=conv_out, dw=dw, dx=dx, mp=mp, sw=sw, ap=ap,
             max_restored=max_restored, avg_restored=avg_restored, dc_out=dc_out, dcb_dw=dcb_dw, dcb_dx=dcb_dx,
             c2h=c2h, conv64=conv64, dw64=dw64, dx64=dx64)
    d.update(super_arrays("fine", fine))
    d.update(super_arrays("coarse", coarse))
    return d


def fig2(ref: Ref) -> dict:
    pixels = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [3, 1, 0], [4, 1, 0], [1, 2, 0], [2, 2, 0], [3, 2, 0]],
                      np.int32)
    offsets = np.array([0, 0, 0, 2, 2, 1, 1, 2], np.uint8)
    feats = np.arange(8, dtype=np.float32).reshape(1, 8)
    s = ref.make_set(2, 8, pixels, feats)
    p = ref.build_psh(s, 0, offsets, 2)
    return dict(pixels=pixels, offsets=offsets, features=feats, hash=p.hash, tags=p.tags,
                meta=np.array([p.n, p.hash_dim, p.offset_dim, p.hash_slot((3, 1)), p.query((3, 1))], np.int64))


def shell32(ref: Ref) -> dict:
    s = ref.sphere_set(32, True)
    fine_l = ref.build_psh(s, mix_seed(1, 0))
    coarse_l = ref.build_psh(ref.coarsen(s), mix_seed(1, 1))
    fine, coarse = ref.build_super([fine_l]), ref.build_super([coarse_l])
    spec, pool = (3, 1, 0, 8, 16), (2, 2, 0, 8, 8)
    data = ref.random_matrix(8, fine.total_columns(), 5)
    w = ref.random_matrix(16, 8 * 27, 6)
    dout = ref.random_matrix(16, fine.total_columns(), 7)
    cols = ref.hash2col(fine, data, fine, spec)
    out = ref.conv_forward(fine, data, fine, w, spec)
    dw, dx = ref.conv_backward(dout, w, cols, fine, fine, spec)
    mp, sw = ref.max_pool(fine, data, coarse, pool)
    un = ref.max_unpool(mp, sw, fine, coarse, pool)
    d = {k: np.array(sha(v)) for k, v in dict(cols=cols, conv_out=out, dw=dw, dx=dx, mp=mp, sw=sw, unpool=un).items()}
    d["n"] = np.array([fine.total_columns(), coarse.total_columns()], np.int64)
    d["hash_sha"] = np.array(sha(fine.hash))
    return d


def main():
    ref = Ref()
    for t in TRIALS:
        np.savez_compressed(os.path.join(OUT, f"inst_{t:03d}.npz"), **instance(ref, t))
    np.savez_compressed(os.path.join(OUT, "fig2.npz"), **fig2(ref))
    np.savez_compressed(os.path.join(OUT, "shell32.npz"), **shell32(ref))
    print("wrote", len(TRIALS), "instances + fig2 + shell32 to", OUT)


if __name__ == "__main__":
    main()
