"""Native net-layer timing vs the HBM roofline (256^3 shell x 8, voxel-major, CUDA events).

    python scripts/kbench_net.py [C]
Algorithmic bytes (element sizes: bf16 2, fp32 4, switch 1, map entry 4):
  max_pool (bf16)   C*Nf*2 + Nc*C*(2+1) + Nc*8*4
  max_unpool (bf16) Nf*(4+1) + Nc*C*(2+1) + Nf*C*2
  switch_gather     Nc*C*(1+2) + Nc*8*4 + Nc*C*2
  bn_relu fwd       N*C*(4+4 stats passes + 4 apply read + 4 xhat + 2 out)
  bn_relu bwd       N*C*(2*(2+4) + 2)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1803_11385_b200 import _lib  # noqa: E402
from paper_1803_11385_b200.ops import ConvSpec, field_map  # noqa: E402
from paper_1803_11385_b200.psh import SuperPsh  # noqa: E402
from scripts.kbench_ref import timeit  # noqa: E402


def p(t):
    return C.c_void_p(t.data_ptr())


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    peak = json.load(open(bench.PEAKS_PATH))["hbm_gbs"] if os.path.exists(bench.PEAKS_PATH) else 6650.0
    lv = bench.shell_levels(256)
    fine, coarse = SuperPsh.from_levels([lv[0]] * 8), SuperPsh.from_levels([lv[1]] * 8)
    nf, nc = fine.total_columns(), coarse.total_columns()
    L, BF = _lib.lib, _lib.HC_DTYPE_BF16
    pm = field_map(fine, coarse, ConvSpec(2, 2, 0, c, c))
    par = torch.empty(nf, dtype=torch.int32, device="cuda")
    prow = torch.empty(nf, dtype=torch.int8, device="cuda")
    _lib.check(L.hc_native_pool_parents(p(pm), nc, 8, nf, p(par), p(prow), None))
    x = (torch.rand((nf, c), device="cuda") * 2 - 1).to(torch.bfloat16)
    y = torch.empty((nc, c), dtype=torch.bfloat16, device="cuda")
    sw = torch.empty((nc, c), dtype=torch.int8, device="cuda")
    dx = torch.empty((nf, c), dtype=torch.bfloat16, device="cuda")
    yf = torch.randn((nf, c), device="cuda")
    xhat = torch.empty_like(yf)
    rm, rv, inv = torch.zeros(c, device="cuda"), torch.ones(c, device="cuda"), torch.empty(c, device="cuda")
    ws = torch.empty(int(L.hc_native_bn_workspace(nf, c)), dtype=torch.uint8, device="cuda")
    rows = [
        ("max_pool", lambda: L.hc_native_max_pool(p(pm), nc, 8, p(x), BF, c, p(y), p(sw), None),
         c * nf * 2 + nc * c * 3 + nc * 32),
        ("max_unpool", lambda: L.hc_native_max_unpool(p(par), p(prow), nf, p(y), BF, c, p(sw), p(dx), None),
         nf * 5 + nc * c * 3 + nf * c * 2),
        ("switch_gather", lambda: L.hc_native_switch_gather(p(pm), nc, 8, p(dx), BF, c, p(sw), p(y), None),
         nc * c * 3 + nc * 32 + nc * c * 2),
        ("bn_relu_fwd", lambda: L.hc_native_bn_relu_forward(p(yf), nf, c, 1, 0.1, 1e-5, p(rm), p(rv), p(inv),
                                                            p(xhat), p(dx), p(ws), ws.numel(), None),
         nf * c * 18),
        ("bn_relu_bwd", lambda: L.hc_native_bn_relu_backward(p(dx), BF, p(xhat), p(inv), nf, c, p(x), p(ws),
                                                             ws.numel(), None),
         nf * c * 14),
    ]
    for name, fn, nbytes in rows:
        ms = timeit(fn)
        gbs = nbytes / (ms / 1e3) / 1e9
        print(f"C={c:4d} native {name:14s} {ms:7.3f} ms  {gbs:8.1f} GB/s  {100 * gbs / peak:5.1f}% of HBM", flush=True)


if __name__ == "__main__":
    main()
