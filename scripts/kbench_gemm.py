"""Reference-layout contraction timing (csrc/gemm_tc.cu vs gemm_fast.cu), CUDA events.

    python scripts/kbench_gemm.py [C] [N]         (HCB_TC_GEMM=0 forces the FFMA kernels;
                                                   HCB_GEMM_OPS=fwd,dW,dcol HCB_GEMM_MODES=fast,tf32)
The three products of one materialised conv layer C -> C over N voxels (default 256^3 x 8
shells): fwd Y = W cols (matmul), dW = dY cols^T (matmul_trans_b), dcols = W^T dY
(matmul_trans_a). Flops 2*C*27C*N each; minimum bytes: the column matrix (27*C*N*4) read
(fwd, dW) or written (dcols) plus the C x N operand.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1803_11385_b200 import ops  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    C = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 1826368
    peaks = json.load(open(bench.PEAKS_PATH)) if os.path.exists(bench.PEAKS_PATH) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    K = 27 * C
    w = torch.rand((C, K), device="cuda") * 2 - 1
    cols = torch.rand((K, N), device="cuda") * 2 - 1
    dy = torch.rand((C, N), device="cuda") * 2 - 1
    flops = 2.0 * C * K * N
    colbytes = 4.0 * K * N + 4.0 * C * N
    tag = "ffma" if os.environ.get("HCB_TC_GEMM") == "0" else "tc"
    modes = os.environ.get("HCB_GEMM_MODES", "fast,tf32").split(",")
    ops_sel = os.environ.get("HCB_GEMM_OPS", "fwd,dW,dcol").split(",")
    for mode in modes:
        with ops.math_mode(mode):
            for name, fn in (("fwd  matmul", lambda: ops.matmul(w, cols)),
                             ("dW   matmul_trans_b", lambda: ops.matmul_trans_b(dy, cols)),
                             ("dcol matmul_trans_a", lambda: ops.matmul_trans_a(w, dy))):
                if name.split()[0] not in ops_sel:
                    continue
                ms = timeit(fn)
                tf = flops / (ms / 1e3) / 1e12
                gbs = colbytes / (ms / 1e3) / 1e9
                print(f"[{tag}/{mode}] C={C} N={N} {name:22s} {ms:8.3f} ms  {tf:7.1f} TF/s  "
                      f"{gbs:7.1f} GB/s ({100 * gbs / hbm:4.1f}% of HBM)", flush=True)
        if tag == "ffma":
            break


if __name__ == "__main__":
    main()
