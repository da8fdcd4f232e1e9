"""Reference-layout operator timing vs the HBM roofline (256^3 shell x 8, CUDA events).

    python scripts/kbench_ref.py [C]
Algorithmic bytes per SURVEY.md §8d: hash2col/col2hash (27+1)*C*N*4 + 10*M + 3*R + 16*N;
max_pool C*Nf*4 + C*Nc*8; max_unpool C*Nc*8 + C*Nf*4; field map 27*N*4 + 10*M + 3*R + 16*N.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1803_11385_b200 import ops  # noqa: E402
from paper_1803_11385_b200.ops import ConvSpec  # noqa: E402
from paper_1803_11385_b200.psh import SuperPsh  # noqa: E402


def timeit(fn, reps=10):
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
    C = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    peak = json.load(open(bench.PEAKS_PATH))["hbm_gbs"] if os.path.exists(bench.PEAKS_PATH) else 6650.0
    res = int(os.environ.get("HCB_RES", "256"))
    batch = int(os.environ.get("HCB_BATCH", "8"))
    lv = bench.shell_levels(res)
    fine = SuperPsh.from_levels([lv[0]] * batch)
    coarse = SuperPsh.from_levels([lv[1]] * batch)
    N, Nc, M, R = fine.total_columns(), coarse.total_columns(), fine.M, fine.R
    sp, pool = ConvSpec(3, 1, 0, C, C), ConvSpec(2, 2, 0, C, C)
    x = torch.rand((C, N), device="cuda") * 2 - 1
    cols = ops.hash2col(fine, x, fine, sp)
    mp = ops.max_pool(fine, x, coarse, pool)
    rows = [
        ("field_map", lambda: ops.field_map(fine, fine, sp), 27 * N * 4 + 10 * M + 3 * R + 16 * N),
        ("hash2col", lambda: ops.hash2col(fine, x, fine, sp), 28 * C * N * 4 + 10 * M + 3 * R + 16 * N),
        ("col2hash", lambda: ops.col2hash(cols, fine, fine, sp), 28 * C * N * 4 + 10 * M + 3 * R + 16 * N),
        ("max_pool", lambda: ops.max_pool(fine, x, coarse, pool), C * N * 4 + C * Nc * 8),
        ("max_unpool", lambda: ops.max_unpool(mp.output, mp.switches, fine, coarse, pool, check_now=False),
         C * Nc * 8 + C * N * 4),
        ("avg_pool", lambda: ops.avg_pool(fine, x, coarse, pool), C * N * 4 + C * Nc * 4),
    ]
    out = {}
    for name, fn, nbytes in rows:
        ms = timeit(fn)
        gbs = nbytes / (ms / 1e3) / 1e9
        out[name] = {"ms": ms, "GBps": gbs, "frac_hbm": gbs / peak}
        print(f"C={C:4d} {name:20s} {ms:7.3f} ms  {gbs:8.1f} GB/s  {100 * gbs / peak:5.1f}% of HBM", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
