"""Kernel-level A/B timing of the native conv kernels (CUDA events, warm, 256^3 x 8 shells).

    python scripts/kbench.py [C ...]
Prints one line per (C, kernel, field-map layout): ms and achieved TFLOP/s.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1803_11385_b200 import conv  # noqa: E402
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
    cs = [int(a) for a in sys.argv[1:]] or [16, 64, 128]
    res = int(os.environ.get("HCB_RES", "256"))
    batch = int(os.environ.get("HCB_BATCH", "8"))
    lv = bench.shell_levels(res)
    s = SuperPsh.from_levels([lv[0]] * batch)
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("HCB_"))
    n = s.total_columns()
    for c in cs:
        spec = ConvSpec(3, 1, 0, c, c)
        fl = 2.0 * c * 27 * c * n
        x = (torch.rand((n, c), device="cuda") * 2 - 1).to(torch.bfloat16)
        w = torch.rand((c, c * 27), device="cuda") * 2 - 1
        wp = conv.pack_weights(w, c, c, 27, False)
        for name, lay in (("tiled", conv.TILED),):
            fm = conv.field_map_native(s, s, spec, lay)
            t_map = timeit(lambda: conv.field_map_native(s, s, spec, lay))
            t_fwd = timeit(lambda: conv.gather_gemm(fm, x, wp, c, torch.bfloat16))
            t_dw = timeit(lambda: conv.conv_dw(fm, x, x))
            print(f"[{tag}] C={c:4d} {name:6s} map {t_map:.3f} ms | fwd {t_fwd:.3f} ms {fl / t_fwd / 1e9:7.1f} TF/s"
                  f" | dW {t_dw:.3f} ms {fl / t_dw / 1e9:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
