"""fwd gather-GEMM at C_in = 64 with C_out in {16, 32, 64, 128}: how much of the time follows N
(B operand + MMA) versus the gather (fixed by C_in)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_1803_11385_b200 import conv
from paper_1803_11385_b200.ops import ConvSpec
from paper_1803_11385_b200.psh import SuperPsh
from scripts.kbench import timeit
lv = bench.shell_levels(256)
s = SuperPsh.from_levels([lv[0]] * 8)
n = s.total_columns()
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x = (torch.rand((n, ci), device="cuda") * 2 - 1).to(torch.bfloat16)
fm = conv.field_map_native(s, s, ConvSpec(3, 1, 0, ci, ci), conv.TILED)
for co in (16, 32, 64, 128):
    w = torch.rand((co, ci * 27), device="cuda") * 2 - 1
    wp = conv.pack_weights(w, co, ci, 27, False)
    t = timeit(lambda: conv.gather_gemm(fm, x, wp, co, torch.bfloat16))
    print(f"C_in={ci} C_out={co:4d} fwd {t:.3f} ms  {2.0 * co * 27 * ci * n / t / 1e9:7.1f} TF/s", flush=True)
