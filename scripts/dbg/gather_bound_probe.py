"""Is the C=64 forward bound by L2 gather traffic or by the per-row issue work? Same kernel,
same instruction stream; only the field map changes: taps with dx = +-1 set to -1 (zero-fill
cp.async: no L2 read) -> 1/3 of the gathered bytes."""
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
n, C = s.total_columns(), 64
x = (torch.rand((n, C), device="cuda") * 2 - 1).to(torch.bfloat16)
w = torch.rand((C, C * 27), device="cuda") * 2 - 1
wp = conv.pack_weights(w, C, C, 27, False)
fm = conv.field_map_native(s, s, ConvSpec(3, 1, 0, C, C), conv.TILED)
t_full = timeit(lambda: conv.gather_gemm(fm, x, wp, C, torch.bfloat16))
m = fm.data.view(-1, 27, 128)
hits = float((m >= 0).float().mean())
m2 = m.clone()
m2[:, 0::3, :] = -1
m2[:, 2::3, :] = -1
fm2 = conv.FieldMap(m2.contiguous(), fm.n, fm.taps, fm.layout)
t_third = timeit(lambda: conv.gather_gemm(fm2, x, wp, C, torch.bfloat16))
m3 = torch.full_like(m, -1)
fm3 = conv.FieldMap(m3, fm.n, fm.taps, fm.layout)
t_none = timeit(lambda: conv.gather_gemm(fm3, x, wp, C, torch.bfloat16))
print(f"hit fraction {hits:.3f}: all taps {t_full:.3f} ms | dx=0 taps only (1/3 of the L2 gathers) {t_third:.3f} ms"
      f" | no gathers (all zero-fill) {t_none:.3f} ms")
