"""Does K0 (issue-bound probes) overlap with the HBM-bound hi/lo splits on a side stream?"""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_1803_11385_b200 import conv, ops
from paper_1803_11385_b200.psh import SuperPsh
lv = bench.shell_levels(256)
f = SuperPsh.from_levels([lv[0]] * 8)
N = f.total_columns()
sp = ops.ConvSpec(3, 1, 0, 64, 64)
x = torch.rand((N, 64), device="cuda"); dy = torch.rand((N, 64), device="cuda")
s2 = torch.cuda.Stream()
def seq():
    m = conv.field_map_native(f, f, sp, conv.TILED)
    return m, conv.split(x), conv.split(dy)
def ovl():
    ev = torch.cuda.Event()
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        m = conv.field_map_native(f, f, sp, conv.TILED)
        ev.record()
    a, b = conv.split(x), conv.split(dy)
    torch.cuda.current_stream().wait_event(ev)
    return m, a, b
for name, fn in (("seq", seq), ("ovl", ovl), ("seq", seq), ("ovl", ovl)):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    print(name, round(e0.elapsed_time(e1) / 20, 4), "ms")
