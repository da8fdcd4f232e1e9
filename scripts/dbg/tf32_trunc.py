"""Does the tf32 tensor core truncate fp32 operands (ignore the low 13 bits) or round them?"""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1803_11385_b200 import ops
torch.manual_seed(0)
a = torch.rand((64, 256), device="cuda") * 2 - 1
b = torch.rand((256, 1024), device="cuda") * 2 - 1
def trunc(x):
    return (x.view(torch.int32) & 0xFFFFE000).view(torch.float32)
def rnd(x):  # round to nearest even at bit 13
    i = x.view(torch.int32)
    return ((i + 0x0FFF + ((i >> 13) & 1)) & 0xFFFFE000).view(torch.float32)
with ops.math_mode("tf32"):
    c_raw = ops.matmul(a, b)
    c_tr = ops.matmul(trunc(a), trunc(b))
    c_rn = ops.matmul(rnd(a), rnd(b))
print("raw==trunc", torch.equal(c_raw, c_tr), "raw==round", torch.equal(c_raw, c_rn),
      "max|raw-trunc|", float((c_raw - c_tr).abs().max()), "max|raw-rnd|", float((c_raw - c_rn).abs().max()))
