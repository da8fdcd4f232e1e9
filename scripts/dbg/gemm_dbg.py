import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1803_11385_b200 import ops
torch.manual_seed(0)
ra, k, cb = 64, 64, 256
for name, fn, A, B, ref in [
    ("nn", ops.matmul, (ra, k), (k, cb), lambda a, b: a @ b),
    ("nt", ops.matmul_trans_b, (ra, k), (cb, k), lambda a, b: a @ b.T),
    ("tn", ops.matmul_trans_a, (k, ra), (k, cb), lambda a, b: a.T @ b)]:
    for init in ("ones", "rand"):
        a = torch.ones(A, device="cuda") if init == "ones" else torch.rand(A, device="cuda")
        b = torch.ones(B, device="cuda") if init == "ones" else torch.rand(B, device="cuda")
        r = ref(a.double(), b.double())
        for mode in ("fast", "tf32"):
            with ops.math_mode(mode):
                c = fn(a, b)
            torch.cuda.synchronize()
            err = float((c.double() - r).norm() / r.norm())
            print(f"{name} {init} {mode}: mean {float(c.mean()):.4f} (ref {float(r.mean()):.4f}) zeros {float((c == 0).double().mean()):.3f} err {err:.2e}", flush=True)
