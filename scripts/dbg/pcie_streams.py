"""PCIe copy throughput on the GPU box: one vs several streams per direction, H2D / D2H alone and
duplex, for the e2e step's byte counts (0.94 GB each way). Pinned host memory, CUDA events."""
import torch
n = 935542784 // 4
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(n, device="cuda"); d_out = torch.empty(n, device="cuda")
cur = torch.cuda.current_stream()


def run(k, h2d=True, d2h=True, reps=4):
    sa = [torch.cuda.Stream() for _ in range(k)]
    sb = [torch.cuda.Stream() for _ in range(k)]
    part = (n + k - 1) // k

    def once():
        for i in range(k):
            lo, hi = i * part, min(n, (i + 1) * part)
            if h2d:
                with torch.cuda.stream(sa[i]):
                    d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
            if d2h:
                with torch.cuda.stream(sb[i]):
                    h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
    once()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(cur)
    for x in sa + sb:
        x.wait_stream(cur)
    for _ in range(reps):
        once()
    for x in sa + sb:
        cur.wait_stream(x)
    e.record(cur)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    what = "duplex" if h2d and d2h else ("H2D" if h2d else "D2H")
    print(f"{what:6s} streams/direction {k}: {ms:6.2f} ms -> {n * 4 / ms / 1e6:5.1f} GB/s each way")


for k in (1, 2, 4):
    run(k, True, False)
    run(k, False, True)
    run(k, True, True)
