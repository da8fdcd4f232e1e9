import torch
n = 935542784 // 4
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(n, device="cuda"); d_out = torch.empty(n, device="cuda")
a, b = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    with torch.cuda.stream(a): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(b): h_out.copy_(d_out, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
cur = torch.cuda.current_stream()
s.record(cur); a.wait_stream(cur); b.wait_stream(cur)
for _ in range(5):
    with torch.cuda.stream(a): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(b): h_out.copy_(d_out, non_blocking=True)
cur.wait_stream(a); cur.wait_stream(b); e.record(cur); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print("duplex: %.2f ms per (0.94 GB H2D + 0.94 GB D2H) -> %.1f GB/s each way" % (ms, n * 4 / ms / 1e6))
s.record(cur)
for _ in range(5): d_in.copy_(h_in, non_blocking=True)
e.record(cur); torch.cuda.synchronize()
print("H2D alone: %.2f ms" % (s.elapsed_time(e) / 5))
