import os, time, torch
p = torch.cuda.get_device_properties(0)
bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
base = f"/sys/bus/pci/devices/{bus}"
print("bus", bus, "numa", open(base + "/numa_node").read().strip() if os.path.exists(base) else "?",
      "cpus", open(base + "/local_cpulist").read().strip() if os.path.exists(base) else "?", "ncpu", os.cpu_count(),
      "affinity", len(os.sched_getaffinity(0)))
def bw(tag):
    h = torch.empty(235_000_000, dtype=torch.float32, pin_memory=True)
    d = torch.empty_like(h, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    h2d = 5 * h.numel() * 4 / (s.elapsed_time(e) / 1e3) / 1e9
    s.record()
    for _ in range(5): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    d2h = 5 * h.numel() * 4 / (s.elapsed_time(e) / 1e3) / 1e9
    print(tag, "H2D %.1f GB/s D2H %.1f GB/s" % (h2d, d2h), flush=True)
bw("default")
if os.path.exists(base + "/local_cpulist"):
    cl = open(base + "/local_cpulist").read().strip()
    cpus = set()
    for part in cl.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    os.sched_setaffinity(0, cpus)
    bw("numa-local")
