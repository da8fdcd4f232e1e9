"""Key counters of every kernel in an ncu report (raw page): time, DRAM/L2/L1 throughput,
tensor pipe, issue activity, top warp-stall reasons."""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
keys = [("time_ms", "gpu__time_duration.sum"), ("dram_rd_MB", "dram__bytes_read.sum"),
        ("dram_wr_MB", "dram__bytes_write.sum"), ("lts_sectors", "lts__t_sectors.sum"),
        ("L2%", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L1%", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
        ("tensor%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("issue%", "sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
        ("lsu%", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        ("inst", "smsp__inst_executed.sum")]
for r in data:
    name = r[col["Kernel Name"]][:60]
    out = []
    for k, m in keys:
        if m in col:
            out.append(f"{k}={r[col[m]]}")
    stalls = []
    for h, i in col.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print(name, " ".join(out))
    print("   stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:7]))
