"""Summarise an ncu --set full report (and an optional launch-list CSV) for profiles/.

    python scripts/ncu_summary.py REPORT.ncu-rep [launches.csv] > profiles/xxx.md
Also writes profiles/ncu_traffic.json: per bench op, DRAM bytes (read+write) per launch
from the full capture (bench.py reads it into roofline.traffic), and profiles/ncu_kernels.json:
per bench op, the counters that bound it (DRAM bytes, tensor pipe, the tensor core's and the
LSU's shared-memory pipes, L2 hit rate) — bench.py attaches them to its per-kernel entries.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OP_OF = {"k_field_map": "field_map", "k_conv_dw": "dW_conv", "k_conv_fwd": "fwd_conv", "k_split_vm": "split_pack",
         "k_hash2col": "hash2col", "k_col2hash": "col2hash",
         # reference-layout contraction (gemm_tc.cu: <MMA-A MN-major, MMA-B MN-major, ...>)
         "k_gemm_tf32<1, 0": "fwd_gemm", "k_gemm_tf32<0, 0": "dW_gemm", "k_gemm_tf32<1, 1": "dcols_gemm"}
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]
# extra counters kept per op in ncu_kernels.json (not printed in the table)
EXTRA = [("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
         ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "tc_smem_pipe_pct"),
         ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "lsu_smem_pipe_pct"),
         ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
         ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum", "bf16_mma_flop")]


def scale(v, unit):
    u = unit.strip().lower()
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
            "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    return v * mult.get(u, 1.0)


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    print(f"### ncu --set full: `{os.path.basename(rep)}`\n")
    print("| kernel | " + " | ".join(name for _, name in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    traffic = {}
    counters = {}
    for d in data:
        name = d[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.replace("unnamed>::", "").strip()
        cells = []
        vals = {}
        for m, label in METRICS:
            if m not in hdr:
                cells.append("-")
                continue
            i = hdr.index(m)
            try:
                v = float(d[i])
            except ValueError:
                cells.append(d[i])
                continue
            if label in ("DRAM read", "DRAM write"):
                v = scale(v, units[i]) / 1e6
                cells.append(f"{v:.1f} MB")
            elif label == "time":
                v = scale(v, units[i])
                cells.append(f"{v:.3f} ms")
            else:
                cells.append(f"{v:.1f}")
            vals[label] = v
        print(f"| `{name[:60]}` | " + " | ".join(cells) + " |")
        for k, op in OP_OF.items():
            if k in name and "DRAM read" in vals:
                traffic.setdefault(op, vals["DRAM read"] * 1e6 + vals.get("DRAM write", 0) * 1e6)
                if op not in counters:
                    c = {"kernel": name[:80], "time_ms": vals.get("time"),
                         "dram_bytes": vals["DRAM read"] * 1e6 + vals.get("DRAM write", 0) * 1e6}
                    for m, key in EXTRA:
                        if m in hdr:
                            try:
                                c[key] = float(d[hdr.index(m)])
                            except ValueError:
                                pass
                    counters[op] = c
    if len(sys.argv) > 2:
        print("\n### launch list (cold, serialised — compare shares, not absolutes)\n")
        txt = open(sys.argv[2]).read()
        lines = [ln for ln in txt.splitlines() if ln.startswith('"')]
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        h = rows[0]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        ui = h.index("Metric Unit")
        tot = {}
        for r in rows[1:]:
            k = r[ki].split("(")[0].replace("void ", "").strip()
            try:
                t = scale(float(r[vi].replace(",", "")), r[ui])
            except ValueError:
                continue
            tot[k] = tot.get(k, 0.0) + t
        s = sum(tot.values()) or 1.0
        print("| kernel | total ms | share |\n|---|---|---|")
        for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
            print(f"| `{k[:70]}` | {t:.3f} | {100 * t / s:.1f}% |")
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    merged = json.load(open(path)) if os.path.exists(path) else {}
    merged.update(traffic)  # captures of other workloads keep their entries
    json.dump(merged, open(path, "w"), indent=1)
    kpath = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    kmerged = json.load(open(kpath)) if os.path.exists(kpath) else {}
    kmerged.update(counters)
    json.dump(kmerged, open(kpath, "w"), indent=1)


if __name__ == "__main__":
    main()
