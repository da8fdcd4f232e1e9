"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python scripts/launch_table.py launches.csv [steps]"""
import csv
import io
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
txt = open(sys.argv[1]).read()
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = {}, {}
for r in rows[1:]:
    k = r[ki].split("(")[0].replace("void ", "").replace("hcb::<unnamed>::", "")[:70]
    v = float(r[vi].replace(",", "")) * UNIT.get(r[ui].strip(), 1.0)
    tot[k] = tot.get(k, 0.0) + v
    cnt[k] = cnt.get(k, 0) + 1
s = sum(tot.values())
print(f"| kernel | us per step | share | launches per step |\n|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:30]:
    print(f"| `{k}` | {v / steps:.1f} | {100 * v / s:.1f}% | {cnt[k] / steps:.0f} |")
print(f"| total | {s / steps:.1f} | | {sum(cnt.values()) / steps:.0f} |")
