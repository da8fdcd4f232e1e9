"""Top SASS lines of one kernel in an ncu report by stall samples (source page)."""
import csv, io, subprocess, sys

rep, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{pat}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hidx = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hdr = rows[hidx[0]]
end = hidx[1] - 1 if len(hidx) > 1 else len(rows)
data = [r for r in rows[hidx[0] + 1:end] if r and r[0].startswith("0x")]
iS, iE, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
tot = sum(float(r[iS] or 0) for r in data)
print(f"samples {tot:.0f}, warp-instructions {sum(float(r[iE] or 0) for r in data):.0f}")
top = sorted(data, key=lambda r: -float(r[iS] or 0))[:n]
for r in sorted(top, key=lambda r: int(r[0], 16)):
    print(f"{r[0][-5:]} {float(r[iS]) / tot * 100:5.1f}% exec {float(r[iE]):10.0f}  {r[iSrc][:80]}")
