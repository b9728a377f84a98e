"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
data = [r for r in rows[hdr + 1:] if len(r) > si and r[si].isdigit()]
tot = sum(int(r[si]) for r in data) or 1
for r in sorted(data, key=lambda r: -int(r[si]))[:k]:
    print(f"{int(r[si]) * 100.0 / tot:5.1f}%  {r[ie]:>10}  {r[1].strip()[:90]}")
