"""Top SASS instructions by warp-stall samples from an ncu report (source page, SASS view)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ci = hdr.index("Warp Stall Sampling (All Samples)"); si = hdr.index("Source")
tot = sum(float(r[ci] or 0) for r in data if len(r) > ci)
data.sort(key=lambda r: -float(r[ci] or 0) if len(r) > ci else 0)
print(f"total samples {tot:.0f}")
for r in data[:top]:
    print(f"{float(r[ci]):8.0f} {100*float(r[ci])/tot:5.1f}%  {r[0][-5:]}  {r[si].strip()[:90]}")
