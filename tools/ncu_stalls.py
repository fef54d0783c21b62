"""Top SASS instructions by warp-stall samples with their dominant stall reasons
(ncu source page, SASS view): python tools/ncu_stalls.py report.ncu-rep [top]."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
ci = hdr.index("Warp Stall Sampling (All Samples)")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
f = lambda x: float(x or 0)
tot = sum(f(r[ci]) for r in data)
agg = {hdr[i]: sum(f(r[i]) for r in data) for i in st}
print(f"total samples {tot:.0f}; by reason: " + ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
data.sort(key=lambda r: -f(r[ci]))
for r in data[:top]:
    rs = sorted(((f(r[i]), hdr[i][6:]) for i in st), reverse=True)[:2]
    print(f"{f(r[ci]):7.0f} {100*f(r[ci])/tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in rs if v))
