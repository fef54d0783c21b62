"""Warp-stall samples per CUDA source line of an ncu report (needs -lineinfo +
--import-source on): the source-level view of where the kernel's warps wait."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = "?"; rows = []
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if len(r) > 5 and r[0] not in ("", "Line No") and r[4] not in ("", "-"):
        try:
            rows.append((float(r[4]), f, r[0], r[1].strip()))
        except ValueError:
            pass
tot = sum(x[0] for x in rows)
rows.sort(reverse=True)
print(f"total samples {tot:.0f}")
for v, f, ln, src in rows[:top]:
    print(f"{v:7.0f} {100 * v / tot:5.1f}%  {f}:{ln}  {src[:100]}")
