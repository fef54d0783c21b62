"""Turn the ncu captures in gpurun_out/ into the committed evidence under profiles/:
per-layer key-metric summaries, top stalled SASS lines, the launch list, and
profiles/ncu_traffic.json (DRAM bytes per 7-layer step, read by bench.py)."""
import json, os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RND = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = os.path.join(ROOT, "gpurun_out")
prof = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)
sys.path.insert(0, ROOT)
import bench
total = 0.0
per = {}
for l in bench.LAYERS:
    rep = os.path.join(out, f"prof_{l[0]}.ncu-rep")
    if not os.path.exists(rep):
        print("missing", rep); continue
    s = subprocess.run([sys.executable, os.path.join(ROOT, "tools/ncu_summary.py"), rep], capture_output=True, text=True).stdout
    open(os.path.join(prof, f"{RND}_{l[0]}_ncu_raw.txt"), "w").write(s)
    h = subprocess.run([sys.executable, os.path.join(ROOT, "tools/ncu_stalls.py"), rep, "40"], capture_output=True, text=True).stdout
    h += "\n-- per CUDA source line --\n"
    h += subprocess.run([sys.executable, os.path.join(ROOT, "tools/ncu_lines.py"), rep, "25"], capture_output=True, text=True).stdout
    open(os.path.join(prof, f"{RND}_{l[0]}_ncu_hot_sass.txt"), "w").write(h)
    rd = wr = None
    for line in s.splitlines():
        parts = line.split()
        if parts and parts[0] == "dram__bytes_read.sum": rd = (float(parts[1]), parts[2])
        if parts and parts[0] == "dram__bytes_write.sum": wr = (float(parts[1]), parts[2])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if rd and wr:
        b = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
        per[l[0]] = b; total += b
if os.path.exists(os.path.join(out, "launches.csv")):
    shutil.copy(os.path.join(out, "launches.csv"), os.path.join(prof, f"{RND}_launches_bench.csv"))
json.dump({"tf32": total if per else None, "unit": "bytes per 7-layer step (dram read+write, ncu --set full, one capture per layer)",
           "per_layer": per}, open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(per, indent=1), total)
