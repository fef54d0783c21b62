"""Per-kernel device timeline of one CUDA-graph replay of the 7 BASELINE layers:
%globaltimer stamps of every CTA (CGB_DEBUG_SW=64 stats slots), relative to the
first CTA entry: start/end of each kernel and the gaps between consecutive kernels."""
import os, sys
os.environ["CGB_DEBUG_SW"] = "64"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _prof  # noqa: E402,F401  (profiling build: CGB_* env knobs)
import paper_2005_06410_b200 as cg
import bench
BATCH_TL = int(os.environ.get("TL_BATCH", "128"))
tensors = bench.make_layer_tensors(cg, torch, bench.LAYERS, BATCH_TL, 0, 1)
def step():
    for layer, cp, F, I, O in tensors:
        cg.conv(F, I, cp, algo="fused", precision="tf32", out=O)
step(); torch.cuda.synchronize()
s2 = torch.cuda.Stream(); s2.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s2):
    step()
torch.cuda.current_stream().wait_stream(s2); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
cg.lib.cgb_debug_sw_stats(None, 4096)  # zero all slots, then exactly one replay
g.replay()
torch.cuda.synchronize()
buf = np.zeros((8, 1024, 16), dtype=np.uint64)
cg.lib.cgb_debug_sw_stats(buf.ctypes.data, 4096)
rows = []
for sl in range(8):
    ent = buf[sl, :, 8].astype(np.int64); ext = buf[sl, :, 12].astype(np.int64)
    mst = buf[sl, :, 9].astype(np.int64); men = buf[sl, :, 10].astype(np.int64)
    ok = ent > 0
    if ok.sum() == 0:
        continue
    ee = buf[sl, :, 11].astype(np.int64)
    rows.append((ent[ok].min(), np.median(ent[ok]), mst[mst > 0].min() if (mst > 0).any() else 0,
                 men[men > 0].max() if (men > 0).any() else 0, ext[ok].max(), ok.sum(),
                 np.percentile(men[men > 0], [10, 50, 90]) if (men > 0).any() else [0, 0, 0],
                 np.percentile(ee[ee > 0], [10, 50, 90]) if (ee > 0).any() else [0, 0, 0],
                 np.percentile(ext[ok], [10, 50, 90])))
rows.sort()
t0 = rows[0][0]
prev_end = None
for r in rows:
    e0, emed, ms, me, x1, n, mep, eep, xp = r
    gap = (e0 - prev_end) / 1e3 if prev_end else 0
    print(f"entry {(e0 - t0) / 1e3:8.2f} (median {(emed - t0) / 1e3:8.2f})  first mma {(ms - t0) / 1e3:8.2f}  "
          f"last mma end {(me - t0) / 1e3:8.2f}  exit {(x1 - t0) / 1e3:8.2f}  span {(x1 - e0) / 1e3:6.2f}  "
          f"overlap/gap vs prev exit {gap:6.2f}  ctas {n}")
    print("      mma end p10/50/90 " + " ".join(f"{(v - t0) / 1e3:8.2f}" for v in mep) +
          "   epi end " + " ".join(f"{(v - t0) / 1e3:8.2f}" for v in eep) +
          "   exit " + " ".join(f"{(v - t0) / 1e3:8.2f}" for v in xp))
    prev_end = x1
print(f"total {(rows[-1][4] - t0) / 1e3:.1f} us")
