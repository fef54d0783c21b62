"""Run one BASELINE layer through the fused operator (for ncu / quick timing).

Timing: `reps` launches enqueued back-to-back between two CUDA events (host launch
overhead hidden behind device execution), after `warm` warm-up launches."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _prof  # noqa: E402,F401  (profiling build: CGB_* env knobs)
import paper_2005_06410_b200 as cg
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--layer", default="r50_3x3_56_64")
ap.add_argument("--precision", default="tf32")
ap.add_argument("--algo", default="fused")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--batch", type=int, default=128)
a = ap.parse_args()
layer = [l for l in bench.LAYERS if l[0] == a.layer][0]
(layer, cp, F, I, O), = bench.make_layer_tensors(cg, torch, [layer], a.batch, 0, 1)
st = torch.cuda.current_stream()
for _ in range(a.warm):
    cg.conv(F, I, cp, algo=a.algo, precision=a.precision, out=O)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for r in range(a.reps):
    cg.conv(F, I, cp, algo=a.algo, precision=a.precision, out=O)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
fl = bench.flops(cp)
if int(os.environ.get("CGB_DEBUG_SW", "0")) & 64:
    import numpy as np
    buf = np.zeros((148, 16), dtype=np.uint64)
    cg.lib.cgb_debug_sw_stats(buf.ctypes.data, 148)
    lead = buf[:, 4] > 0  # CTAs whose MMA thread ran (pair leaders)
    tot, wt, wa, wb, nt, ew, eb = [buf[:, i].astype(np.float64) for i in range(7)]
    print(f"  MMA thread cycles (leaders): total max {tot[lead].max():.0f} mean {tot[lead].mean():.0f}; wait t_empty "
          f"{wt[lead].mean():.0f} a_full {wa[lead].mean():.0f} b_full {wb[lead].mean():.0f}; segments max "
          f"{nt.max():.0f} min {nt[lead].min():.0f}; epilogue wait {ew.mean():.0f} busy {eb.mean():.0f}")
    ts = buf[:, 8:14].astype(np.int64)
    ok = ts[:, 0] > 0
    t0 = ts[ok, 0].min()
    rel = (ts[ok] - t0) / 1000.0  # us from the first CTA's entry
    names = ["entry", "mma_start", "mma_end", "epi_end", "exit", "prod_end"]
    for i, n in enumerate(names):
        col = rel[:, i][ts[ok, i] > 0]
        if len(col):
            print(f"  {n:9s} us: min {col.min():7.2f} median {np.median(col):7.2f} max {col.max():7.2f}")

print(f"{a.layer} {a.precision} {cg.last_path()} {ms*1e3:.1f} us  {fl / ms / 1e9:.1f} TFLOPS")

if os.environ.get("CGB_CLOCKS"):
    # sustained run (~2 s) with nvidia-smi clock sampling
    cs = bench.ClockSampler(torch.cuda.current_device())
    cs.start()
    import time
    n = max(1, int(2.0 / (ms * 1e-3)))
    e0.record(st)
    for r in range(n):
        cg.conv(F, I, cp, algo=a.algo, precision=a.precision, out=O)
    e1.record(st)
    torch.cuda.synchronize()
    clk = cs.stop()
    ms2 = e0.elapsed_time(e1) / n
    print(f"  sustained {n} launches: {ms2*1e3:.1f} us  {fl / ms2 / 1e9:.1f} TFLOPS  clocks {clk}")
