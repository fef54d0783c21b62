"""Run one BASELINE layer through the fused operator a few times (for ncu / quick timing)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_06410_b200 as cg
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--layer", default="r50_3x3_56_64")
ap.add_argument("--precision", default="tf32")
ap.add_argument("--algo", default="fused")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--batch", type=int, default=128)
a = ap.parse_args()
layer = [l for l in bench.LAYERS if l[0] == a.layer][0]
(layer, cp, F, I, O), = bench.make_layer_tensors(cg, torch, [layer], a.batch, 0, 1)
st = torch.cuda.current_stream()
ts = []
for r in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    cg.conv(F, I, cp, algo=a.algo, precision=a.precision, out=O)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
fl = bench.flops(cp)
print(a.layer, a.precision, cg.last_path(), "ms", ["%.4f" % t for t in ts], "TFLOPS %.1f" % (fl / min(ts) / 1e9))
