"""Same-process A/B of dispatch knobs (cgb_set_tuning) on BASELINE layers.

  python tools/ab_tune.py --layers r50_3x3_s2_56_128,r50_3x3_56_64 --variants '{}' '{"tps":1}' --rounds 7

Each round times every (layer, variant) once, interleaved, as `reps` back-to-back
launches after an L2 flush (CUDA events); reports the mean per (layer, variant) in us (single-launch event timings are quantised
to ~2 us on B200, so average many rounds).
Also `--graph`: the whole 7-layer bench step as one CUDA-graph replay per variant.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2005_06410_b200 as cg  # noqa: E402
from paper_2005_06410_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="bench")
ap.add_argument("--variants", nargs="+", default=["{}"])
ap.add_argument("--rounds", type=int, default=7)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--precision", default="tf32")
ap.add_argument("--batch", type=int, default=0, help="override the stated batch")
ap.add_argument("--graph", action="store_true", help="time the whole list as one graph replay per variant")
ap.add_argument("--verbose", action="store_true", help="print each launch's configuration (stderr)")
a = ap.parse_args()
if a.verbose:
    cg.set_tuning("verbose", 1)

by_name = {l[0]: (cfg, l, cp, dist) for cfg, l, cp, dist in configs.all_layers()}
names = [l[0] for l in configs.C2] if a.layers == "bench" else a.layers.split(",")
variants = [json.loads(v) for v in a.variants]
tensors = []
for n in names:
    cfg, l, cp, dist = by_name[n]
    if a.batch:
        cp = dict(cp, b=a.batch)
    F, I = configs.make_tensors(torch, cg.empty_tensor4, cp, dist, configs.layer_seed(n))
    h, w = configs.out_hw(cp)
    O = cg.empty_tensor4(cp["k_n"], h, w, cp["b"])
    tensors.append((n, cp, F, I, O))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def run_all(v=None):
    """The layer list; a variant's knobs apply to every layer, or only to v["only"]."""
    v = dict(v or {})
    only = v.pop("only", None)
    for n, cp, F, I, O in tensors:
        if only is None or n == only:
            with cg.tuning(**v):
                cg.conv(F, I, cp, precision=a.precision, out=O)
        else:
            cg.conv(F, I, cp, precision=a.precision, out=O)


times = {}
graphs = {}
if a.graph:
    for vi, v in enumerate(variants):
        run_all(v)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        s2.wait_stream(st)
        with torch.cuda.stream(s2):
            run_all(v)
        st.wait_stream(s2)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            run_all(v)
        graphs[vi] = g
for r in range(a.rounds):
    for vi, v in enumerate(variants):
        if a.graph:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(a.reps):
                flush.zero_()
                graphs[vi].replay()
            flush.zero_()
            e0.record(st)
            graphs[vi].replay()
            e1.record(st)
            torch.cuda.synchronize()
            times.setdefault(("step", vi), []).append(e0.elapsed_time(e1) * 1e3)
            continue
        vv = dict(v)
        vv.pop("only", None)
        with cg.tuning(**vv):
            for n, cp, F, I, O in tensors:
                cg.conv(F, I, cp, precision=a.precision, out=O)  # warm / config
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(a.reps):
                    cg.conv(F, I, cp, precision=a.precision, out=O)
                e1.record(st)
                torch.cuda.synchronize()
                times.setdefault((n, vi), []).append(e0.elapsed_time(e1) * 1e3 / a.reps)
keys = ["step"] if a.graph else names
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    print("sm clock now", pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), "MHz; throttle reasons",
          hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
except Exception as e:  # noqa: BLE001
    print("no nvml", e)
print("variant".ljust(40) + "".join(k[-14:].rjust(15) for k in keys) + "      sum")
for vi, v in enumerate(variants):
    meds = [statistics.mean(times[(k, vi)]) for k in keys]
    print(json.dumps(v)[:40].ljust(40) + "".join(f"{m:15.1f}" for m in meds) + f"{sum(meds):9.1f}")
