#!/usr/bin/env python
"""The paper's workspace claim on HBM (PAPER P1, test_convgemm.cpp:231-242):
the explicit path materialises B-hat (k x n floats) in device memory, the fused path needs
none (TF32) or only the filter split (3xTF32). For the BASELINE layers this records, per
layer: B-hat bytes, the device workspace each path takes, the time of each path (explicit
= im2col kernel + GEMM over B-hat), and whether the explicit path survives a workspace
limit (the ScratchTracker limit -> AllocationFailure, like the reference's).

  python tools/workspace_demo.py [--limit-gb 4] [--out FILE]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench_configs as bc  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _prof  # noqa: E402,F401  (profiling build: CGB_* env knobs)
import paper_2005_06410_b200 as cg  # noqa: E402


def timed(fn, reps=3):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--limit-gb", type=float, default=4.0)
    ap.add_argument("--precision", default="tf32")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    limit = int(a.limit_gb * (1 << 30))
    rows = []
    layers = bc.CONFIGS["C2"] + bc.CONFIGS["C4"] + bc.CONFIGS["C5"][:3]
    for layer in layers:
        cp = layer["cp"]
        F, I, O = bc.tensors(layer)
        bhat = cg.im2col_workspace_bytes(cp)
        r = dict(layer=layer["name"], bhat_bytes=bhat,
                 ws_explicit=cg.conv_workspace_bytes(cp, "explicit", a.precision),
                 ws_fused=cg.conv_workspace_bytes(cp, "fused", a.precision))
        r["us_fused"] = round(timed(lambda: cg.conv(F, I, cp, "fused", a.precision, out=O)), 1)
        cg.lib.cgb_scratch_release()
        try:
            r["us_explicit"] = round(timed(lambda: cg.conv(F, I, cp, "explicit", a.precision, out=O)), 1)
        except (cg.AllocationFailure, MemoryError) as e:  # B-hat beyond free device memory
            r["us_explicit"] = None
            r["explicit_error"] = str(e)[:120]
        cg.lib.cgb_scratch_release()
        cg.scratch_set_limit(limit)
        try:
            cg.conv(F, I, cp, "explicit", a.precision, out=O)
            torch.cuda.synchronize()
            r[f"explicit_under_{a.limit_gb:g}GB"] = "ok"
        except cg.AllocationFailure:
            r[f"explicit_under_{a.limit_gb:g}GB"] = "AllocationFailure"
        cg.conv(F, I, cp, "fused", a.precision, out=O)
        torch.cuda.synchronize()
        r[f"fused_under_{a.limit_gb:g}GB"] = "ok"
        cg.scratch_set_limit(0)
        cg.lib.cgb_scratch_release()
        rows.append(r)
        print(json.dumps(r), flush=True)
        del F, I, O
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"precision": a.precision, "limit_bytes": limit, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
