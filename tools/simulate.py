#!/usr/bin/env python
"""Run the inference simulator (paper_2005_06410_b200.run_inference, the reference's
run_inference/bench.cpp) over the built-in VGG-16 and ResNet-50 definitions and write the
reference's CSV: python tools/simulate.py --batch 64 --algo convgemm --precision tf32 --out DIR"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _prof  # noqa: E402,F401  (profiling build: CGB_* env knobs)
import paper_2005_06410_b200 as cg  # noqa: E402
from paper_2005_06410_b200 import models  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--models", default="alexnet,vgg16,resnet50")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--algo", default="convgemm")
ap.add_argument("--precision", default="tf32")
ap.add_argument("--min-time", type=float, default=0.05)
ap.add_argument("--check", action="store_true")
ap.add_argument("--out", default=".")
ap.add_argument("--tune", default="{}", help="JSON of cgb_set_tuning knobs")
a = ap.parse_args()
import json  # noqa: E402
for k, v in json.loads(a.tune).items():
    cg.set_tuning(k, v)
for name in a.models.split(","):
    m = models.MODELS[name]()
    rs = cg.run_inference(m, a.batch, algo=a.algo, min_time=a.min_time, check=a.check, precision=a.precision)
    path = os.path.join(a.out, f"sim_{name}_b{a.batch}_{a.algo}_{a.precision}.csv")
    cg.write_csv(path, m, a.batch, a.algo, 1, rs)
    tot_t = sum(r.time_s for r in rs)
    tot_f = sum(r.gflops * r.time_s for r in rs)
    print(f"{name} b={a.batch} {a.algo}/{a.precision}: {len(rs)} layers, {tot_t * 1e3:.2f} ms, "
          f"{tot_f / tot_t / 1e3:.1f} TFLOP/s -> {path}")
