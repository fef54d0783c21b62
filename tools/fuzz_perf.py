#!/usr/bin/env python
"""Throughput of the large random geometries of tests/test_fuzz_gpu.py (draw_big): which
kernel takes each, time, TFLOP/s and roofline fraction -- a look for dispatch outliers away
from the BASELINE shapes. python tools/fuzz_perf.py [--precision tf32] [--n 32]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2005_06410_b200 as cg  # noqa: E402
from test_fuzz_gpu import draw_big  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="tf32")
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--tune", default="{}", help="JSON of cgb_set_tuning knobs")
a = ap.parse_args()
import json  # noqa: E402
for k, v in json.loads(a.tune).items():
    cg.set_tuning(k, v)
pk = bench.peaks()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
for seed in range(a.n):
    cp = draw_big(seed)
    g = torch.Generator(device="cuda").manual_seed(seed)
    F = cg.empty_tensor4(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
    I = cg.empty_tensor4(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
    F.copy_(torch.rand(F.shape, generator=g, device="cuda") * 2 - 1)
    I.copy_(torch.rand(I.shape, generator=g, device="cuda") * 2 - 1)
    O = cg.conv(F, I, cp, precision=a.precision)
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cg.conv(F, I, cp, precision=a.precision, out=O)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[2] * 1e-3
    fl, by = bench.flops(cp), bench.nbytes(cp)
    floor = max(fl / (pk["tf32_tflops"] * 1e12) * (3 if a.precision in ("auto", "3xtf32") else 1), by / (pk["hbm_gbs"] * 1e9))
    rows.append((floor / t, cp, t, fl, cg.last_path()))
for frac, cp, t, fl, path in sorted(rows, key=lambda r: r[0]):
    print(f"{frac:5.2f}  {t * 1e6:8.1f} us  {fl / t / 1e12:6.1f} TFLOP/s  {path:22s} "
          f"{cp['k_n']}x{cp['k_h']}x{cp['k_w']}x{cp['c_i']} on {cp['h_i']}x{cp['w_i']} b={cp['b']} s={cp['s']} p={cp['p']}")
