#!/usr/bin/env python
"""Dispatch check away from the BASELINE shapes: for each random large geometry
(tests/test_fuzz_gpu.py draw_big) time the default dispatch against forced alternatives
(M tile, CTA pairs, stream-K, split-K, tail tiles) and list the geometries where an
alternative wins by more than 10%. python tools/fuzz_dispatch.py [--n 32] [--precision tf32]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_2005_06410_b200 as cg  # noqa: E402
from test_fuzz_gpu import draw_big  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="tf32")
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--first", type=int, default=0)
ap.add_argument("--bn-only", action="store_true", help="only the filter-tile variants, all timings printed")
ap.add_argument("--kn", default="", help="comma list: override k_n of every geometry with each of these")
a = ap.parse_args()
VARIANTS = [{}, {"mt": 1}, {"mt": 2}, {"mt": 4}, {"pair": 0}, {"sk": 0}, {"sk": 2}, {"splitk": -1}, {"splitk": 2},
            {"splitk": 4}, {"tail": 0}, {"bn": 64}, {"bn": 128}, {"bn": 256}]
if a.bn_only:
    VARIANTS = [{}, {"bn": 64}, {"bn": 128}, {"bn": 256}]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(F, I, cp, O):
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cg.conv(F, I, cp, precision=a.precision, out=O)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[2] * 1e3


jobs = []
for seed in range(a.first, a.first + a.n):
    cp = draw_big(seed)
    if a.kn:
        jobs += [(seed, dict(cp, k_n=int(k))) for k in a.kn.split(",")]
    else:
        jobs.append((seed, cp))
for seed, cp in jobs:
    g = torch.Generator(device="cuda").manual_seed(seed)
    F = cg.empty_tensor4(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
    I = cg.empty_tensor4(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
    F.copy_(torch.rand(F.shape, generator=g, device="cuda") * 2 - 1)
    I.copy_(torch.rand(I.shape, generator=g, device="cuda") * 2 - 1)
    O = cg.conv(F, I, cp, precision=a.precision)
    res = []
    for v in VARIANTS:
        try:
            with cg.tuning(**v):
                cg.conv(F, I, cp, precision=a.precision, out=O)
                res.append((timed(F, I, cp, O), v, cg.last_path()))
        except Exception as ex:  # noqa: BLE001
            res.append((float("inf"), v, type(ex).__name__))
    base = res[0][0]
    best = min(res, key=lambda r: r[0])
    if a.bn_only:
        print(f"{cp['k_n']}x{cp['k_h']}x{cp['k_w']}x{cp['c_i']} on {cp['h_i']}x{cp['w_i']} b={cp['b']} s={cp['s']} p={cp['p']}: "
              + "  ".join(f"{'def' if not v else v['bn']}:{t:6.1f}" for t, v, _ in res))
        continue
    flag = "  <-- " if best[0] < 0.9 * base else "      "
    print(f"{cp['k_n']}x{cp['k_h']}x{cp['k_w']}x{cp['c_i']} on {cp['h_i']}x{cp['w_i']} b={cp['b']} s={cp['s']} p={cp['p']}: "
          f"default {base:7.1f} us{flag}best {best[0]:7.1f} us {best[1]} {best[2]}")
