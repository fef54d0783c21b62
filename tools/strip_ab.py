#!/usr/bin/env python
"""h-strips for wide stride-1 images (tuning strip_h): outputs against the default dispatch
(bitwise) and time per layer. python tools/strip_ab.py [--batch 64]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2005_06410_b200 as cg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--strips", default="0,28,56,75,112")
ap.add_argument("--precision", default="tf32")
a = ap.parse_args()
CASES = [(64, 3, 64, 224, 1), (128, 3, 64, 112, 1), (128, 3, 128, 112, 1), (256, 3, 128, 56, 1), (64, 3, 64, 150, 1),
         (64, 5, 32, 131, 2), (96, 3, 48, 201, 0)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k_n, k, c_i, h, p in CASES:
    cp = dict(k_n=k_n, k_h=k, k_w=k, c_i=c_i, h_i=h, w_i=h if h != 201 else 37, b=a.batch, s=1, p=p)
    g = torch.Generator(device="cuda").manual_seed(3)
    F = cg.empty_tensor4(k_n, k, k, c_i)
    I = cg.empty_tensor4(cp["h_i"], cp["w_i"], c_i, a.batch)
    F.copy_(torch.rand(F.shape, generator=g, device="cuda") * 2 - 1)
    I.copy_(torch.rand(I.shape, generator=g, device="cuda") * 2 - 1)
    ref = None
    out = []
    for sh in [int(x) for x in a.strips.split(",")]:
        with cg.tuning(strip_h=sh):
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
        if ref is None:
            ref = O.clone()
        same = torch.equal(O, ref)
        maxd = float((O - ref).abs().max())
        out.append(f"{sh}:{sorted(ts)[2] * 1e3:7.1f}us{'=' if same else f'!{maxd:.1e}'}")
    print(f"{k_n}x{k}x{k}x{c_i} on {cp['h_i']}x{cp['w_i']} p={p} b={a.batch}: " + "  ".join(out))
