#!/usr/bin/env python
"""Shifted window vs the tap-major gather kernel on geometries whose padded plane has many
more rows than outputs (unpadded large filters on small images): time per kernel by the
waste_pct tuning knob. python tools/waste_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2005_06410_b200 as cg  # noqa: E402

CASES = [  # k_n, k, c_i, h, s, p, b
    (512, 5, 192, 7, 1, 0, 64), (256, 7, 16, 20, 1, 0, 50), (256, 5, 128, 6, 1, 0, 128), (256, 7, 64, 9, 1, 0, 128),
    (256, 7, 64, 8, 1, 0, 128), (512, 7, 64, 7, 1, 0, 256), (128, 5, 64, 12, 2, 0, 128), (256, 3, 256, 4, 1, 0, 256),
    (256, 3, 256, 3, 1, 0, 512), (128, 5, 32, 30, 1, 0, 32), (64, 7, 32, 14, 1, 1, 64)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k_n, k, c_i, h, s, p, b in CASES:
    cp = dict(k_n=k_n, k_h=k, k_w=k, c_i=c_i, h_i=h, w_i=h, b=b, s=s, p=p)
    h_o, w_o = cg.output_dims(cp)
    g = torch.Generator(device="cuda").manual_seed(1)
    F = cg.empty_tensor4(k_n, k, k, c_i)
    I = cg.empty_tensor4(h, h, c_i, b)
    F.copy_(torch.rand(F.shape, generator=g, device="cuda") * 2 - 1)
    I.copy_(torch.rand(I.shape, generator=g, device="cuda") * 2 - 1)
    out = []
    for w in (100, 1000000):
        with cg.tuning(waste_pct=w):
            O = cg.conv(F, I, cp, precision="tf32")
            ts = []
            for _ in range(7):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                cg.conv(F, I, cp, precision="tf32", out=O)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            out.append((sorted(ts)[3] * 1e3, cg.last_path()))
    fl = 2.0 * k_n * h_o * w_o * b * k * k * c_i
    print(f"{k_n}x{k}x{k}x{c_i} on {h}x{h} s={s} p={p} b={b} out {h_o}x{w_o} {fl / 1e9:5.1f} GFLOP: "
          f"{out[0][1]} {out[0][0]:7.1f} us | {out[1][1]} {out[1][0]:7.1f} us")
