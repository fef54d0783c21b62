"""Timings of the explicit path's kernels and the fc GEMMs (CUDA events, L2 flushed
before every launch): K1 im2col alone, the explicit conv (K1 + K2), fc6/fc7/fc8 of VGG-16
at b=64 in TF32 and 3xTF32. Prints one line per case with the HBM floor beside it."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2005_06410_b200 as cg  # noqa: E402
from paper_2005_06410_b200 import configs  # noqa: E402

HBM = 6539.2e9
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


by = {l[0]: (c, l, cp, d) for c, l, cp, d in configs.all_layers()}
for name in ("r50_3x3_56_64", "r50_3x3_28_128", "r50_3x3_7_512", "r50_3x3_s2_56_128", "stem_7x7_s2_224", "pw_56_64_256"):
    c, l, cp, d = by[name]
    F, I = configs.make_tensors(torch, cg.empty_tensor4, cp, d, 7)
    m, n, k = cg.gemm_dims(cp)
    ldb = (k + 3) // 4 * 4
    B = torch.empty((n, ldb), device="cuda")
    t1 = timed(lambda: cg.im2col(I, cp, ldb=ldb, out=B))
    bhat = 4 * ldb * n
    io = 4 * (I.numel() + F.numel() + m * n)
    line = f"{name:20s} b={cp['b']:3d} Bhat {bhat/1e6:7.1f} MB  K1 {t1:7.1f} us ({(bhat + 4*I.numel())/t1/1e3:6.0f} GB/s)"
    for prec, flo in (("tf32", 0), ("3xtf32", -1), ("3xtf32", 1)):
        with cg.tuning(k2_flo=flo):
            te = timed(lambda: cg.conv(F, I, cp, algo="explicit", precision=prec))
        tf = timed(lambda: cg.conv(F, I, cp, algo="fused", precision=prec))
        floor = (2 * bhat + io) / HBM * 1e6
        line += f" | {prec}{'/flo' if flo > 0 else ''}: explicit {te:7.1f} us (K2 ~{te - t1:6.1f}; floor {floor:5.0f}) fused {tf:6.1f}"
    print(line, flush=True)
    del B, F, I

g = torch.Generator(device="cuda").manual_seed(3)
for name, m, k in (("fc6", 4096, 25088), ("fc7", 4096, 4096), ("fc8", 1000, 4096)):
    for n in (64, 256):
        A = (torch.rand((k, m), generator=g, device="cuda") * 2 - 1).t()
        B = (torch.rand((n, k), generator=g, device="cuda") * 2 - 1).t()
        C = torch.empty((n, m), device="cuda").t()
        line = f"{name} {m}x{k} n={n:3d} weights {4*m*k/1e6:6.1f} MB floor {4*(m*k + k*n + m*n)/HBM*1e6:5.1f} us"
        for prec in ("tf32", "3xtf32"):
            t = timed(lambda: cg.gemm(A, B, precision=prec, out=C))
            line += f" | {prec} {t:7.1f} us ({2*m*n*k/t/1e6:6.1f} TFLOP/s, {4*m*k/t/1e3:5.0f} GB/s)"
        print(line, flush=True)
