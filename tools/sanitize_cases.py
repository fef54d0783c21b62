"""Small launches of every kernel family for compute-sanitizer (racecheck /
memcheck / synccheck on small configs): python tools/sanitize_cases.py
Each case is also checked against an fp64 torch convolution, so a sanitizer pass that
changed the result would show."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2005_06410_b200 as cg  # noqa: E402


def ref64(F, I, cp):
    # F: k_n,k_h,k_w,c_i ; I: h,w,c,b (logical shapes) -> O: k_n,h_o,w_o,b
    w = F.permute(0, 3, 1, 2).double()
    x = I.permute(3, 2, 0, 1).double()
    y = torch.nn.functional.conv2d(x, w, stride=cp["s"], padding=cp["p"])
    return y.permute(1, 2, 3, 0)


def run(name, cp, algo="fused", prec="tf32", **tune):
    g = torch.Generator(device="cuda").manual_seed(11)
    F = cg.empty_tensor4(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
    I = cg.empty_tensor4(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
    F.copy_(torch.rand(F.shape, generator=g, device="cuda") * 2 - 1)
    I.copy_(torch.rand(I.shape, generator=g, device="cuda") * 2 - 1)
    with cg.tuning(**tune):
        O = cg.conv(F, I, cp, algo=algo, precision=prec)
    torch.cuda.synchronize()
    err = float((O.double() - ref64(F, I, cp)).abs().max())
    k = cp["k_h"] * cp["k_w"] * cp["c_i"]
    tol = (2e-3 if prec == "tf32" else 2e-5) * k ** 0.5
    print(f"{name:28s} {algo:8s} {prec:6s} path={cg.last_path():22s} max abs err {err:.2e} {'ok' if err <= tol else 'FAIL'}",
          flush=True)
    assert err <= tol, name


c3 = dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=14, w_i=14, b=2, s=1, p=1)
for prec in ("tf32", "3xtf32"):
    run("shifted 3x3 pair", c3, prec=prec)
    run("shifted 3x3 single CTA", c3, prec=prec, pair=0)
    run("shifted stream-K forced", dict(c3, b=5), prec=prec, sk=2)
    run("shifted tail tiles forced", dict(c3, h_i=28, w_i=28, b=3), prec=prec, tail=2)
    run("shifted split-K", dict(k_n=128, k_h=3, k_w=3, c_i=128, h_i=7, w_i=7, b=2, s=1, p=1), prec=prec, splitk=3)
    run("shifted stride 2", dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=14, w_i=14, b=2, s=2, p=1), prec=prec)
    run("1x1 TMA-fed A", dict(k_n=64, k_h=1, k_w=1, c_i=64, h_i=8, w_i=8, b=3, s=1, p=0), prec=prec)
    run("w-im2col stem", dict(k_n=64, k_h=7, k_w=7, c_i=3, h_i=32, w_i=32, b=2, s=2, p=3), prec=prec)
    run("gather (waste > 1.7)", dict(k_n=32, k_h=3, k_w=3, c_i=16, h_i=4, w_i=4, b=3, s=1, p=3), prec=prec)
    run("reference-order implicit", dict(k_n=20, k_h=3, k_w=2, c_i=5, h_i=9, w_i=8, b=2, s=3, p=1), prec=prec)
    run("explicit K1+K2", c3, algo="explicit", prec=prec, k2_flo=-1)
    run("explicit K1+K2 filter-lo", c3, algo="explicit", prec=prec, k2_flo=1)
    run("explicit K2 split-K", dict(k_n=256, k_h=3, k_w=3, c_i=64, h_i=6, w_i=6, b=2, s=1, p=1), algo="explicit",
        prec=prec, splitk=4)
run("ffma implicit", c3, prec="ffma")
run("ffma explicit", c3, algo="explicit", prec="ffma")
run("conv_direct", dict(c3, b=1), algo="direct", prec="ffma")
print("all cases ok")
