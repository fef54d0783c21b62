"""Generate tests/golden/*.npz from the REFERENCE itself (run in the build
container, where /root/reference exists; the fixtures travel, the reference
does not).

Inputs come from the reference tests' own generator streams
(proj/tests/oracles.hpp:48-91: std::mt19937_64, uniform[-1,1] drawn in double
and cast), outputs from the reference operator compiled from its sources
(oracle/_ref/libconvgemm_ref.so -> conv_gemm / conv_im2col_gemm / conv_direct /
im2col, proj/include/convgemm/conv.hpp:24-91, im2col.hpp:77-120).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference  # noqa: E402

KEYS = ("k_n", "k_h", "k_w", "c_i", "h_i", "w_i", "b", "s", "p")


def cp_vec(cp):
    return np.array([cp[k] for k in KEYS], dtype=np.int64)


def main():
    R = Reference()
    out = {}
    # 1. acceptance criterion 1 stream (acceptance.cpp:51-85, seed 101): the first
    #    64 random configs with their inputs, drawn in the reference's order.
    g = R.rng(101)
    for i in range(64):
        cp = g.conv_params(8, 3)
        F = g.tensor(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
        I = g.tensor(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
        threads = i % 3 + 1
        out[f"rand{i}_cp"] = cp_vec(cp)
        out[f"rand{i}_F"] = F
        out[f"rand{i}_I"] = I
        out[f"rand{i}_O"] = R.conv_gemm(F, I, cp, threads=threads)
        out[f"rand{i}_Odirect"] = R.conv_direct(F, I, cp)
        out[f"rand{i}_B"] = R.im2col(I, cp, threads=threads)
    out["n_rand"] = np.array(64)
    # 2. medium shapes covering BASELINE geometry classes at small extents
    #    (3x3 s1 p1, 3x3 s2, 1x1, 7x7 s2 p3 low-c_i stem, K > kc=640 two blocks,
    #    non-multiple-of-4 filter counts, batch-straddling pixel tiles).
    medium = [
        dict(k_n=32, k_h=3, k_w=3, c_i=32, h_i=14, w_i=14, b=2, s=1, p=1),
        dict(k_n=48, k_h=3, k_w=3, c_i=24, h_i=15, w_i=15, b=2, s=2, p=1),
        dict(k_n=64, k_h=1, k_w=1, c_i=64, h_i=7, w_i=7, b=3, s=1, p=0),
        dict(k_n=16, k_h=7, k_w=7, c_i=3, h_i=30, w_i=30, b=2, s=2, p=3),
        dict(k_n=40, k_h=3, k_w=3, c_i=96, h_i=9, w_i=9, b=2, s=1, p=1),
        dict(k_n=13, k_h=3, k_w=2, c_i=5, h_i=11, w_i=10, b=3, s=1, p=0),
        dict(k_n=64, k_h=3, k_w=3, c_i=3, h_i=16, w_i=16, b=2, s=1, p=1),
    ]
    g = R.rng(36)
    for i, cp in enumerate(medium):
        F = g.tensor(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
        I = g.tensor(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
        out[f"med{i}_cp"] = cp_vec(cp)
        out[f"med{i}_F"] = F
        out[f"med{i}_I"] = I
        out[f"med{i}_O"] = R.conv_gemm(F, I, cp, threads=2)
        out[f"med{i}_Oexplicit"] = R.conv_im2col_gemm(F, I, cp, threads=3)
    out["n_med"] = np.array(len(medium))
    # 3. float64 (the reference's f64 instantiations, README.md:38-40): conv_gemm /
    #    conv_im2col_gemm / conv_direct / im2col at double precision on the acceptance
    #    stream (seed 202), plus two shapes with K > kc (two and four kc blocks, the second
    #    with kc = 100) and a gemm -- the device f64 path must match these bit for bit.
    g = R.rng(202)
    f64_cases = [g.conv_params(8, 3) for _ in range(24)]
    f64_cases += [dict(k_n=40, k_h=3, k_w=3, c_i=96, h_i=9, w_i=9, b=2, s=1, p=1),
                  dict(k_n=24, k_h=3, k_w=3, c_i=40, h_i=8, w_i=7, b=2, s=2, p=1)]
    kcs = [640] * 25 + [100]
    for i, cp in enumerate(f64_cases):
        F = g.tensor(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"], dtype=np.float64)
        I = g.tensor(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"], dtype=np.float64)
        bp = (120, 3072, kcs[i], 8, 12)
        out[f"f64_{i}_cp"] = cp_vec(cp)
        out[f"f64_{i}_kc"] = np.array(kcs[i])
        out[f"f64_{i}_F"] = F
        out[f"f64_{i}_I"] = I
        out[f"f64_{i}_O"] = R.conv_gemm(F, I, cp, threads=2, bp=bp)
        out[f"f64_{i}_Oexplicit"] = R.conv_im2col_gemm(F, I, cp, threads=1, bp=bp)
        out[f"f64_{i}_Odirect"] = R.conv_direct(F, I, cp)
        out[f"f64_{i}_B"] = R.im2col(I, cp)
    out["n_f64"] = np.array(len(f64_cases))
    A = g.tensor(37, 700, 1, 1, dtype=np.float64).reshape(37, 700, order="F")
    Bm = g.tensor(700, 19, 1, 1, dtype=np.float64).reshape(700, 19, order="F")
    out["f64_gemm_A"], out["f64_gemm_B"] = A, Bm
    out["f64_gemm_C"] = R.gemm(A, Bm, threads=2)
    path = os.path.join(HERE, "reference_conv.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
