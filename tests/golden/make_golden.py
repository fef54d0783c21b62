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
    path = os.path.join(HERE, "reference_conv.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
