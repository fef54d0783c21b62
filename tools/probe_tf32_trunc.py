"""Probe (DESIGN §9 item 2): what does the tcgen05 kind::tf32 MMA do with the low 13
mantissa bits of raw fp32 operands — truncate, round to nearest, or keep them?

One nonzero channel per output so no accumulation rounding interferes: O = F · x with
F = 1 and x = 1 + m·2^-13 for m = 0..15 (bits below the tf32 mantissa). Run on each
operand path: the 1x1 layer with h*w % 4 == 0 goes through the TMA-fed A path (raw fp32
straight from I), the 3x3 layer through the producer-staged window.
"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2005_06410_b200 as cg


def dev(a):
    a = np.asfortranarray(a, dtype=np.float32); d = a.shape
    return torch.from_numpy(a.reshape(-1, order='F').copy()).cuda().view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0)


def host(t):
    d = t.shape; return t.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy().reshape(d, order='F')


def tf32_trunc(x):
    return (np.asarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def tf32_rn(x):  # round half away from zero on the 13 dropped bits (cvt.rna.tf32.f32)
    u = np.asarray(x, np.float32).view(np.uint32)
    return ((u + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


def probe(name, kh, hi, wi, p):
    kn, ci, b = 128, 32, 1
    F = np.zeros((kn, kh, kh, ci), np.float32, order='F')
    F[:, kh // 2, kh // 2, 0] = 1.0            # centre tap, channel 0 only
    I = np.zeros((hi, wi, ci, b), np.float32, order='F')
    m = np.arange(hi * wi) % 16
    I[:, :, 0, 0] = (1.0 + m * 2.0 ** -13).reshape(hi, wi, order='F').astype(np.float32)
    cp = dict(k_n=kn, k_h=kh, k_w=kh, c_i=ci, h_i=hi, w_i=wi, b=b, s=1, p=p)
    O = host(cg.conv(dev(F), dev(I), cp, precision='tf32'))[0, :, :, 0]
    x = I[:, :, 0, 0]
    verdict = {k: bool(np.array_equal(O, f(x))) for k, f in
               (("truncate", tf32_trunc), ("round", tf32_rn), ("full_fp32", lambda v: v))}
    print(name, verdict, "sample x:", x.ravel(order='F')[:8], "O:", O.ravel(order='F')[:8])
    return verdict


def probe_filter(name, kh, hi, wi, p):
    """Same on the filter operand: F[n] = 1 + (n % 16)·2^-13 on the centre tap, I = 1."""
    kn, ci, b = 128, 32, 1
    F = np.zeros((kn, kh, kh, ci), np.float32, order='F')
    F[:, kh // 2, kh // 2, 0] = (1.0 + (np.arange(kn) % 16) * 2.0 ** -13).astype(np.float32)
    I = np.zeros((hi, wi, ci, b), np.float32, order='F'); I[:, :, 0, 0] = 1.0
    cp = dict(k_n=kn, k_h=kh, k_w=kh, c_i=ci, h_i=hi, w_i=wi, b=b, s=1, p=p)
    O = host(cg.conv(dev(F), dev(I), cp, precision='tf32'))[:, 0, 0, 0]
    x = F[:, kh // 2, kh // 2, 0]
    verdict = {k: bool(np.array_equal(O, f(x))) for k, f in
               (("truncate", tf32_trunc), ("round", tf32_rn), ("full_fp32", lambda v: v))}
    print(name, verdict, "O:", O[:8])
    return verdict


if __name__ == "__main__":
    probe_filter("filter operand 1x1", 1, 16, 16, 0)
    probe_filter("filter operand 3x3", 3, 16, 16, 1)
    v1 = probe("1x1 TMA-fed A (16x16)", 1, 16, 16, 0)
    v3 = probe("3x3 staged window (16x16)", 3, 16, 16, 1)
    print("RESULT", {"1x1": v1, "3x3": v3})
