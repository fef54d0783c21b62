"""Full-batch fp64 cross-check on the device -- TEST INFRASTRUCTURE (also used by
bench.py's parity block, after the timed region).

The CPU oracle (oracle/) is the parity anchor, but at BASELINE batch sizes it only
finishes on sampled images. This checker covers EVERY output of a full-batch launch:
the convolution recomputed in float64 by torch (cuDNN fp64, accumulation error
~1e-16, far below the 1e-5 bar), and the north-star per-output error
|O - O_ref| / (||F[i_k]|| * ||B[:, col]||) -- the same normalisation as
oracle.per_output_error -- with ||B[:, col]||^2 = conv(I^2, ones) (the squared norm of
the lowered column, im2col.hpp:71-76, zero padding included).
"""
from __future__ import annotations


def nchw(torch, I):
    """I (h, w, c, b) leftmost-fastest -> (b, c, h, w) view."""
    return I.permute(3, 2, 1, 0).permute(0, 1, 3, 2)


def per_output_error_fp64(torch, F, I, O, cp, chunk=None):
    """Max normalised per-output error of O against an fp64 recomputation (all images)."""
    import torch.nn.functional as tf
    b = cp["b"]
    s, p = cp["s"], cp["p"]
    W = F.permute(0, 3, 1, 2).to(torch.float64)  # (k_n, c_i, k_h, k_w)
    fn = W.pow(2).sum(dim=(1, 2, 3)).sqrt()  # ||F[i_k]||
    ones = torch.ones((1, cp["c_i"], cp["k_h"], cp["k_w"]), dtype=torch.float64, device=F.device)
    if chunk is None:
        per_img = cp["h_i"] * cp["w_i"] * cp["c_i"] * 8 * 3 + cp["k_n"] * cp["h_i"] * cp["w_i"] * 8 * 3
        chunk = max(1, min(b, (2 << 30) // max(per_img, 1)))
    worst = 0.0
    for i0 in range(0, b, chunk):
        i1 = min(b, i0 + chunk)
        x = nchw(torch, I[..., i0:i1]).to(torch.float64)
        # (b, c, h, w) with h = first spatial index: conv over (h, w) with (k_h, k_w)
        ref = tf.conv2d(x, W, stride=s, padding=p)  # (b, k_n, h_o, w_o)
        bn = tf.conv2d(x * x, ones, stride=s, padding=p).sqrt()  # (b, 1, h_o, w_o)
        got = O[..., i0:i1].permute(3, 0, 1, 2).to(torch.float64)  # (b, k_n, h_o, w_o)
        scale = fn.view(1, -1, 1, 1) * bn
        d = (got - ref).abs()
        e = torch.where(scale > 0, d / torch.where(scale > 0, scale, torch.ones_like(scale)), d)
        worst = max(worst, float(e.max()))
        del x, ref, bn, got, d, e, scale
    return worst
