"""The BASELINE.json workloads as layer geometries (shared by bench.py, the tools and
the full-size parity tests).

Every config keeps the batch it is stated at in BASELINE.json ``configs``:
C1 b=8, C2 (ResNet-50 v1.5 3x3, the bench step) b=128, C3 (1x1) b=256, C4 (stem)
b=256, C5 (VGG-16, 13 layers) b=64. Input distributions follow BASELINE.json and
SURVEY.md §8(d): uniform[-1,1] for I and F, except the stem (I uniform[0,1],
F N(0, 0.05^2)).
"""
from __future__ import annotations

import zlib

# (name, k_n, k, c_i, h_i, s, p) -- square images and filters
C1 = [("c1_3x3_56_64", 64, 3, 64, 56, 1, 1)]
C2 = [
    ("r50_3x3_56_64", 64, 3, 64, 56, 1, 1),
    ("r50_3x3_28_128", 128, 3, 128, 28, 1, 1),
    ("r50_3x3_14_256", 256, 3, 256, 14, 1, 1),
    ("r50_3x3_7_512", 512, 3, 512, 7, 1, 1),
    ("r50_3x3_s2_56_128", 128, 3, 128, 56, 2, 1),
    ("r50_3x3_s2_28_256", 256, 3, 256, 28, 2, 1),
    ("r50_3x3_s2_14_512", 512, 3, 512, 14, 2, 1),
]
C3 = [
    ("pw_56_64_256", 256, 1, 64, 56, 1, 0),
    ("pw_14_1024_256", 256, 1, 1024, 14, 1, 0),
    ("pw_7_2048_512", 512, 1, 2048, 7, 1, 0),
    ("pw_7_512_2048", 2048, 1, 512, 7, 1, 0),
]
C4 = [("stem_7x7_s2_224", 64, 7, 3, 224, 2, 3)]
C5 = [
    ("vgg_224_3_64", 64, 3, 3, 224, 1, 1),
    ("vgg_224_64_64", 64, 3, 64, 224, 1, 1),
    ("vgg_112_64_128", 128, 3, 64, 112, 1, 1),
    ("vgg_112_128_128", 128, 3, 128, 112, 1, 1),
    ("vgg_56_128_256", 256, 3, 128, 56, 1, 1),
    ("vgg_56_256_256a", 256, 3, 256, 56, 1, 1),
    ("vgg_56_256_256b", 256, 3, 256, 56, 1, 1),
    ("vgg_28_256_512", 512, 3, 256, 28, 1, 1),
    ("vgg_28_512_512a", 512, 3, 512, 28, 1, 1),
    ("vgg_28_512_512b", 512, 3, 512, 28, 1, 1),
    ("vgg_14_512_512a", 512, 3, 512, 14, 1, 1),
    ("vgg_14_512_512b", 512, 3, 512, 14, 1, 1),
    ("vgg_14_512_512c", 512, 3, 512, 14, 1, 1),
]

CONFIGS = {  # config -> (stated batch, layers, input distribution)
    "C1": (8, C1, "uniform"),
    "C2": (128, C2, "uniform"),
    "C3": (256, C3, "uniform"),
    "C4": (256, C4, "stem"),
    "C5": (64, C5, "uniform"),
}


def layer_cp(layer, b):
    _, k_n, k, c_i, h_i, s, p = layer
    return dict(k_n=k_n, k_h=k, k_w=k, c_i=c_i, h_i=h_i, w_i=h_i, b=b, s=s, p=p)


def out_hw(cp):
    return ((cp["h_i"] - cp["k_h"] + 2 * cp["p"]) // cp["s"] + 1,
            (cp["w_i"] - cp["k_w"] + 2 * cp["p"]) // cp["s"] + 1)


def flops(cp):
    """BASELINE.json metric numerator: 2*k_n*h_o*w_o*b*k_h*k_w*c_i (bench.cpp:160-161)."""
    h_o, w_o = out_hw(cp)
    return 2 * cp["k_n"] * h_o * w_o * cp["b"] * cp["k_h"] * cp["k_w"] * cp["c_i"]


def nbytes(cp):
    """Compulsory HBM traffic 4*(|I| + |F| + |O|)."""
    h_o, w_o = out_hw(cp)
    return 4 * (cp["h_i"] * cp["w_i"] * cp["c_i"] * cp["b"] + cp["k_n"] * cp["k_h"] * cp["k_w"] * cp["c_i"]
                + cp["k_n"] * h_o * w_o * cp["b"])


def all_layers():
    """[(config, layer tuple, cp at the stated batch, distribution)] over C1..C5."""
    out = []
    for cfg, (b, layers, dist) in CONFIGS.items():
        for layer in layers:
            out.append((cfg, layer, layer_cp(layer, b), dist))
    return out


def layer_seed(name: str, base: int = 20177) -> int:
    """Stable per-layer seed (crc32, not Python's salted hash)."""
    return base + zlib.crc32(name.encode()) % 100000


def make_tensors(torch, empty_tensor4, cp, dist, seed, device="cuda"):
    """Seeded F, I (leftmost-fastest CUDA tensors) with the config's distribution."""
    g = torch.Generator(device=device).manual_seed(seed)
    F = empty_tensor4(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"], device=device)
    I = empty_tensor4(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"], device=device)
    if dist == "stem":
        F.copy_(torch.randn(F.shape, generator=g, device=device) * 0.05)
        I.copy_(torch.rand(I.shape, generator=g, device=device))
    else:
        F.copy_(torch.rand(F.shape, generator=g, device=device) * 2 - 1)
        I.copy_(torch.rand(I.shape, generator=g, device=device) * 2 - 1)
    return F, I
