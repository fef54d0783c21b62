"""Built-in model definitions for the simulator, generated from the architectures' rules
(the layer-geometry convention of the reference's model files, models/*.model: one line
per conv / fc / pool, conv geometry at batch 1).

* ``vgg16()`` -- thirteen 3x3/s1/p1 convolutions in five blocks of 2, 2, 3, 3, 3 (widths
  64, 128, 256, 512, 512), a 2x2 pool after each block, fc 4096, 4096, 1000.
* ``resnet50()`` -- ResNet-50 v1 bottlenecks: 7x7/s2/p3 stem, stem pool to 56x56, then
  stages of 3, 4, 6, 3 blocks (widths 64, 128, 256, 512, expansion 4). The stride sits on
  the block's first 1x1 conv (v1), and a projection shortcut (1x1, same stride) follows
  the three convs of the first block of every stage; fc 1000.

* ``alexnet()`` -- the five convolutions of the single-tower AlexNet (11x11/s4, 5x5, three
  3x3; widths 64, 192, 384, 384, 256), pools to 26, 13 and 6, fc 4096, 4096, 1000. The
  reference's file lists every conv unpadded and with the input extents 224, 55, 27, 13,
  13 (each line is an independent layer geometry, not a shape-propagated chain); the
  same table is kept here so the sweep times the same GEMMs (m x n x k) as the reference.

All can be written out as model text (``ModelSpec.to_text``) and parsed back.
"""
from __future__ import annotations

from .simulator import LayerSpec, ModelSpec


def _conv(k_n, k, c_i, h, s, p):
    from . import ConvParams
    return LayerSpec("conv", conv=ConvParams(k_n, k, k, c_i, h, h, 1, s, p))


def vgg16() -> ModelSpec:
    m = ModelSpec("vgg16")
    h, c = 224, 3
    for width, convs in ((64, 2), (128, 2), (256, 3), (512, 3), (512, 3)):
        for _ in range(convs):
            m.layers.append(_conv(width, 3, c, h, 1, 1))
            c = width
        h //= 2
        m.layers.append(LayerSpec("pool", pool_h=h, pool_w=h, pool_c=c))
    k = h * h * c
    for out in (4096, 4096, 1000):
        m.layers.append(LayerSpec("fc", fc_m=out, fc_k=k))
        k = out
    return m


def resnet50() -> ModelSpec:
    m = ModelSpec("resnet50")
    m.layers.append(_conv(64, 7, 3, 224, 2, 3))
    h, c = 56, 64
    m.layers.append(LayerSpec("pool", pool_h=h, pool_w=h, pool_c=c))
    for stage, (width, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        for blk in range(blocks):
            s = 2 if (stage > 0 and blk == 0) else 1
            h_out = h // s
            m.layers.append(_conv(width, 1, c, h, s, 0))
            m.layers.append(_conv(width, 3, width, h_out, 1, 1))
            m.layers.append(_conv(4 * width, 1, width, h_out, 1, 0))
            if blk == 0:
                m.layers.append(_conv(4 * width, 1, c, h, s, 0))  # projection shortcut
            c, h = 4 * width, h_out
    m.layers.append(LayerSpec("fc", fc_m=1000, fc_k=c))
    return m


def alexnet() -> ModelSpec:
    m = ModelSpec("alexnet")
    # (filters, kernel, stride, input extent) per conv; a pool (output extent) follows where given
    table = ((64, 11, 4, 224, 26), (192, 5, 1, 55, 13), (384, 3, 1, 27, None), (384, 3, 1, 13, None),
             (256, 3, 1, 13, 6))
    c = 3
    for width, k, s, h, pool in table:
        m.layers.append(_conv(width, k, c, h, s, 0))
        c = width
        if pool:
            m.layers.append(LayerSpec("pool", pool_h=pool, pool_w=pool, pool_c=c))
    k = 6 * 6 * c
    for out in (4096, 4096, 1000):
        m.layers.append(LayerSpec("fc", fc_m=out, fc_k=k))
        k = out
    return m


MODELS = {"alexnet": alexnet, "vgg16": vgg16, "resnet50": resnet50}
