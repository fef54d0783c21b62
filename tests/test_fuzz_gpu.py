"""Seeded random-geometry sweep of the B200 operator against the oracle, at sizes between
the reference's acceptance stream (extents <= 8, tests/golden) and the BASELINE configs.

The reference's acceptance test draws its geometries from a generator stream
(/root/reference/proj/tests/acceptance.cpp:51-85) capped at tiny extents; the dispatcher
here has many more branches than the reference (shifted window / w-im2col / TMA-fed 1x1 /
tap-major gather / reference-order implicit GEMM / explicit K1+K2 / FFMA, CTA pairs,
stream-K, split-K, tail tiles), chosen by geometry. This sweep draws geometries that land
on all of them -- non-square filters and images, strides 1-4, padding 0-3, channel
counts around the 16/32-channel chunk edges, filter counts that are not multiples of 4 or
32, ragged batches -- and checks every output against the plain-C restatement (pinned
bitwise to the reference) under the north-star per-output bars.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2005_06410_b200 as cg  # noqa: E402
from oracle.oracle import Restatement, output_dims_py, per_output_error  # noqa: E402
from test_parity_gpu import TOL, rand_inputs, to_dev, to_host  # noqa: E402

N_CASES = 128


def draw(seed):
    """One geometry; 0.002-0.8 GFLOP so the oracle takes about a second at most."""
    rng = np.random.default_rng(7000 + seed)
    while True:
        k_h = int(rng.choice([1, 1, 2, 3, 3, 3, 4, 5, 7, 11]))
        k_w = k_h if rng.random() < 0.7 else int(rng.choice([1, 2, 3, 5, 7]))
        s = int(rng.choice([1, 1, 1, 2, 2, 3, 4]))
        p = int(rng.integers(0, min(3, max(k_h, k_w)) + 1))
        c_i = int(rng.choice([1, 3, 4, 8, 15, 16, 17, 24, 31, 32, 33, 48, 64, 96, 100, 128, 160, 256]))
        k_n = int(rng.choice([1, 3, 4, 10, 16, 30, 32, 36, 64, 96, 100, 128, 192, 256, 260, 512]))
        h_i = int(rng.integers(max(1, k_h - 2 * p), 60))
        w_i = h_i if rng.random() < 0.6 else int(rng.integers(max(1, k_w - 2 * p), 60))
        b = int(rng.choice([1, 2, 3, 5, 8, 13, 24, 40, 64]))
        cp = dict(k_n=k_n, k_h=k_h, k_w=k_w, c_i=c_i, h_i=h_i, w_i=w_i, b=b, s=s, p=p)
        if h_i + 2 * p < k_h or w_i + 2 * p < k_w:
            continue
        h_o, w_o = output_dims_py(cp)
        fl = 2.0 * k_n * h_o * w_o * b * k_h * k_w * c_i
        if 2e6 <= fl <= 8e8:
            return cp


@pytest.fixture(scope="module")
def orc():
    return Restatement()


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_geometry(orc, seed):
    cp = draw(seed)
    F, I = rand_inputs(cp, 8000 + seed)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    dF, dI = to_dev(F), to_dev(I)
    seen = []
    for algo, prec in (("fused", "auto"), ("fused", "tf32"), ("explicit", "auto"), ("explicit", "tf32")):
        O = to_host(cg.conv(dF, dI, cp, algo=algo, precision=prec))
        seen.append(cg.last_path())
        err = per_output_error(O, ref, scale)
        assert err <= TOL[prec], (cp, algo, prec, cg.last_path(), err)
    # the fp32-accurate default twice: bitwise reproducible whatever path took it
    a = cg.conv(dF, dI, cp, algo="fused", precision="auto")
    b = cg.conv(dF, dI, cp, algo="fused", precision="auto")
    assert torch.equal(a, b), (cp, seen)


def test_sweep_reaches_every_kernel_family():
    """The drawn geometries are not all taken by one kernel: the sweep is only worth its
    time if the dispatcher's branches are exercised."""
    paths = set()
    for seed in range(N_CASES):
        cp = draw(seed)
        F, I = rand_inputs(cp, 8000 + seed)
        for prec in ("auto", "tf32"):
            cg.conv(to_dev(F), to_dev(I), cp, algo="fused", precision=prec)
            paths.add(cg.last_path())
    assert len(paths) >= 4, paths


# ---------------------------------------------------------------- large random geometries
N_BIG = 32


def draw_big(seed):
    """Geometries of 2-25 GFLOP (hundreds to thousands of tiles: CTA pairs, tail tiles,
    stream-K rounds, split-K, wide windows), the sizes where the dispatcher's cost model
    decides; too big for the CPU oracle on every image."""
    rng = np.random.default_rng(9100 + seed)
    while True:
        k = int(rng.choice([1, 3, 3, 3, 5, 7]))
        s = int(rng.choice([1, 1, 2]))
        p = int(rng.choice([0, k // 2, k // 2]))
        c_i = int(rng.choice([3, 16, 32, 48, 64, 96, 128, 192, 256, 384, 512]))
        k_n = int(rng.choice([32, 64, 96, 128, 192, 256, 320, 512]))
        h_i = int(rng.choice([7, 12, 14, 20, 27, 28, 33, 56, 64, 75, 112]))
        w_i = h_i if rng.random() < 0.7 else int(rng.choice([7, 14, 20, 28, 40, 56]))
        b = int(rng.choice([5, 16, 24, 32, 50, 64, 100, 128]))
        cp = dict(k_n=k_n, k_h=k, k_w=k, c_i=c_i, h_i=h_i, w_i=w_i, b=b, s=s, p=p)
        if h_i + 2 * p < k or w_i + 2 * p < k:
            continue
        h_o, w_o = output_dims_py(cp)
        fl = 2.0 * k_n * h_o * w_o * b * k * k * c_i
        io_bytes = 4.0 * (h_i * w_i * c_i * b + k_n * h_o * w_o * b)
        if 2e9 <= fl <= 2.5e10 and io_bytes <= 1.5e9:
            return cp


@pytest.mark.parametrize("seed", range(N_BIG))
def test_random_geometry_large(orc, seed):
    from fp64ref import per_output_error_fp64
    cp = draw_big(seed)
    g = torch.Generator(device="cuda").manual_seed(9200 + seed)
    F = cg.empty_tensor4(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
    I = cg.empty_tensor4(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
    F.copy_(torch.rand(F.shape, generator=g, device="cuda") * 2 - 1)
    I.copy_(torch.rand(I.shape, generator=g, device="cuda") * 2 - 1)
    img = cp["b"] // 2  # one image against the oracle (the anchor), every output against fp64
    cp1 = dict(cp, b=1)
    Fh, Ih = to_host(F), to_host(I[..., img:img + 1])
    ref = orc.conv_gemm(np.asfortranarray(Fh), np.asfortranarray(Ih), cp1)
    scale = orc.output_scale(np.asfortranarray(Fh), np.asfortranarray(Ih), cp1)
    for prec in ("tf32", "auto"):
        O = cg.conv(F, I, cp, algo="fused", precision=prec)
        path = cg.last_path()
        err = per_output_error_fp64(torch, F, I, O, cp)
        assert err <= TOL[prec], (cp, prec, path, err)
        e1 = per_output_error(to_host(O[..., img:img + 1]), ref, scale)
        assert e1 <= TOL[prec], (cp, prec, path, e1)
        O2 = cg.conv(F, I, cp, algo="fused", precision=prec)
        assert torch.equal(O, O2), (cp, prec, path)


# ---------------------------------------------------------------- high-waste shifted windows
N_WASTE = 48


def draw_waste(seed):
    """Inside the shifted-window domain (stride <= 2, <= 64 taps, c_i >= 16, k_n % 4 == 0) with
    far more padded-plane rows than outputs: filters almost as large as the image, little or
    no padding, 1-4 outputs per dimension (the geometries the old 1.7x waste cap kept away
    from this kernel)."""
    rng = np.random.default_rng(9500 + seed)
    while True:
        k_h = int(rng.integers(2, 9))
        k_w = int(rng.integers(1, 9))
        if k_h * k_w > 64:
            continue
        s = int(rng.choice([1, 2]))
        p = int(rng.choice([0, 0, 1]))
        o_h, o_w = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        h_i = (o_h - 1) * s + k_h - 2 * p + int(rng.integers(0, s))
        w_i = (o_w - 1) * s + k_w - 2 * p + int(rng.integers(0, s))
        if h_i < 1 or w_i < 1:
            continue
        c_i = int(rng.choice([16, 24, 32, 40, 64, 96, 160]))
        k_n = int(rng.choice([4, 32, 64, 100, 128, 256, 320]))
        b = int(rng.choice([1, 3, 8, 20, 64, 150]))
        cp = dict(k_n=k_n, k_h=k_h, k_w=k_w, c_i=c_i, h_i=h_i, w_i=w_i, b=b, s=s, p=p)
        ho, wo = output_dims_py(cp)
        if ho < 1 or wo < 1:
            continue
        if 2.0 * k_n * ho * wo * b * k_h * k_w * c_i <= 6e8:
            return cp


@pytest.mark.parametrize("seed", range(N_WASTE))
def test_high_waste_geometry(orc, seed):
    cp = draw_waste(seed)
    F, I = rand_inputs(cp, 9600 + seed)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    dF, dI = to_dev(F), to_dev(I)
    for prec in ("tf32", "auto"):
        O = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
        path = cg.last_path()
        err = per_output_error(O, ref, scale)
        assert err <= TOL[prec], (cp, prec, path, err)
    assert path in ("tcgen05-shifted", "tcgen05-gather"), (cp, path)
    with cg.tuning(waste_pct=170):  # the capped dispatch (gather kernel) agrees within the same bar
        O2 = to_host(cg.conv(dF, dI, cp, algo="fused", precision="auto"))
    assert per_output_error(O2, ref, scale) <= TOL["auto"], (cp, cg.last_path())
