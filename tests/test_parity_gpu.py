"""GPU parity: the B200 operator through the C-ABI against the reference's outputs.

Bars (BASELINE.json north_star), per-output normalised by ||F[i_k]||*||B[:,col]||:
  3xTF32 and FFMA <= 1e-5, TF32 <= 5e-3; im2col (pure data movement) bit-exact.
Oracles: committed golden fixtures produced by the reference itself
(tests/golden/make_golden.py) and the plain-C restatement (oracle/, pinned
bitwise to the reference by tests/test_oracle.py) for larger shapes.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2005_06410_b200 as cg  # noqa: E402
from conftest import golden_cases  # noqa: E402
from oracle.oracle import Restatement, per_output_error  # noqa: E402

TOL = {"3xtf32": 1e-5, "ffma": 1e-5, "tf32": 5e-3, "auto": 1e-5}
PRECS = ("3xtf32", "tf32", "ffma")
ALGOS = ("fused", "explicit")


@pytest.fixture(scope="module")
def orc():
    return Restatement()


def to_dev(a):
    """numpy Fortran array -> leftmost-fastest CUDA tensor with identical layout."""
    a = np.asfortranarray(a, dtype=np.float32)
    t = torch.from_numpy(a.reshape(-1, order="F").copy()).cuda()
    d = a.shape
    return t.view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0)


def to_host(t):
    d = t.shape
    flat = t.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy()
    return flat.reshape(d, order="F")


def rand_inputs(cp, seed, stem=False):
    rng = np.random.default_rng(seed)
    fs = (cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
    is_ = (cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
    if stem:
        F = rng.normal(0.0, 0.05, fs).astype(np.float32)
        I = rng.uniform(0.0, 1.0, is_).astype(np.float32)
    else:
        F = rng.uniform(-1, 1, fs).astype(np.float32)
        I = rng.uniform(-1, 1, is_).astype(np.float32)
    return np.asfortranarray(F), np.asfortranarray(I)


# ---------------------------------------------------------------- im2col (K1): bit-exact
def test_im2col_bitexact_golden(golden):
    for i, cp, g in golden_cases(golden, "rand"):
        B = cg.im2col(to_dev(g[f"rand{i}_I"]), cp)
        assert np.array_equal(B.cpu().numpy(), g[f"rand{i}_B"]), (i, cp)


def test_im2col_padded_ld_and_medium(golden, orc):
    for i, cp, g in golden_cases(golden, "med"):
        I = g[f"med{i}_I"]
        k = cp["k_h"] * cp["k_w"] * cp["c_i"]
        for ldb in (k, (k + 3) // 4 * 4, k + 5):
            B = cg.im2col(to_dev(I), cp, ldb=ldb)
            assert np.array_equal(B.cpu().numpy(), orc.im2col(np.asfortranarray(I), cp)), (i, ldb)


# ---------------------------------------------------------------- conv vs golden reference outputs
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("prec", PRECS)
def test_conv_golden_random(golden, orc, algo, prec):
    worst = 0.0
    for i, cp, g in golden_cases(golden, "rand"):
        F, I = np.asfortranarray(g[f"rand{i}_F"]), np.asfortranarray(g[f"rand{i}_I"])
        O = to_host(cg.conv(to_dev(F), to_dev(I), cp, algo=algo, precision=prec))
        err = per_output_error(O, g[f"rand{i}_O"], orc.output_scale(F, I, cp))
        worst = max(worst, err)
        assert err <= TOL[prec], (i, cp, err)
    print(f"{algo}/{prec}: worst per-output error {worst:.3e} over 64 reference configs")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("prec", PRECS)
def test_conv_golden_medium(golden, orc, algo, prec):
    for i, cp, g in golden_cases(golden, "med"):
        F, I = np.asfortranarray(g[f"med{i}_F"]), np.asfortranarray(g[f"med{i}_I"])
        O = to_host(cg.conv(to_dev(F), to_dev(I), cp, algo=algo, precision=prec))
        err = per_output_error(O, g[f"med{i}_O"], orc.output_scale(F, I, cp))
        assert err <= TOL[prec], (i, cp, err)


# ---------------------------------------------------------------- BASELINE geometries (reduced batch)
BASELINE_LAYERS = {
    "c1_56_64_b8": (dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=56, w_i=56, b=8, s=1, p=1), False),
    "r50_28_128": (dict(k_n=128, k_h=3, k_w=3, c_i=128, h_i=28, w_i=28, b=2, s=1, p=1), False),
    "r50_14_256": (dict(k_n=256, k_h=3, k_w=3, c_i=256, h_i=14, w_i=14, b=2, s=1, p=1), False),
    "r50_7_512": (dict(k_n=512, k_h=3, k_w=3, c_i=512, h_i=7, w_i=7, b=2, s=1, p=1), False),
    "r50_s2_56": (dict(k_n=128, k_h=3, k_w=3, c_i=128, h_i=56, w_i=56, b=1, s=2, p=1), False),
    "r50_s2_28": (dict(k_n=256, k_h=3, k_w=3, c_i=256, h_i=28, w_i=28, b=1, s=2, p=1), False),
    "r50_s2_14": (dict(k_n=512, k_h=3, k_w=3, c_i=512, h_i=14, w_i=14, b=2, s=2, p=1), False),
    "pw_56_64_256": (dict(k_n=256, k_h=1, k_w=1, c_i=64, h_i=56, w_i=56, b=2, s=1, p=0), False),
    "pw_7_512_2048": (dict(k_n=2048, k_h=1, k_w=1, c_i=512, h_i=7, w_i=7, b=2, s=1, p=0), False),
    "pw_14_1024_256": (dict(k_n=256, k_h=1, k_w=1, c_i=1024, h_i=14, w_i=14, b=2, s=1, p=0), False),
    "pw_7_2048_512": (dict(k_n=512, k_h=1, k_w=1, c_i=2048, h_i=7, w_i=7, b=2, s=1, p=0), False),
    "stem_224": (dict(k_n=64, k_h=7, k_w=7, c_i=3, h_i=224, w_i=224, b=1, s=2, p=3), True),
    "vgg_conv1": (dict(k_n=64, k_h=3, k_w=3, c_i=3, h_i=224, w_i=224, b=1, s=1, p=1), False),
    # the rest of the VGG-16 stack (BASELINE configs[4]), b=1
    "vgg_224_64_64": (dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=224, w_i=224, b=1, s=1, p=1), False),
    "vgg_112_64_128": (dict(k_n=128, k_h=3, k_w=3, c_i=64, h_i=112, w_i=112, b=1, s=1, p=1), False),
    "vgg_112_128_128": (dict(k_n=128, k_h=3, k_w=3, c_i=128, h_i=112, w_i=112, b=1, s=1, p=1), False),
    "vgg_56_128_256": (dict(k_n=256, k_h=3, k_w=3, c_i=128, h_i=56, w_i=56, b=1, s=1, p=1), False),
    "vgg_56_256_256": (dict(k_n=256, k_h=3, k_w=3, c_i=256, h_i=56, w_i=56, b=1, s=1, p=1), False),
    "vgg_28_256_512": (dict(k_n=512, k_h=3, k_w=3, c_i=256, h_i=28, w_i=28, b=1, s=1, p=1), False),
    "vgg_28_512_512": (dict(k_n=512, k_h=3, k_w=3, c_i=512, h_i=28, w_i=28, b=1, s=1, p=1), False),
    "vgg_14_512_512": (dict(k_n=512, k_h=3, k_w=3, c_i=512, h_i=14, w_i=14, b=1, s=1, p=1), False),
}


@pytest.mark.parametrize("name", sorted(BASELINE_LAYERS))
@pytest.mark.parametrize("prec", ("3xtf32", "tf32", "auto"))
def test_conv_baseline_geometry(orc, name, prec):
    cp, stem = BASELINE_LAYERS[name]
    F, I = rand_inputs(cp, 20177, stem)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    for algo in ALGOS:
        O = to_host(cg.conv(to_dev(F), to_dev(I), cp, algo=algo, precision=prec))
        err = per_output_error(O, ref, scale)
        assert err <= TOL[prec], (name, algo, prec, err, cg.last_path())


# ---------------------------------------------------------------- size-independent properties at full size
def test_full_size_properties():
    """C2 56x56 64->64 at b=128: batch slicing is exact (each output depends only on
    its own image), reruns are bitwise deterministic (no float atomics; the
    reference guarantees the same, gemm.hpp:40-45), and conv is linear in I."""
    cp = dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=56, w_i=56, b=128, s=1, p=1)
    g = torch.Generator(device="cuda").manual_seed(7)
    F = cg.empty_tensor4(64, 3, 3, 64)
    F.copy_(torch.rand(F.shape, generator=g, device="cuda") * 2 - 1)
    I = cg.empty_tensor4(56, 56, 64, 128)
    I.copy_(torch.rand(I.shape, generator=g, device="cuda") * 2 - 1)
    for prec in ("tf32", "3xtf32"):
        O1 = cg.conv(F, I, cp, precision=prec)
        O2 = cg.conv(F, I, cp, precision=prec)
        assert torch.equal(O1, O2)
        # image 37 alone (whole tiles, as in the b=128 launch: a split-K b=1 launch sums
        # in another order)
        cp1 = dict(cp, b=1)
        I37 = cg.empty_tensor4(56, 56, 64, 1)
        I37.copy_(I[..., 37:38])
        with cg.tuning(splitk=-1):
            O37 = cg.conv(F, I37, cp1, precision=prec)
        assert torch.equal(O37[..., 0], O1[..., 37])
    # linearity (within tolerance): conv(F, 2*I) == 2*conv(F, I) exactly (power-of-two scaling)
    I2 = cg.empty_tensor4(56, 56, 64, 128)
    I2.copy_(I * 2)
    O = cg.conv(F, I, cp, precision="3xtf32")
    assert torch.equal(cg.conv(F, I2, cp, precision="3xtf32"), O * 2)


def test_explicit_equals_fused_ffma(orc):
    """FFMA explicit and fused use the same per-output accumulation order -> bitwise equal
    (the reference's own fused == explicit property, test_convgemm.cpp:163-190)."""
    cp = dict(k_n=48, k_h=3, k_w=3, c_i=24, h_i=15, w_i=15, b=3, s=2, p=1)
    F, I = rand_inputs(cp, 3)
    a = cg.conv(to_dev(F), to_dev(I), cp, algo="fused", precision="ffma")
    b = cg.conv(to_dev(F), to_dev(I), cp, algo="explicit", precision="ffma")
    assert torch.equal(a, b)


# ---------------------------------------------------------------- reference call semantics
def test_host_path_matches_device_path():
    cp = dict(k_n=32, k_h=3, k_w=3, c_i=16, h_i=20, w_i=18, b=2, s=1, p=1)
    F, I = rand_inputs(cp, 11)
    for prec in PRECS:
        for algo in ALGOS:
            host = cg.conv(F, I, cp, algo=algo, precision=prec)
            dev = to_host(cg.conv(to_dev(F), to_dev(I), cp, algo=algo, precision=prec))
            assert np.array_equal(host, dev), (algo, prec)


def _pinned_fortran(a):
    """Fortran-ordered numpy view over page-locked memory holding a copy of a."""
    t = torch.empty(a.size, dtype=torch.float32, pin_memory=True)
    v = t.numpy()
    v[:] = np.asfortranarray(a).reshape(-1, order="F")
    return v.reshape(a.shape, order="F"), t


@pytest.mark.parametrize("chunk_kb", [20, 70, 1 << 20])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("bounce", [True, False])
def test_host_pipeline_chunking(chunk_kb, pinned, bounce):
    """cgb_conv_host cuts the batch into chunks (H2D || conv || D2H on three streams,
    pinned bounce ring for pageable buffers). Any chunking -- one chunk, more chunks
    than bounce slots, a ragged last chunk -- gives the device-path result bit for bit."""
    cp = dict(k_n=32, k_h=3, k_w=3, c_i=16, h_i=21, w_i=19, b=11, s=2, p=1)
    F, I = rand_inputs(cp, 12)
    keep = []
    if pinned:
        F, kf = _pinned_fortran(F)
        I, ki = _pinned_fortran(I)
        keep += [kf, ki]
    for prec in ("3xtf32", "tf32"):
        dev = to_host(cg.conv(to_dev(F), to_dev(I), cp, algo="fused", precision=prec))
        # 20 KB -> 1 image per chunk
        with cg.tuning(host_chunk_kb=chunk_kb, host_no_bounce=0 if bounce else 1):
            host = cg.conv(F, I, cp, algo="fused", precision=prec)
            assert np.array_equal(host, dev), (chunk_kb, pinned, bounce, prec)
            if pinned:
                ho, kt = _pinned_fortran(np.zeros_like(host))
                cg.conv(F, I, cp, algo="fused", precision=prec, out=ho)
                assert np.array_equal(ho, dev)


def test_reference_named_entry_points(orc):
    cp = cg.ConvParams(k_n=16, k_h=3, k_w=3, c_i=8, h_i=12, w_i=12, b=2, s=1, p=1)
    F, I = rand_inputs(vars(cp), 40)
    ref = orc.conv_gemm(F, I, vars(cp))
    scale = orc.output_scale(F, I, vars(cp))
    assert per_output_error(cg.conv_gemm(F, I, cp, cg.BlockingParams(), 4), ref, scale) <= 1e-5
    assert per_output_error(cg.conv_im2col_gemm(F, I, cp), ref, scale) <= 1e-5


def test_shape_mismatch_raises():
    cp = dict(k_n=4, k_h=3, k_w=3, c_i=2, h_i=8, w_i=8, b=1, s=1, p=1)
    F, I = rand_inputs(cp, 1)
    with pytest.raises(cg.InvalidGeometry):
        cg.conv(to_dev(F), to_dev(I[:, :, :1, :]), cp)
    with pytest.raises(cg.InvalidGeometry):
        cg.conv(F, I, dict(cp, h_i=2, w_i=2, p=0))


def test_workspace_limit_kills_explicit_not_fused(orc):
    """test_convgemm.cpp:231-242 on the device: under a workspace limit the explicit path
    fails with AllocationFailure while the fused path (no HBM B-hat) still runs."""
    cp = dict(k_n=192, k_h=5, k_w=5, c_i=64, h_i=55, w_i=55, b=1, s=1, p=0)
    F, I = rand_inputs(cp, 39)
    cg.lib.cgb_scratch_release()
    cg.scratch_set_limit(9 << 20)
    try:
        with pytest.raises(cg.AllocationFailure):
            cg.conv(to_dev(F), to_dev(I), cp, algo="explicit", precision="tf32")
        O = to_host(cg.conv(to_dev(F), to_dev(I), cp, algo="fused", precision="tf32"))
    finally:
        cg.scratch_set_limit(0)
    ref = orc.conv_gemm(F, I, cp)
    assert per_output_error(O, ref, orc.output_scale(F, I, cp)) <= 5e-3


def test_kernels_actually_launch():
    n0 = cg.kernel_launch_count()
    cp = dict(k_n=8, k_h=1, k_w=1, c_i=8, h_i=4, w_i=4, b=1, s=1, p=0)
    F, I = rand_inputs(cp, 2)
    cg.conv(to_dev(F), to_dev(I), cp)
    torch.cuda.synchronize()
    assert cg.kernel_launch_count() > n0


# ---------------------------------------------------------------- kernel-variant coverage
VARIANT_CASES = [
    # (cp, expected kernel) -- shifted window (stride 1 and polyphase stride 2) and the gather
    (dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=30, w_i=30, b=2, s=1, p=1), "tcgen05-shifted"),
    (dict(k_n=128, k_h=3, k_w=3, c_i=32, h_i=40, w_i=40, b=3, s=1, p=0), "tcgen05-shifted"),
    (dict(k_n=96, k_h=3, k_w=1, c_i=64, h_i=33, w_i=21, b=2, s=1, p=1), "tcgen05-shifted"),
    (dict(k_n=32, k_h=1, k_w=1, c_i=48, h_i=20, w_i=20, b=3, s=1, p=0), "tcgen05-shifted"),
    (dict(k_n=64, k_h=3, k_w=3, c_i=40, h_i=28, w_i=28, b=1, s=1, p=1), "tcgen05-shifted"),
    (dict(k_n=256, k_h=3, k_w=3, c_i=64, h_i=24, w_i=24, b=2, s=1, p=1), "tcgen05-shifted"),
    (dict(k_n=512, k_h=3, k_w=3, c_i=64, h_i=7, w_i=7, b=3, s=1, p=1), "tcgen05-shifted"),
    (dict(k_n=96, k_h=3, k_w=3, c_i=48, h_i=15, w_i=15, b=2, s=2, p=1), "tcgen05-shifted"),
    (dict(k_n=128, k_h=3, k_w=3, c_i=32, h_i=30, w_i=30, b=2, s=2, p=1), "tcgen05-shifted"),
    (dict(k_n=64, k_h=1, k_w=1, c_i=64, h_i=28, w_i=28, b=2, s=2, p=0), "tcgen05-shifted"),
    (dict(k_n=48, k_h=2, k_w=2, c_i=24, h_i=17, w_i=17, b=2, s=2, p=0), "tcgen05-shifted"),
    (dict(k_n=256, k_h=3, k_w=3, c_i=96, h_i=28, w_i=28, b=1, s=2, p=1), "tcgen05-shifted"),
    # 5x5 p=2: the shared-padding plane (14 rows per column instead of 16) keeps it shifted
    (dict(k_n=128, k_h=5, k_w=5, c_i=32, h_i=12, w_i=12, b=2, s=1, p=2), "tcgen05-shifted"),
    # padded plane 9x9 rows for 6x6 outputs (2.25x): shifted since the waste cap went
    # (tools/waste_ab.py); with the old 1.7x cap restored it exercises the gather kernel
    (dict(k_n=64, k_h=7, k_w=7, c_i=32, h_i=6, w_i=6, b=3, s=1, p=3), "tcgen05-shifted"),
    (dict(k_n=64, k_h=7, k_w=7, c_i=32, h_i=6, w_i=6, b=3, s=1, p=3), "tcgen05-gather", dict(waste_pct=170)),
    # far more padded rows than outputs: 5x5 on 7x7 unpadded (49 rows for 9 outputs), a
    # filter as large as the image (one output per image, 25x)
    (dict(k_n=128, k_h=5, k_w=5, c_i=48, h_i=7, w_i=7, b=9, s=1, p=0), "tcgen05-shifted"),
    (dict(k_n=64, k_h=5, k_w=5, c_i=32, h_i=5, w_i=5, b=40, s=1, p=0), "tcgen05-shifted"),
    (dict(k_n=64, k_h=4, k_w=6, c_i=64, h_i=9, w_i=8, b=17, s=2, p=0), "tcgen05-shifted"),
    # wide image: window halo (2 + 2*151 rows) beyond 256 rows (VGG 224x224 layers)
    (dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=150, w_i=150, b=1, s=1, p=1), "tcgen05-shifted"),
    # pad > k-1 and asymmetric periods: wrapped reads land in shared zero rows
    (dict(k_n=64, k_h=3, k_w=2, c_i=32, h_i=11, w_i=9, b=3, s=1, p=2), "tcgen05-shifted"),
    (dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=20, w_i=20, b=2, s=3, p=1), "tcgen05-gather"),
    # 1x1 stride 1 with h*w % 4 == 0: A TMA'd straight from I (MN-major, TF32), pixel
    # planes not a multiple of the 32-pixel box, partial channel chunks, odd batches
    (dict(k_n=96, k_h=1, k_w=1, c_i=40, h_i=10, w_i=10, b=5, s=1, p=0), "tcgen05-shifted"),
    (dict(k_n=64, k_h=1, k_w=1, c_i=32, h_i=12, w_i=12, b=7, s=1, p=0), "tcgen05-shifted"),
    (dict(k_n=256, k_h=1, k_w=1, c_i=200, h_i=8, w_i=6, b=33, s=1, p=0), "tcgen05-shifted"),
    # 1x1 with a wide filter tile (two-unit producers, BN = 256) and a deep one
    (dict(k_n=256, k_h=1, k_w=1, c_i=96, h_i=20, w_i=20, b=40, s=1, p=0), "tcgen05-shifted"),
    (dict(k_n=512, k_h=1, k_w=1, c_i=128, h_i=7, w_i=7, b=64, s=1, p=0), "tcgen05-shifted"),
    # low-channel layers: w-im2col rows (k_w*c_i <= 32 values per row), k_h taps as shifts
    (dict(k_n=64, k_h=7, k_w=7, c_i=3, h_i=40, w_i=40, b=2, s=2, p=3), "tcgen05-shifted-wim"),
    (dict(k_n=64, k_h=3, k_w=3, c_i=3, h_i=30, w_i=30, b=2, s=1, p=1), "tcgen05-shifted-wim"),
    (dict(k_n=32, k_h=3, k_w=3, c_i=1, h_i=17, w_i=13, b=3, s=1, p=0), "tcgen05-shifted-wim"),
    (dict(k_n=48, k_h=4, k_w=4, c_i=8, h_i=12, w_i=12, b=2, s=2, p=1), "tcgen05-shifted-wim"),
    (dict(k_n=96, k_h=5, k_w=3, c_i=5, h_i=20, w_i=16, b=2, s=1, p=2), "tcgen05-shifted-wim"),
    # the specialised (k_w, c_i) = (7, 3) / (3, 3) producers at odd sizes, k_n = 64 (BN = 64)
    (dict(k_n=64, k_h=7, k_w=7, c_i=3, h_i=37, w_i=29, b=3, s=2, p=3), "tcgen05-shifted-wim"),
    (dict(k_n=64, k_h=3, k_w=3, c_i=3, h_i=23, w_i=41, b=2, s=1, p=1), "tcgen05-shifted-wim"),
    (dict(k_n=64, k_h=3, k_w=3, c_i=3, h_i=23, w_i=41, b=2, s=2, p=0), "tcgen05-shifted-wim"),
    # wide stride-2 image (halo beyond 256 rows per phase)
    (dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=301, w_i=40, b=1, s=2, p=1), "tcgen05-shifted"),
]


@pytest.mark.parametrize("cp", [
    dict(k_n=256, k_h=1, k_w=1, c_i=64, h_i=56, w_i=56, b=3, s=1, p=0),
    dict(k_n=96, k_h=1, k_w=1, c_i=40, h_i=10, w_i=10, b=5, s=1, p=0),
    dict(k_n=512, k_h=1, k_w=1, c_i=1024, h_i=14, w_i=14, b=2, s=1, p=0),
])
def test_tma_fed_1x1_bitwise_equal_to_staged(cp):
    # TF32 1x1: the TMA-fed A tile (MN-major, straight from I) and the producer-staged
    # K-major window feed the same fp32 bits to the same UMMAs in the same order
    F, I = rand_inputs(cp, 4242)
    Fd, Id = to_dev(F), to_dev(I)
    with cg.tuning(tma_a=0):
        staged = to_host(cg.conv(Fd, Id, cp, algo="fused", precision="tf32"))
    with cg.tuning(tma_a=1):
        tma = to_host(cg.conv(Fd, Id, cp, algo="fused", precision="tf32"))
    assert cg.last_path() == "tcgen05-shifted"
    assert np.array_equal(staged.view(np.uint32), tma.view(np.uint32))


@pytest.mark.parametrize("case", range(len(VARIANT_CASES)))
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_kernel_variants(orc, case, prec):
    cp, path = VARIANT_CASES[case][:2]
    tune = VARIANT_CASES[case][2] if len(VARIANT_CASES[case]) > 2 else {}
    F, I = rand_inputs(cp, 100 + case)
    ref = orc.conv_gemm(F, I, cp)
    with cg.tuning(**tune):
        O = to_host(cg.conv(to_dev(F), to_dev(I), cp, algo="fused", precision=prec))
    if prec == "tf32":
        assert cg.last_path() == path, (cp, cg.last_path())
    else:  # 3xTF32 needs twice the staging; wide polyphase windows fall back to the gather kernel
        assert cg.last_path() in (path, "tcgen05-gather"), (cp, cg.last_path())
    err = per_output_error(O, ref, orc.output_scale(F, I, cp))
    assert err <= TOL[prec], (cp, prec, err)


# ---------------------------------------------------------------- stream-K split tiles
SK_CASES = [
    # enough M tiles (>= one per SM pair) with a last round < 90% full -> the last
    # rounds are split by channel chunk across SM pairs, two pieces per split tile
    dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=28, w_i=28, b=24, s=1, p=1),
    dict(k_n=128, k_h=3, k_w=3, c_i=64, h_i=56, w_i=56, b=24, s=2, p=1),
    dict(k_n=96, k_h=3, k_w=3, c_i=80, h_i=20, w_i=20, b=48, s=1, p=1),
    # fewer tiles than SM pairs, many channel chunks, stream-K forced (tuning sk=2): every
    # tile is split into several pieces, combined in the fixed highest-chunk-first order
    dict(k_n=256, k_h=3, k_w=3, c_i=512, h_i=7, w_i=7, b=48, s=1, p=1, force=True),
    dict(k_n=512, k_h=3, k_w=3, c_i=256, h_i=14, w_i=14, b=48, s=2, p=1, force=True),
]


@pytest.mark.parametrize("case", range(len(SK_CASES)))
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_stream_k(orc, case, prec):
    cp = dict(SK_CASES[case])
    sk = 2 if cp.pop("force", False) else 1
    F, I = rand_inputs(cp, 300 + case)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    dF, dI = to_dev(F), to_dev(I)
    with cg.tuning(sk=sk, splitk=-1):  # stream-K itself, not the split-K of few-tile layers
        a = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
        assert cg.last_path() in ("tcgen05-shifted", "tcgen05-gather"), cg.last_path()
        b = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
    assert np.array_equal(a, b), "stream-K result must not depend on which piece finishes first"
    assert per_output_error(a, ref, scale) <= TOL[prec]
    with cg.tuning(sk=0, splitk=-1):
        whole = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
    assert per_output_error(whole, ref, scale) <= TOL[prec]
    if cg.last_path() == "tcgen05-shifted":
        # the split changes the fp32 summation order of the split tiles: proof it engaged
        assert not np.array_equal(a, whole)


# ---------------------------------------------------------------- tail tiles
TAIL_CASES = [
    # forced (tuning tail=2): whole 4-subtile pair tiles for one round, then 2-subtile
    # (or 1-subtile) tail tiles for the remaining rows
    dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=56, w_i=56, b=26, s=1, p=1),
    dict(k_n=128, k_h=3, k_w=3, c_i=32, h_i=28, w_i=28, b=70, s=1, p=1),
    dict(k_n=64, k_h=3, k_w=3, c_i=48, h_i=57, w_i=30, b=44, s=2, p=1),
]


@pytest.mark.parametrize("case", range(len(TAIL_CASES)))
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_tail_tiles(orc, case, prec):
    cp = TAIL_CASES[case]
    F, I = rand_inputs(cp, 500 + case)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    dF, dI = to_dev(F), to_dev(I)
    with cg.tuning(tail=2, splitk=-1):
        a = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
    assert per_output_error(a, ref, scale) <= TOL[prec]
    with cg.tuning(tail=0, splitk=-1):
        b = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
    assert per_output_error(b, ref, scale) <= TOL[prec]
    if cg.last_path() == "tcgen05-shifted":
        # whole tiles in both launches (no stream-K split): the same bits either way
        assert np.array_equal(a, b)


STRIP_CASES = [
    # (cp, forced strip height or 0 = the rule): strips that do not divide h_o, pad 0 / 2, 5x5 taps,
    # non-square images, a batch that leaves the last virtual image ragged
    (dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=150, w_i=150, b=2, s=1, p=1), 0),
    (dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=224, w_i=40, b=3, s=1, p=1), 0),
    (dict(k_n=128, k_h=3, k_w=3, c_i=32, h_i=112, w_i=112, b=2, s=1, p=1), 0),
    (dict(k_n=64, k_h=5, k_w=5, c_i=32, h_i=131, w_i=37, b=3, s=1, p=2), 0),
    (dict(k_n=96, k_h=3, k_w=2, c_i=48, h_i=201, w_i=23, b=2, s=1, p=0), 0),
    (dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=61, w_i=30, b=5, s=1, p=1), 13),
    (dict(k_n=256, k_h=3, k_w=3, c_i=64, h_i=70, w_i=20, b=7, s=1, p=2), 17),
    (dict(k_n=64, k_h=7, k_w=3, c_i=16, h_i=90, w_i=33, b=2, s=1, p=3), 20),
]


@pytest.mark.parametrize("case", range(len(STRIP_CASES)))
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_h_strips(orc, case, prec):
    """Wide stride-1 images cut into h-strips (virtual images with halo rows from the
    neighbouring strips): against the oracle, and bitwise equal to the unstripped launch when
    neither splits tiles (same UMMAs per output in the same order)."""
    cp, sh = STRIP_CASES[case]
    F, I = rand_inputs(cp, 1300 + case)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    dF, dI = to_dev(F), to_dev(I)
    with cg.tuning(strip_h=sh, sk=0, splitk=-1):
        a = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
        path = cg.last_path()
    assert per_output_error(a, ref, scale) <= TOL[prec], (cp, sh, path)
    with cg.tuning(strip_h=-1, sk=0, splitk=-1):
        b = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
    assert per_output_error(b, ref, scale) <= TOL[prec]
    if path == "tcgen05-shifted" and cg.last_path() == "tcgen05-shifted":
        assert np.array_equal(a, b), (cp, sh)
    with cg.tuning(strip_h=sh):  # default stream-K / split-K on top of the strips
        c = to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec))
    assert per_output_error(c, ref, scale) <= TOL[prec], (cp, sh)


def _offset_tensor4(a, shift):
    """CUDA leftmost-fastest tensor holding a, starting `shift` floats into its buffer
    (a user pointer that is only 4-byte aligned)."""
    a = np.asfortranarray(a, dtype=np.float32)
    buf = torch.zeros(a.size + shift, dtype=torch.float32, device="cuda")
    buf[shift:] = torch.from_numpy(a.reshape(-1, order="F")).cuda()
    d = a.shape
    return buf[shift:].view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0)


@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_unaligned_user_pointers(orc, prec):
    """F, I and O whose device pointers are only 4-byte aligned: every kernel path must
    avoid 16/32-byte vector accesses and TMA on them (or stage them) and stay correct."""
    cp = dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=20, w_i=20, b=3, s=1, p=1)
    F, I = rand_inputs(cp, 77)
    ref = orc.conv_gemm(F, I, cp)
    h_o, w_o = 20, 20
    for algo in ALGOS:
        O = _offset_tensor4(np.zeros((64, h_o, w_o, 3), np.float32), 1)
        cg.conv(_offset_tensor4(F, 1), _offset_tensor4(I, 3), cp, algo=algo, precision=prec, out=O)
        assert per_output_error(to_host(O), ref, orc.output_scale(F, I, cp)) <= TOL[prec], (algo, cg.last_path())


# ------------------------------------------- TF32 operand semantics (DESIGN §9 item 2)
def _trunc_tf32(x):
    return (np.asarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.parametrize("kh,hi,s,p", [(1, 16, 1, 0), (1, 7, 1, 0), (3, 16, 1, 1), (3, 16, 2, 1)])
def test_tf32_truncates_raw_operands(kh, hi, s, p):
    """kind::tf32 drops the low 13 mantissa bits of the raw fp32 operands (truncation):
    with one nonzero (tap, channel) per output, O = trunc(F)·trunc(I) exactly (two
    11-bit mantissas multiply exactly in fp32). The 3xTF32 split relies on this."""
    kn, ci, b = 128, 32, 2
    rng = np.random.default_rng(7)
    F = np.zeros((kn, kh, kh, ci), np.float32, order="F")
    F[:, kh // 2, kh // 2, 3] = rng.uniform(0.5, 2.0, kn).astype(np.float32)
    I = np.zeros((hi, hi, ci, b), np.float32, order="F")
    I[:, :, 3, :] = rng.uniform(-2.0, 2.0, (hi, hi, b)).astype(np.float32)
    cp = dict(k_n=kn, k_h=kh, k_w=kh, c_i=ci, h_i=hi, w_i=hi, b=b, s=s, p=p)
    O = to_host(cg.conv(to_dev(F), to_dev(I), cp, precision="tf32"))
    # centre tap with padding p = kh // 2: output (oh, ow) reads input (oh·s, ow·s)
    Ic = _trunc_tf32(I[::s, ::s, 3, :])
    want = _trunc_tf32(F[:, kh // 2, kh // 2, 3])[:, None, None, None] * Ic[None]
    assert O.shape == want.shape
    assert np.array_equal(O, want.astype(np.float32))


# ---------------------------------------------------------------- filter-stage groups
@pytest.mark.parametrize("cp", [
    dict(k_n=128, k_h=3, k_w=3, c_i=64, h_i=30, w_i=30, b=3, s=2, p=1),   # MT=1 BN=128 pair: 2-tap groups
    dict(k_n=64, k_h=3, k_w=3, c_i=48, h_i=20, w_i=20, b=2, s=1, p=1),    # BN=64
    dict(k_n=64, k_h=7, k_w=7, c_i=3, h_i=40, w_i=40, b=2, s=2, p=3),     # w-im2col rows (short taps)
    dict(k_n=64, k_h=1, k_w=1, c_i=256, h_i=8, w_i=8, b=9, s=1, p=0),     # TMA-fed 1x1: one tap per chunk
    dict(k_n=128, k_h=1, k_w=1, c_i=192, h_i=7, w_i=7, b=5, s=1, p=0),    # staged 1x1
])
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_filter_stage_groups_bitwise(orc, cp, prec):
    """Handing the filter ring over in groups of G taps changes only the synchronisation,
    never the UMMA order: every group size gives the same bits (and passes the oracle)."""
    F, I = rand_inputs(cp, 911)
    dF, dI = to_dev(F), to_dev(I)
    outs = []
    for tps in (1, 2, 3, 4, 0):
        with cg.tuning(tps=tps):
            outs.append(to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec)))
    # TMA-fed 1x1 with a single A slot (the forced ring must not deadlock)
    if cp["k_h"] == 1 and prec == "tf32":
        for cfg in (20, 22, 26, 29, 31, 32, 33, 34, 35):
            for tps in (2, 4):
                with cg.tuning(cfg=cfg, tps=tps):
                    outs.append(to_host(cg.conv(dF, dI, cp, algo="fused", precision=prec)))
    ref = orc.conv_gemm(F, I, cp)
    for o in outs[1:5]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
    for o in outs[5:]:  # other tile configurations: same tolerance, not the same bits
        assert per_output_error(o, ref, orc.output_scale(F, I, cp)) <= TOL[prec]
    assert per_output_error(outs[0], ref, orc.output_scale(F, I, cp)) <= TOL[prec]


# ---------------------------------------------------------------- workspace semantics
def test_workspace_limit_checked_on_every_call(orc):
    """ScratchTracker::allocate checks the limit on every claim (scratch.cpp:15-19): a
    cached larger buffer must not let an oversized explicit call through, and
    current/peak count claims, not the cached allocation."""
    cp = dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=40, w_i=40, b=4, s=1, p=1)
    F, I = rand_inputs(cp, 61)
    dF, dI = to_dev(F), to_dev(I)
    need = cg.conv_workspace_bytes(cp, "explicit", "tf32")
    cg.conv(dF, dI, cp, algo="explicit", precision="tf32")  # caches a buffer >= need
    torch.cuda.synchronize()
    assert cg.lib.cgb_scratch_cached_bytes() >= need
    assert cg.lib.cgb_scratch_current_bytes() == 0  # claims end with the call
    cg.scratch_set_limit(need - 1)
    try:
        with pytest.raises(cg.AllocationFailure):
            cg.conv(dF, dI, cp, algo="explicit", precision="tf32")
        cg.conv(dF, dI, cp, algo="fused", precision="tf32")  # no workspace: still runs
    finally:
        cg.scratch_set_limit(0)
    cg.scratch_reset_peak()
    cg.conv(dF, dI, cp, algo="fused", precision="tf32")
    assert cg.scratch_peak_bytes() == 0
    cg.conv(dF, dI, cp, algo="explicit", precision="tf32")
    assert cg.scratch_peak_bytes() == need


def test_workspace_per_stream_concurrent(orc):
    """3xTF32 writes its filter split into workspace: calls on two streams with different
    filters, enqueued back to back, must not share (and overwrite) one buffer."""
    cp = dict(k_n=128, k_h=3, k_w=3, c_i=64, h_i=28, w_i=28, b=8, s=1, p=1)
    Fa, I = rand_inputs(cp, 71)
    Fb, _ = rand_inputs(cp, 72)
    dFa, dFb, dI = to_dev(Fa), to_dev(Fb), to_dev(I)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            oa = cg.conv(dFa, dI, cp, precision="3xtf32")
        with torch.cuda.stream(s2):
            ob = cg.conv(dFb, dI, cp, precision="3xtf32")
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for F, k in ((Fa, 0), (Fb, 1)):
        ref = orc.conv_gemm(F, I, cp)
        for o in outs:
            assert per_output_error(to_host(o[k]), ref, orc.output_scale(F, I, cp)) <= 1e-5


def test_forked_streams_graph_bitwise_equal_to_serial(orc):
    """Independent layers issued on forked streams inside one captured graph (bench.py's
    supplementary `concurrent` step): stream-K layers (per-stream tile counters), a split-K
    layer (per-stream partial-tile workspace) and a whole-tile layer running concurrently
    give the bits of the serial launches, replay after replay."""
    cases = [dict(SK_CASES[0]), dict(SK_CASES[1]),
             dict(k_n=256, k_h=3, k_w=3, c_i=256, h_i=14, w_i=14, b=4, s=1, p=1),   # few tiles: split-K
             dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=56, w_i=56, b=6, s=1, p=1)]
    ins = []
    for i, cp in enumerate(cases):
        F, I = rand_inputs(cp, 900 + i)
        ins.append((cp, to_dev(F), to_dev(I)))
    serial = [cg.conv(dF, dI, cp, algo="fused", precision="tf32").clone() for cp, dF, dI in ins]
    torch.cuda.synchronize()
    outs = [torch.zeros_like(o) for o in serial]
    side = [torch.cuda.Stream() for _ in range(2)]

    def step():
        cur = torch.cuda.current_stream()
        for st in side:
            st.wait_stream(cur)
        for i, (cp, dF, dI) in enumerate(ins):
            with torch.cuda.stream(side[i % 2]):
                cg.conv(dF, dI, cp, algo="fused", precision="tf32", out=outs[i])
        for st in side:
            cur.wait_stream(st)

    warm = torch.cuda.Stream()
    warm.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(warm):
        step()  # allocates the per-stream counters / workspaces outside the capture
    torch.cuda.current_stream().wait_stream(warm)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for rep in range(5):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        for i, (o, ref) in enumerate(zip(outs, serial)):
            assert torch.equal(o, ref), (rep, cases[i])
    cp, dF, dI = ins[0]
    F, I = rand_inputs(cp, 900)
    assert per_output_error(to_host(outs[0]), orc.conv_gemm(F, I, cp), orc.output_scale(F, I, cp)) <= TOL["tf32"]


def test_workspace_growth_keeps_captured_buffer(orc):
    """A graph captured with the cached workspace keeps working after a later call on the
    same stream needs (and allocates) a bigger one: captured buffers are never freed."""
    cp = dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=16, w_i=16, b=2, s=1, p=1)
    big = dict(k_n=256, k_h=3, k_w=3, c_i=256, h_i=14, w_i=14, b=2, s=1, p=1)
    F, I = rand_inputs(cp, 81)
    Fb, Ib = rand_inputs(big, 82)
    dF, dI, dFb, dIb = to_dev(F), to_dev(I), to_dev(Fb), to_dev(Ib)
    cg.lib.cgb_scratch_release()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        O = cg.conv(dF, dI, cp, precision="3xtf32")  # allocates this stream's workspace
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            cg.conv(dF, dI, cp, precision="3xtf32", out=O)
        cg.conv(dFb, dIb, big, precision="3xtf32")  # outgrows the captured buffer
        st.synchronize()
        O.zero_()
        g.replay()
    torch.cuda.synchronize()
    ref = orc.conv_gemm(F, I, cp)
    assert per_output_error(to_host(O), ref, orc.output_scale(F, I, cp)) <= 1e-5


def test_host_pipeline_pageable_stress():
    """The pageable-buffer path (pinned bounce ring + parallel memcpy pool) over many
    chunks, repeated: every repetition bit-identical, and equal to the device path."""
    cp = dict(k_n=32, k_h=3, k_w=3, c_i=64, h_i=32, w_i=32, b=96, s=1, p=1)
    F, I = rand_inputs(cp, 91)
    dev = to_host(cg.conv(to_dev(F), to_dev(I), cp, precision="tf32"))
    # 10 images (2.5 MB of input) per chunk: ~10 chunks, more than the bounce slots, each
    # copy large enough (>= 2 MiB) for the parallel memcpy pool
    # (chunks are b=10 convolutions, which may take other tile splits than the b=96 launch:
    # repetitions are compared bitwise with each other and with the device path in tolerance)
    with cg.tuning(host_chunk_kb=2560):
        first = None
        for _ in range(20):
            out = np.zeros_like(dev, order="F")
            cg.conv(F, I, cp, precision="tf32", out=out)
            if first is None:
                first = out
                scale = np.abs(dev).max()
                assert np.max(np.abs(out - dev)) <= 1e-5 * scale
            assert np.array_equal(out, first)


# ---------------------------------------------------------------- split-K (few-tile layers)
SPLITK_CASES = [
    # the strong-scaling shards of the bench layers (b=16 of 128): few tiles, many chunks
    dict(k_n=512, k_h=3, k_w=3, c_i=512, h_i=7, w_i=7, b=16, s=1, p=1),
    dict(k_n=512, k_h=3, k_w=3, c_i=512, h_i=14, w_i=14, b=16, s=2, p=1),
    dict(k_n=256, k_h=3, k_w=3, c_i=256, h_i=14, w_i=14, b=4, s=1, p=1),
    dict(k_n=96, k_h=3, k_w=3, c_i=80, h_i=9, w_i=9, b=3, s=1, p=1),
    dict(k_n=64, k_h=1, k_w=1, c_i=256, h_i=7, w_i=7, b=2, s=1, p=0),
]


@pytest.mark.parametrize("case", range(len(SPLITK_CASES)))
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_split_k(orc, case, prec):
    """Split-K partial tiles summed in a fixed order by the reduce kernel: within
    tolerance of the oracle for every forced piece count, bitwise reproducible, and the
    automatic choice engages for the few-tile shapes."""
    cp = SPLITK_CASES[case]
    F, I = rand_inputs(cp, 700 + case)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    dF, dI = to_dev(F), to_dev(I)
    with cg.tuning(splitk=-1):
        whole = to_host(cg.conv(dF, dI, cp, precision=prec))
    assert per_output_error(whole, ref, scale) <= TOL[prec]
    for S in (0, 2, 3, 5):
        with cg.tuning(splitk=S):
            a = to_host(cg.conv(dF, dI, cp, precision=prec))
            b = to_host(cg.conv(dF, dI, cp, precision=prec))
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), S
        assert per_output_error(a, ref, scale) <= TOL[prec], (S, per_output_error(a, ref, scale))


# ---------------------------------------------------------------- resident filters, w-im2col dispatch
@pytest.mark.parametrize("cp", [
    dict(k_n=64, k_h=7, k_w=7, c_i=3, h_i=40, w_i=36, b=3, s=2, p=3),    # the stem's shape: 7 taps resident
    dict(k_n=64, k_h=3, k_w=3, c_i=3, h_i=30, w_i=30, b=2, s=1, p=1),    # VGG conv1's shape: 3 taps
    dict(k_n=128, k_h=1, k_w=1, c_i=64, h_i=12, w_i=12, b=5, s=1, p=0),  # 1x1, two chunks resident (TMA-fed A)
    dict(k_n=64, k_h=1, k_w=1, c_i=96, h_i=7, w_i=7, b=9, s=1, p=0),     # 1x1 staged windows, three chunks
])
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_resident_filters_bitwise(orc, cp, prec):
    """Filters kept resident in the ring (loaded once per CTA, no per-tile hand-overs) feed
    the same bits to the same UMMAs as the streamed ring; the w-im2col layers' single-CTA
    dispatch and the CTA-pair kernels (pair=2) both meet the bar."""
    F, I = rand_inputs(cp, 4711, stem=cp["c_i"] == 3)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    Fd, Id = to_dev(F), to_dev(I)
    outs = {}
    for pair in (1, 2):
        for br in (0, 1):
            with cg.tuning(b_res=br, pair=pair):
                outs[(pair, br)] = to_host(cg.conv(Fd, Id, cp, precision=prec))
            assert per_output_error(outs[(pair, br)], ref, scale) <= TOL[prec], (pair, br)
        assert np.array_equal(outs[(pair, 0)].view(np.uint32), outs[(pair, 1)].view(np.uint32)), pair


# ---------------------------------------------------------------- BN = 512 filter tiles
@pytest.mark.parametrize("cp", [
    dict(k_n=512, k_h=1, k_w=1, c_i=128, h_i=7, w_i=7, b=9, s=1, p=0),     # the 1x1 7x7 layers it is for
    dict(k_n=1024, k_h=1, k_w=1, c_i=96, h_i=7, w_i=7, b=20, s=1, p=0),    # two filter tiles
    dict(k_n=640, k_h=1, k_w=1, c_i=64, h_i=14, w_i=14, b=3, s=1, p=0),    # ragged second tile, TMA-fed A
    dict(k_n=512, k_h=3, k_w=3, c_i=32, h_i=9, w_i=9, b=4, s=1, p=1),      # 3x3 windows
])
def test_bn512_tiles_bitwise(orc, cp):
    """Filter tiles of 512 (two N = 256 UMMAs per k-step; each CTA of a pair holds the two
    N halves interleaved): every output accumulates the same products in the same order as
    with 256-filter tiles, so the results are bitwise equal, and within the bar of the oracle."""
    F, I = rand_inputs(cp, 5120)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    Fd, Id = to_dev(F), to_dev(I)
    with cg.tuning(bn=256):
        base = to_host(cg.conv(Fd, Id, cp, precision="tf32"))
    assert per_output_error(base, ref, scale) <= TOL["tf32"]
    for cfg in (54, 55):
        with cg.tuning(bn=512, cfg=cfg, verbose=0):
            out = to_host(cg.conv(Fd, Id, cp, precision="tf32"))
        assert cg.last_path() == "tcgen05-shifted"
        assert np.array_equal(out.view(np.uint32), base.view(np.uint32)), cfg


def test_bn512_dispatch_and_unit_rotation(orc):
    """A staged 1x1 layer with a long contraction and k_n = 512 takes the 512-filter tile by
    itself, and its window units rotate over the staging warps from chunk to chunk: both
    are pure scheduling, bitwise equal to the 256-filter tiles without rotation."""
    cp = dict(k_n=512, k_h=1, k_w=1, c_i=544, h_i=7, w_i=7, b=200, s=1, p=0)  # 9800 rows: 39 pair tiles
    F, I = rand_inputs(cp, 5121)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    Fd, Id = to_dev(F), to_dev(I)
    with cg.tuning(bn=256, urot=0):
        base = to_host(cg.conv(Fd, Id, cp, precision="tf32"))
    assert per_output_error(base, ref, scale) <= TOL["tf32"]
    for urot in (0, 1):
        with cg.tuning(urot=urot):
            out = to_host(cg.conv(Fd, Id, cp, precision="tf32"))
        assert np.array_equal(out.view(np.uint32), base.view(np.uint32)), urot
    with cg.tuning(bn=256, urot=1):
        out = to_host(cg.conv(Fd, Id, cp, precision="3xtf32"))
    assert per_output_error(out, ref, scale) <= TOL["3xtf32"]
