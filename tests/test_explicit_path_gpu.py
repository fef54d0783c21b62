"""GPU parity of the explicit path's two kernels.

K1 im2col (simt_kernels.cu, slab kernel): pure data movement, bit-exact against the
oracle's im2col (pinned to im2col.hpp:77-120 by tests/test_oracle.py) over every tiling
branch: h tiles (h_o > 64), w tiles, channel blocks with a remainder, strides, padding
wider than the filter needs, caller leading dimensions beyond K.

K2 GEMM over the lowered matrix (k2_gemm.cu, both operands TMA-fed): against the
oracle's conv_gemm / gemm under the north-star per-output bars, over every filter tile
width, ragged K / k_n / n, split-K (automatic for fc shapes and forced), and both ways
of producing the 3xTF32 filter lo tile (pre-split by K5, or split in the kernel).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2005_06410_b200 as cg  # noqa: E402
from oracle.oracle import Restatement, per_output_error  # noqa: E402
from test_parity_gpu import TOL, rand_inputs, to_dev, to_host  # noqa: E402


@pytest.fixture(scope="module")
def orc():
    return Restatement()


IM2COL_CASES = [
    dict(k_n=4, k_h=3, k_w=3, c_i=64, h_i=56, w_i=56, b=2, s=1, p=1),     # one slab per (image, column)
    dict(k_n=4, k_h=3, k_w=3, c_i=128, h_i=56, w_i=56, b=1, s=2, p=1),    # stride 2, channel blocks
    dict(k_n=4, k_h=3, k_w=3, c_i=70, h_i=30, w_i=20, b=2, s=1, p=1),     # channel remainder (70 = 64 + 6)
    dict(k_n=4, k_h=3, k_w=3, c_i=20, h_i=150, w_i=9, b=1, s=1, p=1),     # h tiles (h_o = 150 > 64)
    dict(k_n=4, k_h=7, k_w=7, c_i=3, h_i=224, w_i=64, b=1, s=2, p=3),     # the stem's shape (K = 147, ld = 148)
    dict(k_n=4, k_h=3, k_w=3, c_i=512, h_i=7, w_i=7, b=3, s=1, p=1),      # w tiles (5 columns per slab)
    dict(k_n=4, k_h=1, k_w=1, c_i=256, h_i=14, w_i=14, b=2, s=1, p=0),    # 1x1
    dict(k_n=4, k_h=2, k_w=5, c_i=9, h_i=13, w_i=17, b=2, s=3, p=4),      # padding beyond the filter, s=3
    dict(k_n=4, k_h=5, k_w=3, c_i=1, h_i=11, w_i=8, b=4, s=1, p=0),       # single channel
]


@pytest.mark.parametrize("case", range(len(IM2COL_CASES)))
def test_im2col_slab_bitexact(orc, case):
    cp = IM2COL_CASES[case]
    _, I = rand_inputs(cp, 900 + case)
    ref = orc.im2col(I, cp)
    k = cp["k_h"] * cp["k_w"] * cp["c_i"]
    for ldb in ((k + 3) // 4 * 4, (k + 3) // 4 * 4 + 8):
        out = torch.full((ref.shape[1], ldb), float("nan"), device="cuda")
        B = cg.im2col(to_dev(I), cp, ldb=ldb, out=out).cpu().numpy()
        assert B.shape == ref.shape
        assert np.array_equal(B.view(np.uint32), ref.view(np.uint32)), (cp, ldb)
        assert not out[:, k:].any(), "rows k..ldb-1 are zero-filled"


EXPLICIT_CASES = [
    dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=28, w_i=28, b=3, s=1, p=1),    # BN=64, many tiles, two rounds
    dict(k_n=24, k_h=3, k_w=3, c_i=5, h_i=9, w_i=9, b=2, s=1, p=1),       # BN=32, K=45 (ragged chunk)
    dict(k_n=128, k_h=3, k_w=3, c_i=32, h_i=14, w_i=14, b=5, s=2, p=1),   # BN=128
    dict(k_n=320, k_h=1, k_w=1, c_i=96, h_i=12, w_i=12, b=9, s=1, p=0),   # BN=256, two filter tiles (one ragged)
    dict(k_n=512, k_h=3, k_w=3, c_i=64, h_i=7, w_i=7, b=2, s=1, p=1),     # one pixel tile, split-K engages
    dict(k_n=10, k_h=3, k_w=3, c_i=4, h_i=8, w_i=8, b=1, s=1, p=0),       # k_n % 4 != 0: padded filter copy
]


@pytest.mark.parametrize("case", range(len(EXPLICIT_CASES)))
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_explicit_k2(orc, case, prec):
    cp = EXPLICIT_CASES[case]
    F, I = rand_inputs(cp, 1000 + case)
    ref = orc.conv_gemm(F, I, cp)
    scale = orc.output_scale(F, I, cp)
    dF, dI = to_dev(F), to_dev(I)
    outs = {}
    for flo in (-1, 1):
        for S in (-1, 0, 3):
            with cg.tuning(k2_flo=flo, splitk=S):
                a = to_host(cg.conv(dF, dI, cp, algo="explicit", precision=prec))
                b = to_host(cg.conv(dF, dI, cp, algo="explicit", precision=prec))
            assert cg.last_path() == "tcgen05-explicit"
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (flo, S)
            err = per_output_error(a, ref, scale)
            assert err <= TOL[prec], (flo, S, err)
            outs[(flo, S)] = a
    if prec == "tf32":  # the filter-lo switch does not exist in plain TF32
        assert np.array_equal(outs[(-1, -1)].view(np.uint32), outs[(1, -1)].view(np.uint32))


def _gemm_case(m, n, k, seed):
    rng = np.random.default_rng(seed)
    A = np.asfortranarray(rng.uniform(-1, 1, (m, k)).astype(np.float32))
    B = np.asfortranarray(rng.uniform(-1, 1, (k, n)).astype(np.float32))
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t()
    Bt = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()
    return A, B, At, Bt


@pytest.mark.parametrize("m,n,k", [(1024, 64, 6272), (512, 130, 2048), (1000, 8, 4096)])
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_fc_gemm_split_k(m, n, k, prec):
    """fc-layer shapes (few pixel tiles, long K): the automatic split-K spreads the weight
    stream over the SMs; the ordered reduce keeps the result bitwise reproducible."""
    from test_simulator import _gemm_ref
    A, B, At, Bt = _gemm_case(m, n, k, m + n + k)
    ref = _gemm_ref(A, B)
    scale = np.outer(np.linalg.norm(A.astype(np.float64), axis=1), np.linalg.norm(B.astype(np.float64), axis=0))
    tol = TOL[prec]
    for flo in (-1, 1):
        for S in (-1, 0, 7):
            with cg.tuning(k2_flo=flo, splitk=S):
                C1 = cg.gemm(At, Bt, precision=prec).cpu().numpy()
                C2 = cg.gemm(At, Bt, precision=prec).cpu().numpy()
            assert np.array_equal(C1.view(np.uint32), C2.view(np.uint32)), (flo, S)
            err = float(np.max(np.abs(C1.astype(np.float64) - ref) / scale))
            assert err <= tol, (flo, S, err)


def test_fc_gemm_takes_no_filter_workspace_for_large_weights():
    """Large static weights in the fp32-accurate mode: the filter lo tile is split in the
    kernel, so the call claims no hi/lo workspace (weights are static)."""
    A, B, At, Bt = _gemm_case(2048, 16, 2048, 5)  # 16 MB of weights
    cg.lib.cgb_scratch_release()
    cg.scratch_reset_peak()
    cg.gemm(At, Bt, precision="3xtf32")
    torch.cuda.synchronize()
    assert cg.scratch_peak_bytes() == 0


# ---------------------------------------------------------------- full size (the shapes the profiles quote)
FULLSIZE_EXPLICIT = ["r50_3x3_56_64", "r50_3x3_s2_56_128", "r50_3x3_7_512", "pw_14_1024_256"]


@pytest.mark.parametrize("name", FULLSIZE_EXPLICIT)
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_explicit_fullsize_fp64(name, prec):
    """The explicit path (K1 slab im2col + K2 TMA-fed GEMM) at the BASELINE layers' stated
    batch -- thousands of pixel tiles per CTA round, the lowered matrix up to 0.9 GB --
    against an fp64 recomputation of every output (tests/fp64ref.py), and K1's lowered
    matrix bit for bit against the oracle on two images."""
    from paper_2005_06410_b200 import configs
    from fp64ref import per_output_error_fp64
    by = {l[0]: (cp, d) for _, l, cp, d in configs.all_layers()}
    cp, dist = by[name]
    F, I = configs.make_tensors(torch, cg.empty_tensor4, cp, dist, configs.layer_seed(name))
    O = cg.conv(F, I, cp, algo="explicit", precision=prec)
    assert cg.last_path() == "tcgen05-explicit"
    err = per_output_error_fp64(torch, F, I, O, cp)
    assert err <= TOL[prec], (name, prec, err)
    if prec == "tf32":
        m, n, k = cg.gemm_dims(cp)
        ldb = (k + 3) // 4 * 4
        B = cg.im2col(I, cp, ldb=ldb)  # (k, n) view, column stride ldb
        per_img = n // cp["b"]
        orc = Restatement()
        for i in (0, cp["b"] - 1):
            img = I[..., i:i + 1]
            flat = img.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy()
            I_h = np.asfortranarray(flat.reshape(tuple(img.shape), order="F"))
            ref = orc.im2col(I_h, dict(cp, b=1))
            got = B[:, i * per_img:(i + 1) * per_img].cpu().numpy()
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (name, i)


@pytest.mark.parametrize("m,n,k", [(4096, 64, 25088), (4096, 256, 4096), (1000, 64, 4096)])
@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
def test_fc_gemm_vgg_shapes_fp64(m, n, k, prec):
    """VGG-16's fc6/fc7/fc8 shapes (the timed ones): split-K over up to 9 pieces per tile,
    against an fp64 product, with the per-output bar."""
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = (torch.rand((k, m), generator=g, device="cuda") * 2 - 1).t()
    B = (torch.rand((n, k), generator=g, device="cuda") * 2 - 1).t()
    C = cg.gemm(A, B, precision=prec)
    ref = A.double() @ B.double()
    scale = A.double().norm(dim=1).view(-1, 1) * B.double().norm(dim=0).view(1, -1)
    err = float(((C.double() - ref).abs() / scale).max())
    assert err <= TOL[prec], (m, n, k, prec, err)
