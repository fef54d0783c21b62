"""GPU: the reference's Python surface semantics (proj/tests/python/test_smoke.py:34-116,
python/convgemm/__init__.py:9-61) on the B200 package, plus the bit-exact paths.

* conv_direct runs on the device bit-identical to the reference's conv_direct<float>
  (its accumulation order, product rounded before the add) -- pinned against the
  reference's own outputs in tests/golden (made by the reference, make_golden.py).
* float64 inputs select the reference's f64 arithmetic on the device's FP64 cores,
  bit-identical to conv_gemm<double> / conv_im2col_gemm<double> / conv_direct<double> /
  im2col<double> / gemm<double> (kc-blocked order, kc from BlockingParams).
* the smoke suite's properties: backends agree (fused vs direct within the reference's
  1e-5 * max(1, max|ref|) bar; FFMA fused == explicit bit for bit, the reference's "same
  engine" property -- the tensor-core precisions differ in summation order by design),
  double precision is exact (fused == direct for K <= kc), gemm against numpy, im2col
  shape/values, the fused path takes no device workspace.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2005_06410_b200 as cg  # noqa: E402
from conftest import golden_cases  # noqa: E402


def random_case(rng, cap=6, dtype=np.float32):
    while True:
        k_n, k_h, k_w, c_i = (int(rng.integers(1, cap + 1)) for _ in range(4))
        h_i, w_i = (int(rng.integers(1, cap + 1)) for _ in range(2))
        s, p, b = int(rng.integers(1, 3)), int(rng.integers(0, 2)), int(rng.integers(1, 3))
        if h_i - k_h + 2 * p >= 0 and w_i - k_w + 2 * p >= 0:
            break
    cp = cg.ConvParams(k_n=k_n, k_h=k_h, k_w=k_w, c_i=c_i, h_i=h_i, w_i=w_i, b=b, s=s, p=p)
    F = np.asfortranarray(rng.uniform(-1, 1, size=(k_n, k_h, k_w, c_i)).astype(dtype))
    I = np.asfortranarray(rng.uniform(-1, 1, size=(h_i, w_i, c_i, b)).astype(dtype))
    return cp, F, I


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def test_conv_direct_bitexact_golden(golden):
    for i, cp, g in golden_cases(golden, "rand"):
        O = cg.conv_direct(g[f"rand{i}_F"], g[f"rand{i}_I"], cp)
        assert np.array_equal(bits(O), bits(g[f"rand{i}_Odirect"])), (i, cp)


def test_conv_direct_device_tensors(golden):
    for i, cp, g in list(golden_cases(golden, "rand"))[:8]:
        F = torch.from_numpy(np.asfortranarray(g[f"rand{i}_F"]).reshape(-1, order="F").copy()).cuda()
        I = torch.from_numpy(np.asfortranarray(g[f"rand{i}_I"]).reshape(-1, order="F").copy()).cuda()
        Fv = F.view(*reversed(g[f"rand{i}_F"].shape)).permute(3, 2, 1, 0)
        Iv = I.view(*reversed(g[f"rand{i}_I"].shape)).permute(3, 2, 1, 0)
        O = cg.conv(Fv, Iv, cp, algo="direct")
        Oh = O.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy().reshape(tuple(O.shape), order="F")
        assert np.array_equal(bits(Oh), bits(g[f"rand{i}_Odirect"]))


def test_f64_bitexact_golden(golden):
    n = int(golden["n_f64"])
    keys = ("k_n", "k_h", "k_w", "c_i", "h_i", "w_i", "b", "s", "p")
    for i in range(n):
        cp = dict(zip(keys, [int(v) for v in golden[f"f64_{i}_cp"]]))
        bp = cg.BlockingParams(kc=int(golden[f"f64_{i}_kc"]))
        F, I = golden[f"f64_{i}_F"], golden[f"f64_{i}_I"]
        assert F.dtype == np.float64
        fused = cg.conv_gemm(F, I, cp, blocking=bp)
        assert fused.dtype == np.float64
        assert np.array_equal(bits(fused), bits(golden[f"f64_{i}_O"])), (i, cp)
        assert np.array_equal(bits(cg.conv_im2col_gemm(F, I, cp, blocking=bp)), bits(golden[f"f64_{i}_Oexplicit"]))
        assert np.array_equal(bits(cg.conv_direct(F, I, cp)), bits(golden[f"f64_{i}_Odirect"]))
        assert np.array_equal(bits(cg.im2col(I, cp)), bits(golden[f"f64_{i}_B"]))


def test_f64_gemm_bitexact_golden(golden):
    C = cg.gemm(golden["f64_gemm_A"], golden["f64_gemm_B"])
    assert np.array_equal(bits(C), bits(golden["f64_gemm_C"]))


def test_dims_functions():
    cp = cg.ConvParams(k_n=64, k_h=11, k_w=11, c_i=3, h_i=224, w_i=224, b=2, s=4, p=0)
    assert cg.output_dims(cp) == (54, 54)
    assert cg.gemm_dims(cp) == (64, 2916 * 2, 363)
    with pytest.raises(cg.InvalidGeometry):
        cg.output_dims(cg.ConvParams(k_n=1, k_h=9, k_w=1, c_i=1, h_i=4, w_i=4))


def test_conv_backends_agree():
    rng = np.random.default_rng(7)
    for _ in range(10):
        cp, F, I = random_case(rng)
        ref = cg.conv_direct(F, I, cp)
        for prec in ("auto", "3xtf32", "ffma"):
            fused = cg.conv_gemm(F, I, cp, threads=2, precision=prec)
            assert ref.shape == fused.shape
            np.testing.assert_allclose(fused, ref, rtol=0, atol=1e-5 * max(1.0, np.abs(ref).max()))
        # the reference's "same engine" property holds for the FFMA kernel (one
        # accumulation order for both operators)
        f = cg.conv_gemm(F, I, cp, precision="ffma")
        e = cg.conv_im2col_gemm(F, I, cp, precision="ffma")
        assert np.array_equal(f, e)


def test_double_precision_is_exact():
    rng = np.random.default_rng(11)
    for _ in range(5):
        cp, F, I = random_case(rng, dtype=np.float64)
        ref = cg.conv_direct(F, I, cp)
        fused = cg.conv_gemm(F, I, cp)
        assert fused.dtype == np.float64
        assert np.array_equal(fused, ref)


def test_gemm_against_numpy():
    rng = np.random.default_rng(13)
    a = np.asfortranarray(rng.uniform(-1, 1, size=(17, 29)))
    b = np.asfortranarray(rng.uniform(-1, 1, size=(29, 23)))
    c = cg.gemm(a, b, threads=2)
    np.testing.assert_allclose(c, a @ b, rtol=1e-12, atol=1e-12)
    c32 = cg.gemm(a.astype(np.float32), b.astype(np.float32))
    np.testing.assert_allclose(c32, a @ b, rtol=0, atol=1e-5 * np.abs(a @ b).max())


def test_im2col_shape_and_values():
    rng = np.random.default_rng(17)
    for dtype in (np.float32, np.float64):
        cp, _, image = random_case(rng, dtype=dtype)
        lowered = cg.im2col(image, cp)
        m, n, k = cg.gemm_dims(cp)
        assert lowered.shape == (k, n)
        assert cg.im2col_workspace_bytes(cp) == 4 * k * n


def test_fused_takes_no_device_workspace():
    """The reference's fused scratch stays within its packing panels
    (test_smoke.py:109-116); on the device the fused TF32 path takes none at all."""
    rng = np.random.default_rng(19)
    cp, F, I = random_case(rng)
    cg.scratch_reset_peak()
    cg.conv_gemm(F, I, cp, precision="tf32")
    assert cg.scratch_peak_bytes() <= cg.convgemm_scratch_bytes(cg.BlockingParams())
