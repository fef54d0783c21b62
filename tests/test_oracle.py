"""CPU: pin the oracle (plain-C restatement, oracle/conv_oracle.c) against the
reference's own outputs -- the committed golden fixtures (generated from the
reference by tests/golden/make_golden.py) and, where it was built here, the
reference library itself (oracle/_ref). Also restates the reference's own
known-answer tests (proj/tests/test_conv.cpp:13-79, test_convgemm.cpp:13-54)."""
import os

import numpy as np
import pytest

from conftest import golden_cases
from oracle.oracle import REFERENCE_SO, OracleError, Reference, Restatement, normalized_max_error

HAVE_REF = os.path.exists(REFERENCE_SO)


@pytest.fixture(scope="module")
def orc():
    return Restatement()


@pytest.fixture(scope="module")
def ref():
    if not HAVE_REF:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return Reference()


def test_restatement_matches_golden_random(orc, golden):
    n = 0
    for i, cp, g in golden_cases(golden, "rand"):
        F, I = g[f"rand{i}_F"], g[f"rand{i}_I"]
        F, I = np.asfortranarray(F), np.asfortranarray(I)
        assert np.array_equal(orc.conv_gemm(F, I, cp), g[f"rand{i}_O"]), (i, cp)
        assert np.array_equal(orc.conv_direct(F, I, cp), g[f"rand{i}_Odirect"]), (i, cp)
        assert np.array_equal(orc.im2col(I, cp), g[f"rand{i}_B"]), (i, cp)
        n += 1
    assert n == 64


def test_restatement_matches_golden_medium(orc, golden):
    for i, cp, g in golden_cases(golden, "med"):
        F, I = np.asfortranarray(g[f"med{i}_F"]), np.asfortranarray(g[f"med{i}_I"])
        O = orc.conv_gemm(F, I, cp)
        assert np.array_equal(O, g[f"med{i}_O"]), (i, cp)
        # fused == explicit, bitwise (test_convgemm.cpp:163-190)
        assert np.array_equal(g[f"med{i}_O"], g[f"med{i}_Oexplicit"])


def test_restatement_matches_reference_live(orc, ref):
    g = ref.rng(2024)
    for it in range(60):
        cp = g.conv_params(9, 3)
        F = g.tensor(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
        I = g.tensor(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
        assert np.array_equal(orc.conv_gemm(F, I, cp), ref.conv_gemm(F, I, cp, threads=it % 3 + 1))
        assert np.array_equal(orc.im2col(I, cp), ref.im2col(I, cp))
    # K > kc = 640: two kc blocks, still bitwise
    cp = dict(k_n=24, k_h=3, k_w=3, c_i=80, h_i=7, w_i=7, b=2, s=1, p=1)
    F = g.tensor(24, 3, 3, 80)
    I = g.tensor(7, 7, 80, 2)
    assert np.array_equal(orc.conv_gemm(F, I, cp), ref.conv_gemm(F, I, cp, threads=2))
    assert np.array_equal(orc.conv_gemm(F, I, cp), ref.conv_im2col_gemm(F, I, cp, threads=3))


def test_reference_pack_equivalence(ref):
    """acceptance.cpp:89-135: fused pack == pack over im2col, bitwise, incl. batch straddles."""
    g = ref.rng(102)
    straddles_total = 0
    for _ in range(30):
        cp = g.conv_params(8, 3)
        bp = [4, 0, 0, 2, 0]
        nr = g.rand_in(1, 4)
        bp = [4, nr * g.rand_in(1, 4), g.rand_in(1, 6), 2, nr]
        I = g.tensor(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
        import ctypes
        from oracle.oracle import _cp_array
        s = ctypes.c_int64()
        bad = ref.lib.ref_pack_check(I.ctypes.data, _cp_array(cp), (ctypes.c_int64 * 5)(*bp), ctypes.byref(s))
        assert bad == 0
        straddles_total += s.value
    assert straddles_total > 0


# ---- known answers restated from the reference's unit tests ----

def _t(shape, fill=None):
    a = np.zeros(shape, dtype=np.float32, order="F")
    if fill is not None:
        a[...] = fill
    return a


def test_known_scalar(orc):  # test_conv.cpp:13-19
    F, I = _t((1, 1, 1, 1), 3.0), _t((1, 1, 1, 1), -2.0)
    cp = (1, 1, 1, 1, 1, 1, 1, 1, 0)
    assert orc.conv_direct(F, I, cp).ravel()[0] == -6.0
    assert orc.conv_gemm(F, I, cp).ravel()[0] == -6.0


def test_known_ones_sum(orc):  # test_conv.cpp:21-28
    F, I = _t((1, 2, 2, 1), 1.0), _t((2, 2, 1, 1), 1.0)
    O = orc.conv_gemm(F, I, (1, 2, 2, 1, 2, 2, 1, 1, 0))
    assert O.size == 1 and O.ravel()[0] == 4.0


def test_known_1x1_stride(orc):  # test_conv.cpp:30-42
    rng = np.random.default_rng(21)
    I = np.asfortranarray(rng.uniform(-1, 1, (5, 5, 1, 1)).astype(np.float32))
    F = _t((1, 1, 1, 1), 2.5)
    O = orc.conv_direct(F, I, (1, 1, 1, 1, 5, 5, 1, 2, 0))
    assert O.shape == (1, 3, 3, 1)
    for h in range(3):
        for w in range(3):
            assert O[0, h, w, 0] == np.float32(2.5) * I[2 * h, 2 * w, 0, 0]


def test_known_patch_column(orc):  # test_conv.cpp:65-79
    I = _t((2, 2, 1, 1))
    I[0, 0, 0, 0], I[0, 1, 0, 0], I[1, 0, 0, 0], I[1, 1, 0, 0] = 1, 2, 3, 4
    B = orc.im2col(I, (1, 2, 2, 1, 2, 2, 1, 1, 0))
    assert B.shape == (4, 1)
    assert B[:, 0].tolist() == [1.0, 3.0, 2.0, 4.0]


def test_known_output_dims(orc):  # test_tensor.cpp:31-44 (AlexNet conv1: 224, 11x11, s4 -> 54)
    assert orc.output_dims((64, 11, 11, 3, 224, 224, 2, 4, 0)) == (54, 54)
    assert orc.output_dims((64, 3, 3, 64, 56, 56, 1, 1, 1)) == (56, 56)
    assert orc.output_dims((64, 7, 7, 3, 224, 224, 1, 2, 3)) == (112, 112)
    with pytest.raises(OracleError):
        orc.output_dims((1, 5, 5, 1, 3, 3, 1, 1, 0))
    with pytest.raises(OracleError):
        orc.output_dims((0, 1, 1, 1, 3, 3, 1, 1, 0))


def test_reference_global_metric_on_golden(orc, golden):
    # direct vs fused agree to the reference's own 1e-5 bound (acceptance.cpp:51-85)
    for i, cp, g in golden_cases(golden, "rand"):
        assert normalized_max_error(g[f"rand{i}_O"], g[f"rand{i}_Odirect"]) <= 1e-5
