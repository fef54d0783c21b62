"""CPU: the full-batch fp64 checker (tests/fp64ref.py) agrees with the oracle's f64
accumulation and normalisation, so the GPU full-size parity tests measure the same
quantity as oracle.per_output_error."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from fp64ref import per_output_error_fp64  # noqa: E402
from oracle.oracle import Restatement, per_output_error  # noqa: E402


def t4(a):
    a = np.asfortranarray(a, dtype=np.float32)
    d = a.shape
    return torch.from_numpy(a.reshape(-1, order="F").copy()).view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0)


@pytest.mark.parametrize("cp", [
    dict(k_n=8, k_h=3, k_w=3, c_i=5, h_i=9, w_i=7, b=3, s=1, p=1),
    dict(k_n=6, k_h=3, k_w=2, c_i=4, h_i=11, w_i=10, b=2, s=2, p=1),
    dict(k_n=4, k_h=7, k_w=7, c_i=3, h_i=20, w_i=18, b=2, s=2, p=3),
    dict(k_n=5, k_h=1, k_w=1, c_i=7, h_i=4, w_i=6, b=3, s=1, p=0),
])
def test_fp64_checker_matches_oracle(cp):
    orc = Restatement()
    rng = np.random.default_rng(3)
    F = np.asfortranarray(rng.uniform(-1, 1, (cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])).astype(np.float32))
    I = np.asfortranarray(rng.uniform(-1, 1, (cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])).astype(np.float32))
    O = orc.conv_gemm(F, I, cp)
    # the reference's fp32 output against fp64: tiny but nonzero, and both checkers agree
    e_orc = per_output_error(O, orc.conv_f64(F, I, cp), orc.output_scale(F, I, cp))
    e_t = per_output_error_fp64(torch, t4(F), t4(I), t4(O), cp, chunk=2)
    assert e_t == pytest.approx(e_orc, rel=1e-6, abs=1e-12)
    # a planted error of known normalised size is reported exactly
    O2 = O.copy()
    scale = orc.output_scale(F, I, cp)
    O2[1, 0, 0, cp["b"] - 1] += 1e-3 * scale[1, 0, 0, cp["b"] - 1]
    e2 = per_output_error_fp64(torch, t4(F), t4(I), t4(O2), cp)
    assert e2 == pytest.approx(1e-3, rel=1e-3)
