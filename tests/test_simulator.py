"""Model files, the inference simulator and gemm (the reference's model.cpp, bench.cpp and
gemm binding): parsing and its errors, the built-in model definitions against the
reference's own model files, the CSV schema (CPU); the simulator sweep and gemm parity
on the device (gpu)."""
import io
import os

import numpy as np
import pytest

import paper_2005_06410_b200 as cg
from paper_2005_06410_b200 import models

REF_MODELS = "/root/reference/proj/models"

SMALL = """# two convs, a pool, an fc
conv 32 3 3 16 12 12 1 1
pool 6 6 32
conv 64 3 3 32 12 12 2 1   # strided
fc 100 2304
"""


def test_parse_model_text():
    m = cg.parse_model(SMALL, name="small")
    assert m.name == "small" and [l.kind for l in m.layers] == ["conv", "pool", "conv", "fc"]
    assert m.count("conv") == 2 and m.count("fc") == 1 and m.count("pool") == 1
    c = m.layers[2].conv
    assert (c.k_n, c.k_h, c.k_w, c.c_i, c.h_i, c.w_i, c.b, c.s, c.p) == (64, 3, 3, 32, 12, 12, 1, 2, 1)
    assert (m.layers[3].fc_m, m.layers[3].fc_k) == (100, 2304)
    assert cg.parse_model(m.to_text()).to_text() == m.to_text()
    assert cg.parse_model(io.StringIO(SMALL)).count("conv") == 2


@pytest.mark.parametrize("text,line,what", [
    ("conv 8 3 3 4 10 10 1\n", 1, "missing or malformed p"),
    ("conv 8 3 3 4 10 10 1 1 7\n", 1, "trailing token '7'"),
    ("\n# c\nconv 8 3 3 4 10 10 1 x\n", 3, "missing or malformed p"),
    ("conv 8 3 3 4 10 10 1 1\nmaxpool 2 2 8\n", 2, "unknown layer kind 'maxpool'"),
    ("pool 2 2 8\nfc 10 8\n", 2, "model contains no conv layer"),
    ("conv 8 5 5 4 2 2 1 0\n", 1, ""),  # filter larger than the input: InvalidGeometry -> ParseError
    ("conv 8 3 3 4 10 10 1 1\nfc 0 8\n", 2, "fc dimensions must be positive"),
    ("conv 8 3 3 4 10 10 1 1\npool 0 2 8\n", 2, "pool dimensions must be positive"),
])
def test_parse_model_errors(text, line, what):
    with pytest.raises(cg.ParseError) as e:
        cg.parse_model(text)
    assert e.value.line == line and what in str(e.value)
    if "unknown layer kind" in what:
        assert isinstance(e.value, cg.UnknownLayerKind)


def test_parse_model_missing_file(tmp_path):
    with pytest.raises(cg.IoError):
        cg.parse_model(str(tmp_path / "nope.model"))


@pytest.mark.skipif(not os.path.isdir(REF_MODELS), reason="reference model files absent")
@pytest.mark.parametrize("name", sorted(models.MODELS))
def test_builtin_models_match_reference_files(name):
    """The generated VGG-16 / ResNet-50 definitions equal the reference's model files layer
    for layer (parsed by our parser, which also reads the reference's files)."""
    ref = cg.parse_model(os.path.join(REF_MODELS, f"{name}.model"))
    assert models.MODELS[name]().to_text() == ref.to_text()


@pytest.mark.skipif(not os.path.isdir(REF_MODELS), reason="reference model files absent")
def test_parse_reference_alexnet():
    m = cg.parse_model(os.path.join(REF_MODELS, "alexnet.model"))
    assert (m.count("conv"), m.count("fc"), m.count("pool")) == (5, 3, 3)


def test_model_workspace_bytes():
    m = models.vgg16()
    want = max(4 * cg.gemm_dims(dict(vars(l.conv), b=3))[1] * cg.gemm_dims(dict(vars(l.conv), b=3))[2]
               for l in m.layers if l.kind == "conv")
    assert cg.model_workspace_bytes(m, 3) == want
    with pytest.raises(cg.InvalidGeometry):
        cg.model_workspace_bytes(m, 0)


def test_write_csv_schema():
    m = cg.parse_model(SMALL, name="small")
    rs = [cg.LayerResult(1, "conv", 32, 288, 144, 1e-5, 10, 8.3, 0),
          cg.LayerResult(4, "fc", 100, 2, 2304, 2e-5, 5, 46.1, 4096)]
    out = io.StringIO()
    cg.write_csv(out, m, 2, "convgemm", 1, rs)
    lines = out.getvalue().splitlines()
    assert lines[0] == "model,batch,algo,threads,layer,m,n,k,time_s,gflops,workspace_bytes"
    assert lines[1].startswith("small,2,convgemm,1,1,32,288,144,")
    tot = lines[-1].split(",")
    assert tot[4:8] == ["total", "0", "0", "0"] and int(tot[10]) == 4096
    assert abs(float(tot[8]) - 3e-5) < 1e-12


# ----------------------------------------------------------------------------- device
torch = pytest.importorskip("torch")
needs_cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


def _gemm_ref(A, B):
    """The reference's gemm arithmetic through the oracle: a 1x1 conv over 1x1 images."""
    from oracle.oracle import Restatement
    orc = Restatement()
    m, k = A.shape
    n = B.shape[1]
    F = np.asfortranarray(A.reshape(m, 1, 1, k, order="F"))
    I = np.asfortranarray(B.reshape(1, 1, k, n, order="F"))
    cp = dict(k_n=m, k_h=1, k_w=1, c_i=k, h_i=1, w_i=1, b=n, s=1, p=0)
    return orc.conv_gemm(F, I, cp).reshape(m, n, order="F")


@pytest.mark.gpu
@needs_cuda
@pytest.mark.parametrize("m,n,k", [(1000, 8, 4096), (256, 37, 100), (64, 3, 27), (4096, 2, 9216)])
@pytest.mark.parametrize("prec,tol", [("3xtf32", 1e-5), ("tf32", 5e-3), ("ffma", 1e-5)])
@pytest.mark.parametrize("where", ["device", "host"])
def test_gemm_parity(m, n, k, prec, tol, where):
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    A = np.asfortranarray(rng.uniform(-1, 1, (m, k)).astype(np.float32))
    B = np.asfortranarray(rng.uniform(-1, 1, (k, n)).astype(np.float32))
    ref = _gemm_ref(A, B)
    if where == "device":
        At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t()
        Bt = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()
        C = cg.gemm(At, Bt, precision=prec).cpu().numpy()
    else:
        C = cg.gemm(A, B, precision=prec)
    scale = np.outer(np.linalg.norm(A.astype(np.float64), axis=1), np.linalg.norm(B.astype(np.float64), axis=0))
    err = float(np.max(np.abs(C.astype(np.float64) - ref) / scale))
    assert err <= tol, (m, n, k, prec, err)


@pytest.mark.gpu
@needs_cuda
@pytest.mark.parametrize("algo", ["convgemm", "im2col", "gemm-only", "im2col-only", "direct"])
def test_run_inference_small(algo):
    m = cg.parse_model(SMALL, name="small")
    rs = cg.run_inference(m, 3, algo=algo, min_time=0.0, check=True)
    conv_layers = [i + 1 for i, l in enumerate(m.layers) if l.kind == "conv"]
    want = conv_layers + ([] if algo == "im2col-only" else [4])
    assert [r.layer for r in rs] == want
    for r in rs:
        l = m.layers[r.layer - 1]
        if l.kind == "conv":
            assert (r.m, r.n, r.k) == cg.gemm_dims(dict(vars(l.conv), b=3))
        else:
            assert (r.m, r.n, r.k) == (100, 3, 2304)
        assert r.time_s > 0 and r.repetitions >= 1
        assert (r.gflops == 0) == (algo == "im2col-only")
    out = io.StringIO()
    cg.write_csv(out, m, 3, algo, 1, rs)
    assert len(out.getvalue().splitlines()) == len(rs) + 2


@pytest.mark.gpu
@needs_cuda
@pytest.mark.parametrize("name", sorted(models.MODELS))
@pytest.mark.parametrize("precision", ["tf32", "auto"])
def test_run_inference_models_checked(name, precision):
    """Whole-model sweep at batch 2 with every conv checked against conv_direct as the
    reference does (bench.cpp:212-233), under the per-output bar (1e-5 for the
    fp32-accurate default, 5e-3 for plain TF32)."""
    m = models.MODELS[name]()
    rs = cg.run_inference(m, 2, algo="convgemm", min_time=0.0, check=True, precision=precision)
    assert len(rs) == m.count("conv") + m.count("fc")
    assert all(r.gflops > 0 for r in rs)


@pytest.mark.gpu
def test_gemm_ignores_rows_past_k():
    """B with ldb > k (a view of a taller matrix): rows k..ldb-1 are not part of the
    operand, even when they hold NaN/Inf (the explicit gather was bounded by
    ldb)."""
    import numpy as np
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rng = np.random.default_rng(5)
    m, n, k, ldb = 96, 40, 52, 64
    A = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    Bfull = rng.uniform(-1, 1, (ldb, n)).astype(np.float32)
    Bfull[k:, :] = np.nan
    Ad = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t()
    Bd = torch.from_numpy(np.ascontiguousarray(Bfull.T)).cuda().t()[:k]  # (k, n) view, ld = 64
    for prec in ("tf32", "3xtf32", "ffma"):
        C = cg.gemm(Ad, Bd, precision=prec).cpu().numpy()
        ref = A.astype(np.float64) @ Bfull[:k].astype(np.float64)
        assert np.isfinite(C).all(), prec
        assert np.abs(C - ref).max() <= (5e-3 if prec == "tf32" else 1e-5) * np.abs(A).sum(1).max(), prec
