"""The C++ drop-in surface (include/convgemm/*.hpp): the REFERENCE's own simulator
sources -- proj/src/bench.cpp (its calls to conv_gemm<float>, conv_im2col_gemm<float>,
im2col<float>, Im2colMatrix, MatrixView, MatrixSource, zero_matrix, gemm<float>,
filters_as_matrix, output_as_matrix, conv_direct<float>, bench.cpp:140-233) and
model.cpp -- compile UNCHANGED against it and link with libconvgemm_b200.so
(VERDICT r01 "what's missing" #2). The binary (tests/cpp/dropin_main.cpp drives it) is
built where /root/reference exists (here, and by __graft_entry__.build() into
tests/cpp/_build/, which travels to the GPU box) and run under -m gpu: every algorithm of
the reference's run_inference over a small model with the reference's own check against
conv_direct on.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/proj/src"
LIBDIR = os.path.join(ROOT, "paper_2005_06410_b200")
PREBUILT = os.path.join(ROOT, "tests", "cpp", "_build", "dropin")


def build_dropin(out):
    """g++ the reference's bench.cpp + model.cpp (unchanged) + the test driver against
    include/ only (no reference header is on the include path)."""
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(REF_SRC, "bench.cpp"), os.path.join(REF_SRC, "model.cpp"),
           os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp"), "-L", LIBDIR, "-lconvgemm_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", out]
    return subprocess.run(cmd, capture_output=True, text=True)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="the reference sources exist only in the build container")
def test_reference_simulator_compiles_unchanged(tmp_path):
    r = build_dropin(str(tmp_path / "dropin"))
    assert r.returncode == 0, r.stderr[-4000:]


@pytest.mark.gpu
def test_reference_simulator_runs_on_b200():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.exists(PREBUILT):
        pytest.skip("tests/cpp/_build/dropin not built (needs /root/reference at build time)")
    env = dict(os.environ, LD_LIBRARY_PATH=LIBDIR)
    r = subprocess.run([PREBUILT], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "dropin OK" in r.stdout
    rows = [l for l in r.stdout.splitlines() if l.startswith("tiny,2,")]
    # 3 conv + 1 fc rows and a total row per algorithm; im2col-only skips the fc layer
    assert len(rows) == 4 * 5 + 4, r.stdout
