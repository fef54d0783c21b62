"""The reference-shaped C++ shim (include/convgemm_b200.hpp) compiles against the
C-ABI library and behaves like the reference API (host checks here; device conv
under -m gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2005_06410_b200")


def build(tmp_path):
    exe = str(tmp_path / "shim_test")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_test.cpp"), "-L", LIBDIR, "-lconvgemm_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_host(tmp_path):
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim_test OK" in r.stdout


@pytest.mark.gpu
def test_shim_device(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    r = subprocess.run([build(tmp_path), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
