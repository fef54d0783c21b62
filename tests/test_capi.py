"""CPU: the C-ABI library loads without a GPU, exports every symbol declared in
include/convgemm_b200.h, and its host-only geometry entry points reproduce the
reference's formulas and error behaviour (conv_params.hpp:27-43, im2col.hpp:36-39,
blocking.hpp:22-29). No device compute runs here."""
import ctypes
import os
import re

import pytest

import paper_2005_06410_b200 as cg
from paper_2005_06410_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "convgemm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cgb_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    syms = header_symbols()
    assert len(syms) >= 19
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/convgemm_b200.h but not exported"
    assert set(syms) == set(_lib.SYMBOLS)


def test_library_is_sm100a_cuda():
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob


def test_output_and_gemm_dims():
    assert cg.output_dims(dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=56, w_i=56, b=128, s=1, p=1)) == (56, 56)
    assert cg.output_dims((64, 3, 3, 128, 56, 56, 128, 2, 1)) == (28, 28)
    assert cg.output_dims((64, 7, 7, 3, 224, 224, 256, 2, 3)) == (112, 112)
    assert cg.gemm_dims((64, 3, 3, 64, 56, 56, 128, 1, 1)) == (64, 401408, 576)
    assert cg.gemm_dims((2048, 1, 1, 512, 7, 7, 256, 1, 0)) == (2048, 12544, 512)
    # AlexNet triples (test_bench.cpp:292-296) at b=1
    assert cg.gemm_dims((64, 11, 11, 3, 227, 227, 1, 4, 0)) == (64, 3025, 363)


def test_invalid_geometry():
    with pytest.raises(cg.InvalidGeometry):
        cg.output_dims((1, 5, 5, 1, 3, 3, 1, 1, 0))  # filter exceeds padded input
    with pytest.raises(cg.InvalidGeometry):
        cg.output_dims((1, 1, 1, 1, 3, 3, 1, 0, 0))  # stride 0
    with pytest.raises(ValueError):
        cg.output_dims((1, 1, 1, 1, 3, 3, 1, 1, -1))


def test_workspace_formulas():
    # test_conv.cpp:191-199 and test_convgemm.cpp:192-211
    assert cg.im2col_workspace_bytes((192, 5, 5, 64, 55, 55, 1, 1, 0)) == 16646400
    assert cg.im2col_workspace_bytes((64, 3, 3, 64, 224, 224, 1, 1, 1)) == 115605504
    assert cg.convgemm_scratch_bytes() == 8171520
    # the B200 fused path in TF32 mode needs no device workspace at all
    assert cg.conv_workspace_bytes((64, 3, 3, 64, 56, 56, 128, 1, 1), "fused", "tf32") == 0
    # explicit path holds B-hat (k rounded to 4) on top
    assert cg.conv_workspace_bytes((64, 3, 3, 64, 56, 56, 1, 1, 1), "explicit", "tf32") >= 576 * 3136 * 4


def test_gemm_workspace_bytes():
    """gemm (fc layers): no workspace in TF32; in 3xTF32 small A takes its hi/lo split, large static
    weights (> 8 MB: VGG fc6, 411 MB) take none -- their lo tile is split in the kernel
    (no per-call re-split of static weights)."""
    assert cg.gemm_workspace_bytes(4096, 64, 25088, "tf32") == 0
    assert cg.gemm_workspace_bytes(4096, 64, 25088, "auto") == 0
    assert cg.gemm_workspace_bytes(1000, 64, 4096, "3xtf32") == 0
    assert cg.gemm_workspace_bytes(256, 64, 512, "3xtf32") == 2 * 256 * 512 * 4
    assert cg.gemm_workspace_bytes(0, 64, 512) == -1


def test_blocking_validation():
    cg._validate_blocking(cg.BlockingParams())
    with pytest.raises(ValueError):
        cg._validate_blocking(cg.BlockingParams(mc=0))
    with pytest.raises(ValueError):
        cg._validate_blocking(cg.BlockingParams(mr=200, mc=120))


def test_version_and_counters():
    assert b"sm_100a" in _lib.lib.cgb_version()
    assert cg.kernel_launch_count() >= 0


def test_gemm_argument_errors():
    """cgb_gemm validates before touching the device (gemm.hpp:51-53 DimensionMismatch)."""
    L = _lib.lib
    # non-positive dimensions -> InvalidGeometry
    assert L.cgb_gemm(0, 1, 4, 1, 4, 1, 4, 0, 4, 4, None, 0, None) == 1
    # lda != m, ldc != m, ldb < k -> DimensionMismatch
    assert L.cgb_gemm(0, 1, 8, 1, 4, 1, 4, 4, 4, 4, None, 0, None) == 2
    assert L.cgb_gemm(0, 1, 4, 1, 4, 1, 8, 4, 4, 4, None, 0, None) == 2
    assert L.cgb_gemm(0, 1, 4, 1, 3, 1, 4, 4, 4, 4, None, 0, None) == 2
    assert b"ld" in L.cgb_last_error()
    # unknown precision, null pointers -> InvalidArgument
    assert L.cgb_gemm(9, 1, 4, 1, 4, 1, 4, 4, 4, 4, None, 0, None) == 4
    assert L.cgb_gemm(0, None, 4, 1, 4, 1, 4, 4, 4, 4, None, 0, None) == 4


def test_low_channel_workspace():
    """The stem (c_i = 3) takes the w-im2col filter array (k_n x k_h x 32, hi/lo in
    3xTF32) as its fused-path workspace."""
    stem = (64, 7, 7, 3, 224, 224, 256, 2, 3)
    assert cg.conv_workspace_bytes(stem, "fused", "tf32") >= 64 * 7 * 32 * 4
    assert cg.conv_workspace_bytes(stem, "fused", "3xtf32") >= 2 * 64 * 7 * 32 * 4


def test_tuning_knobs_roundtrip_and_no_env():
    """Dispatch-policy knobs go through cgb_set_tuning (the product reads no environment
    variables); unknown keys are rejected with the reference's invalid_argument status."""
    import os
    assert cg.get_tuning("sk") == 1
    with cg.tuning(sk=2, tail=0, host_chunk_kb=20):
        assert (cg.get_tuning("sk"), cg.get_tuning("tail"), cg.get_tuning("host_chunk_kb")) == (2, 0, 20)
    assert (cg.get_tuning("sk"), cg.get_tuning("tail")) == (1, 1)
    with pytest.raises(ValueError):
        cg.set_tuning("no_such_knob", 1)
    os.environ["CGB_SW_SK"] = "2"
    try:
        assert cg.get_tuning("sk") == 1  # the product library ignores the environment
    finally:
        del os.environ["CGB_SW_SK"]
    strings = open(cg._lib.LIB_PATH, "rb").read()
    assert b"CGB_DEBUG_SW" not in strings and b"CGB_SW_SK" not in strings
