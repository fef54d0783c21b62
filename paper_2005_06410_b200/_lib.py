"""ctypes binding of the C-ABI (``include/convgemm_b200.h``).

The product path is the CUDA library ``libconvgemm_b200.so`` built in-tree by
``build.py``. There is no CPU fallback: if the library is missing or cannot be
loaded, importing this module raises ``ImportError``.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CGB_LIB_OVERRIDE: tools/ load the profiling build (libconvgemm_b200_prof.so) this way
LIB_PATH = os.environ.get("CGB_LIB_OVERRIDE") or os.path.join(HERE, "libconvgemm_b200.so")

# exported symbols, in include/convgemm_b200.h order
SYMBOLS = (
    "cgb_output_dims", "cgb_gemm_dims", "cgb_im2col_workspace_bytes", "cgb_validate_blocking",
    "cgb_conv_workspace_bytes", "cgb_gemm_workspace_bytes", "cgb_conv", "cgb_conv_gemm", "cgb_conv_im2col_gemm", "cgb_im2col",
    "cgb_gemm", "cgb_conv_host", "cgb_scratch_current_bytes", "cgb_scratch_peak_bytes", "cgb_scratch_reset_peak",
    "cgb_scratch_set_limit", "cgb_scratch_release", "cgb_last_error", "cgb_version",
    "cgb_kernel_launch_count", "cgb_last_path", "cgb_debug_sw_stats", "cgb_set_tuning", "cgb_get_tuning",
    "cgb_scratch_cached_bytes", "cgb_im2col_host", "cgb_gemm_host",
    "cgb_conv_f64", "cgb_conv_host_f64", "cgb_im2col_host_f64", "cgb_gemm_host_f64",
)


class ConvParamsC(ctypes.Structure):
    """cgb_conv_params == convgemm::ConvParams (conv_params.hpp:8-16)."""
    _fields_ = [(n, ctypes.c_int64) for n in ("k_n", "k_h", "k_w", "c_i", "h_i", "w_i", "b", "s", "p")]


class BlockingParamsC(ctypes.Structure):
    """cgb_blocking_params == convgemm::BlockingParams (blocking.hpp:11-17)."""
    _fields_ = [(n, ctypes.c_int64) for n in ("mc", "nc", "kc", "mr", "nr")]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 convolution operator)")
    lib = ctypes.CDLL(LIB_PATH)
    i64, i64p, vp, st = ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.c_int
    cpp = ctypes.POINTER(ConvParamsC)
    bpp = ctypes.POINTER(BlockingParamsC)
    sig = {
        "cgb_output_dims": (st, [cpp, i64p, i64p]),
        "cgb_gemm_dims": (st, [cpp, i64p, i64p, i64p]),
        "cgb_im2col_workspace_bytes": (i64, [cpp]),
        "cgb_validate_blocking": (st, [bpp]),
        "cgb_conv_workspace_bytes": (i64, [ctypes.c_int, ctypes.c_int, cpp]),
        "cgb_gemm_workspace_bytes": (i64, [ctypes.c_int, i64, i64, i64]),
        "cgb_conv": (st, [ctypes.c_int, ctypes.c_int, vp, vp, cpp, vp, vp, ctypes.c_size_t, vp]),
        "cgb_conv_gemm": (st, [vp, vp, cpp, bpp, ctypes.c_int, vp, ctypes.c_int, vp]),
        "cgb_conv_im2col_gemm": (st, [vp, vp, cpp, bpp, ctypes.c_int, vp, ctypes.c_int, vp]),
        "cgb_im2col": (st, [vp, cpp, vp, i64, vp]),
        "cgb_gemm": (st, [ctypes.c_int, vp, i64, vp, i64, vp, i64, i64, i64, i64, vp, ctypes.c_size_t, vp]),
        "cgb_conv_host": (st, [ctypes.c_int, ctypes.c_int, vp, vp, cpp, vp, vp]),
        "cgb_scratch_current_bytes": (ctypes.c_uint64, []),
        "cgb_scratch_peak_bytes": (ctypes.c_uint64, []),
        "cgb_scratch_reset_peak": (None, []),
        "cgb_scratch_set_limit": (None, [ctypes.c_uint64]),
        "cgb_scratch_release": (None, []),
        "cgb_scratch_cached_bytes": (ctypes.c_uint64, []),
        "cgb_im2col_host": (st, [vp, cpp, vp, i64]),
        "cgb_gemm_host": (st, [ctypes.c_int, vp, i64, vp, i64, vp, i64, i64, i64, i64, ctypes.c_int]),
        "cgb_conv_f64": (st, [ctypes.c_int, vp, vp, cpp, bpp, vp, vp]),
        "cgb_conv_host_f64": (st, [ctypes.c_int, vp, vp, cpp, bpp, vp]),
        "cgb_im2col_host_f64": (st, [vp, cpp, vp, i64]),
        "cgb_gemm_host_f64": (st, [vp, i64, vp, i64, vp, i64, i64, i64, i64, bpp, ctypes.c_int]),
        "cgb_last_error": (ctypes.c_char_p, []),
        "cgb_version": (ctypes.c_char_p, []),
        "cgb_kernel_launch_count": (ctypes.c_uint64, []),
        "cgb_last_path": (ctypes.c_int, []),
        "cgb_debug_sw_stats": (ctypes.c_int, [vp, ctypes.c_int]),
        "cgb_set_tuning": (st, [ctypes.c_char_p, i64]),
        "cgb_get_tuning": (st, [ctypes.c_char_p, i64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
