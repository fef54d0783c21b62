"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes loaders for the two CPU checkers:

* ``Restatement`` -> ``oracle/_build/liboracle.so`` (plain-C restatement of the
  reference conv path, ``oracle/conv_oracle.c``; bit-identical to the reference
  operator, pinned by ``tests/test_oracle.py``).
* ``Reference``   -> ``oracle/_ref/libconvgemm_ref.so`` (the reference's own
  header-only library compiled from ``/root/reference`` by ``oracle/Makefile``;
  ``oracle/ref_capi.cpp`` forwards to ``conv_gemm`` / ``conv_im2col_gemm`` /
  ``conv_direct`` / ``im2col`` of ``proj/include/convgemm/conv.hpp`` and
  ``im2col.hpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module, and only to check or to time the CPU baseline. The product
package ``paper_2005_06410_b200`` never imports it.

Tensors are numpy arrays in the reference's leftmost-fastest layouts
(``conv_params.hpp``/``tensor.hpp:28-50``), passed as Fortran-ordered 4-D
arrays: F (k_n, k_h, k_w, c_i), I (h_i, w_i, c_i, b), O (k_n, h_o, w_o, b).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "_build", "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libconvgemm_ref.so")
REFERENCE_SRC = "/root/reference/proj"

_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p

KIND_DIRECT, KIND_EXPLICIT, KIND_FUSED = 0, 1, 2
ERRORS = {1: "InvalidGeometry", 2: "DimensionMismatch", 3: "AllocationFailure",
          4: "invalid_argument", 9: "runtime_error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


def build(reference: bool = True) -> None:
    """Build the restatement and, when /root/reference exists, oracle/_ref."""
    targets = ["oracle"]
    if reference and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _cp_array(cp) -> ctypes.Array:
    vals = [cp[k] for k in ("k_n", "k_h", "k_w", "c_i", "h_i", "w_i", "b", "s", "p")] \
        if isinstance(cp, dict) else list(cp)
    return (ctypes.c_int64 * 9)(*[int(v) for v in vals])


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def output_dims_py(cp) -> tuple[int, int]:
    a = list(_cp_array(cp))
    k_n, k_h, k_w, c_i, h_i, w_i, b, s, p = a
    if min(k_n, k_h, k_w, c_i, h_i, w_i, b, s) < 1 or p < 0:
        raise OracleError(1, "conv extents must be positive (padding non-negative)")
    dh, dw = h_i - k_h + 2 * p, w_i - k_w + 2 * p
    if dh < 0 or dw < 0:
        raise OracleError(1, "filter exceeds padded input")
    return dh // s + 1, dw // s + 1


class Restatement:
    """The plain-C restatement (oracle/conv_oracle.c)."""

    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            build(reference=False)
        lib = ctypes.CDLL(path)
        for name in ("orc_conv_direct_f32", "orc_conv_gemm_f32", "orc_im2col_f32",
                     "orc_conv_f64acc", "orc_output_scale", "orc_output_dims"):
            getattr(lib, name).restype = ctypes.c_int
        lib.orc_conv_direct_f32.argtypes = [_vp, _vp, _i64p, _vp]
        lib.orc_conv_gemm_f32.argtypes = [_vp, _vp, _i64p, ctypes.c_int64, _vp]
        lib.orc_im2col_f32.argtypes = [_vp, _i64p, _vp, ctypes.c_int64]
        lib.orc_conv_f64acc.argtypes = [_vp, _vp, _i64p, _vp]
        lib.orc_output_scale.argtypes = [_vp, _vp, _i64p, _vp]
        lib.orc_output_dims.argtypes = [_i64p, _i64p, _i64p]
        self.lib = lib

    def _check(self, rc):
        if rc:
            raise OracleError(rc)

    def output_dims(self, cp):
        h, w = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.orc_output_dims(_cp_array(cp), ctypes.byref(h), ctypes.byref(w)))
        return h.value, w.value

    def _out(self, cp, dtype=np.float32):
        h_o, w_o = self.output_dims(cp)
        a = list(_cp_array(cp))
        return np.zeros((a[0], h_o, w_o, a[6]), dtype=dtype, order="F")

    def conv_direct(self, F, I, cp):
        O = self._out(cp)
        self._check(self.lib.orc_conv_direct_f32(_ptr(F), _ptr(I), _cp_array(cp), _ptr(O)))
        return O

    def conv_gemm(self, F, I, cp, kc: int = 640):
        O = self._out(cp)
        self._check(self.lib.orc_conv_gemm_f32(_ptr(F), _ptr(I), _cp_array(cp), kc, _ptr(O)))
        return O

    def conv_f64(self, F, I, cp):
        O = self._out(cp, np.float64)
        self._check(self.lib.orc_conv_f64acc(_ptr(F), _ptr(I), _cp_array(cp), _ptr(O)))
        return O

    def output_scale(self, F, I, cp):
        S = self._out(cp, np.float64)
        self._check(self.lib.orc_output_scale(_ptr(F), _ptr(I), _cp_array(cp), _ptr(S)))
        return S

    def im2col(self, I, cp, ldb: int | None = None):
        a = list(_cp_array(cp))
        h_o, w_o = self.output_dims(cp)
        k, n = a[1] * a[2] * a[3], h_o * w_o * a[6]
        ldb = k if ldb is None else ldb
        B = np.zeros((ldb, n), dtype=np.float32, order="F")
        self._check(self.lib.orc_im2col_f32(_ptr(I), _cp_array(cp), _ptr(B), ldb))
        return B


class Reference:
    """The reference operator itself (oracle/_ref/libconvgemm_ref.so)."""

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            build(reference=True)
        lib = ctypes.CDLL(path)
        lib.ref_conv.argtypes = [ctypes.c_int, ctypes.c_int, _vp, _vp, _i64p, _i64p, ctypes.c_int, _vp]
        lib.ref_conv.restype = ctypes.c_int
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_output_dims.argtypes = [_i64p, _i64p, _i64p]
        lib.ref_gemm_dims.argtypes = [_i64p, _i64p, _i64p, _i64p]
        lib.ref_im2col_f32.argtypes = [_vp, _i64p, ctypes.c_int, _vp]
        lib.ref_gemm_f32.argtypes = [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int]
        lib.ref_gemm_f64.argtypes = [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int]
        lib.ref_im2col_f64.argtypes = [_vp, _i64p, ctypes.c_int, _vp]
        lib.ref_im2col_workspace_bytes.argtypes = [_i64p]
        lib.ref_im2col_workspace_bytes.restype = ctypes.c_int64
        lib.ref_convgemm_scratch_bytes.argtypes = [_i64p]
        lib.ref_convgemm_scratch_bytes.restype = ctypes.c_int64
        lib.ref_pack_check.argtypes = [_vp, _i64p, _i64p, _i64p]
        lib.ref_pack_check.restype = ctypes.c_int64
        lib.ref_rng_new.argtypes = [ctypes.c_uint64]
        lib.ref_rng_new.restype = _vp
        lib.ref_rng_free.argtypes = [_vp]
        lib.ref_rng_fill_uniform_f32.argtypes = [_vp, _vp, ctypes.c_int64]
        lib.ref_rng_fill_uniform_f64.argtypes = [_vp, _vp, ctypes.c_int64]
        lib.ref_rng_random_conv_params.argtypes = [_vp, ctypes.c_int64, ctypes.c_int64, _i64p]
        lib.ref_rng_rand_in.argtypes = [_vp, ctypes.c_int64, ctypes.c_int64]
        lib.ref_rng_rand_in.restype = ctypes.c_int64
        lib.ref_scratch_peak_bytes.restype = ctypes.c_uint64
        lib.ref_scratch_set_limit.argtypes = [ctypes.c_uint64]
        self.lib = lib

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def output_dims(self, cp):
        h, w = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.ref_output_dims(_cp_array(cp), ctypes.byref(h), ctypes.byref(w)))
        return h.value, w.value

    def conv(self, kind, F, I, cp, threads=1, bp=None, O=None):
        dtype = np.float64 if F.dtype == np.float64 else np.float32
        a = list(_cp_array(cp))
        if O is None:
            h_o, w_o = output_dims_py(cp)
            O = np.zeros((a[0], h_o, w_o, a[6]), dtype=dtype, order="F")
        bpa = (ctypes.c_int64 * 5)(*bp) if bp is not None else None
        self._check(self.lib.ref_conv(kind, 1 if dtype == np.float64 else 0, _ptr(F), _ptr(I),
                                      _cp_array(cp), bpa, threads, _ptr(O)))
        return O

    def conv_direct(self, F, I, cp):
        return self.conv(KIND_DIRECT, F, I, cp)

    def conv_gemm(self, F, I, cp, threads=1, bp=None, O=None):
        return self.conv(KIND_FUSED, F, I, cp, threads, bp, O)

    def conv_im2col_gemm(self, F, I, cp, threads=1, bp=None, O=None):
        return self.conv(KIND_EXPLICIT, F, I, cp, threads, bp, O)

    def im2col(self, I, cp, threads=1):
        a = list(_cp_array(cp))
        h_o, w_o = output_dims_py(cp)
        f64 = I.dtype == np.float64
        B = np.zeros((a[1] * a[2] * a[3], h_o * w_o * a[6]), dtype=np.float64 if f64 else np.float32, order="F")
        fn = self.lib.ref_im2col_f64 if f64 else self.lib.ref_im2col_f32
        self._check(fn(_ptr(I), _cp_array(cp), threads, _ptr(B)))
        return B

    def gemm(self, A, B, bp=None, threads=1):
        """Column-major C = A @ B through the reference's blocked gemm (gemm.hpp:46-105)."""
        f64 = A.dtype == np.float64
        A = np.asfortranarray(A, dtype=np.float64 if f64 else np.float32)
        B = np.asfortranarray(B, dtype=A.dtype)
        m, k = A.shape
        n = B.shape[1]
        C = np.zeros((m, n), dtype=A.dtype, order="F")
        bpa = (ctypes.c_int64 * 5)(*bp) if bp is not None else None
        fn = self.lib.ref_gemm_f64 if f64 else self.lib.ref_gemm_f32
        self._check(fn(_ptr(A), _ptr(B), _ptr(C), m, n, k, bpa, threads))
        return C

    # --- the reference tests' generators (proj/tests/oracles.hpp:48-91) ---
    def rng(self, seed: int) -> "RefRng":
        return RefRng(self, seed)


class RefRng:
    """std::mt19937_64 stream driving testutil::random_tensor / random_conv_params."""

    def __init__(self, ref: Reference, seed: int):
        self.lib = ref.lib
        self.h = self.lib.ref_rng_new(seed)

    def __del__(self):
        try:
            self.lib.ref_rng_free(self.h)
        except Exception:
            pass

    def tensor(self, d0, d1, d2, d3, dtype=np.float32):
        t = np.zeros((d0, d1, d2, d3), dtype=dtype, order="F")
        fill = self.lib.ref_rng_fill_uniform_f64 if dtype == np.float64 else self.lib.ref_rng_fill_uniform_f32
        fill(self.h, _ptr(t), t.size)
        return t

    def conv_params(self, cap=8, max_batch=3):
        out = (ctypes.c_int64 * 9)()
        self.lib.ref_rng_random_conv_params(self.h, cap, max_batch, out)
        return dict(zip(("k_n", "k_h", "k_w", "c_i", "h_i", "w_i", "b", "s", "p"), list(out)))

    def rand_in(self, lo, hi):
        return self.lib.ref_rng_rand_in(self.h, lo, hi)


def per_output_error(O, ref, scale):
    """North-star metric: max |O - ref| / (||F[i_k]|| * ||B[:, col]||) per output
    (BASELINE.json north_star). Zero-scale outputs are exact zeros."""
    d = np.abs(O.astype(np.float64) - ref.astype(np.float64))
    s = np.where(scale > 0, scale, 1.0)
    return float(np.max(d / s)) if d.size else 0.0


def normalized_max_error(a, ref):
    """The reference's global metric, proj/tests/oracles.hpp:36-46."""
    ref = ref.astype(np.float64)
    scale = max(1.0, float(np.max(np.abs(ref)))) if ref.size else 1.0
    return float(np.max(np.abs(a.astype(np.float64) - ref))) / scale if ref.size else 0.0
