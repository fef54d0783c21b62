"""B200-native convolution operator O = CONV(F, I) (arXiv 2005.06410, "convgemm").

Host-side mirror of the reference's Python surface
(``/root/reference/proj/python/convgemm/__init__.py``, ``python/src/bindings.cpp:113-285``)
over the C-ABI in ``include/convgemm_b200.h``: same names (``conv_gemm``,
``conv_im2col_gemm``, ``im2col``, ``output_dims``, ``gemm_dims``,
``im2col_workspace_bytes``, ``ConvParams``, ``BlockingParams``), same argument
meaning, same exception mapping (``InvalidGeometry``/``DimensionMismatch`` ->
``ValueError``, ``AllocationFailure`` -> ``MemoryError``, bindings.cpp:117-121).

Tensors use the reference's leftmost-fastest layouts (tensor.hpp:28-50):
F (k_n, k_h, k_w, c_i), I (h_i, w_i, c_i, b), O (k_n, h_o, w_o, b), given as
Fortran-ordered 4-D arrays. CUDA ``torch`` tensors run on the device on the current
stream (asynchronous); numpy arrays take the synchronous host path
(``cgb_conv_host``: H2D, kernel, D2H), which is the reference's call semantics.

Extra over the reference: ``precision`` in {"auto", "3xtf32", "tf32", "ffma"}.
"auto" is fp32-accurate (3xTF32 on the tensor cores, FFMA for K < 32).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import BlockingParamsC, ConvParamsC, lib

__all__ = [
    "AllocationFailure", "BlockingParams", "ConvParams", "DimensionMismatch", "InvalidGeometry",
    "conv", "conv_gemm", "conv_im2col_gemm", "convgemm_scratch_bytes", "empty_tensor4", "gemm_dims",
    "im2col", "im2col_workspace_bytes", "output_dims", "scratch_peak_bytes", "scratch_reset_peak",
    "scratch_set_limit", "kernel_launch_count", "last_path", "PRECISIONS", "ALGOS", "gemm", "conv_direct",
    "set_tuning", "get_tuning", "tuning",
    "IoError", "conv_workspace_bytes", "gemm_workspace_bytes", "LayerSpec", "ModelSpec", "LayerResult", "ParseError", "UnknownLayerKind", "parse_model",
    "model_workspace_bytes", "run_inference", "write_csv",
]

ALGOS = {"explicit": 0, "im2col": 0, "fused": 1, "convgemm": 1, "direct": 2}
PRECISIONS = {"auto": 0, "3xtf32": 1, "tf32": 2, "ffma": 3}
PATHS = {0: "none", 1: "tcgen05-implicit", 2: "tcgen05-explicit", 3: "ffma-implicit", 4: "ffma-explicit",
         5: "tcgen05-shifted", 6: "tcgen05-gather", 7: "tcgen05-shifted-wim", 8: "direct"}


class InvalidGeometry(ValueError):
    """convgemm::InvalidGeometry (types.hpp:15)."""


class DimensionMismatch(ValueError):
    """convgemm::DimensionMismatch (types.hpp:19)."""


class AllocationFailure(MemoryError):
    """convgemm::AllocationFailure (types.hpp:23)."""


class IoError(OSError):
    """convgemm::IoError (types.hpp:25-29)."""


class DeviceError(RuntimeError):
    """A CUDA runtime failure inside the operator (no reference equivalent)."""


class Unsupported(ValueError):
    pass


_ERR = {1: InvalidGeometry, 2: DimensionMismatch, 3: AllocationFailure, 4: ValueError, 5: DeviceError,
        6: Unsupported}


def _check(rc: int) -> None:
    if rc:
        raise _ERR.get(rc, RuntimeError)(lib.cgb_last_error().decode())


@dataclass
class ConvParams:
    """convgemm::ConvParams (conv_params.hpp:8-16)."""
    k_n: int = 1
    k_h: int = 1
    k_w: int = 1
    c_i: int = 1
    h_i: int = 1
    w_i: int = 1
    b: int = 1
    s: int = 1
    p: int = 0

    def c(self) -> ConvParamsC:
        return ConvParamsC(self.k_n, self.k_h, self.k_w, self.c_i, self.h_i, self.w_i, self.b, self.s, self.p)

    @staticmethod
    def of(cp) -> "ConvParams":
        if isinstance(cp, ConvParams):
            return cp
        if isinstance(cp, dict):
            return ConvParams(**{k: int(v) for k, v in cp.items()})
        return ConvParams(*[int(v) for v in cp])


@dataclass
class BlockingParams:
    """convgemm::BlockingParams (blocking.hpp:11-17); validated, GPU tiling is internal."""
    mc: int = 120
    nc: int = 3072
    kc: int = 640
    mr: int = 8
    nr: int = 12

    def c(self) -> BlockingParamsC:
        return BlockingParamsC(self.mc, self.nc, self.kc, self.mr, self.nr)


def output_dims(cp) -> tuple[int, int]:
    """(h_o, w_o) = floor((h_i - k_h + 2p)/s) + 1 ... (conv_params.hpp:27-36)."""
    h, w = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.cgb_output_dims(ctypes.byref(ConvParams.of(cp).c()), ctypes.byref(h), ctypes.byref(w)))
    return h.value, w.value


def gemm_dims(cp) -> tuple[int, int, int]:
    """(m, n, k) = (k_n, h_o*w_o*b, k_h*k_w*c_i) (conv_params.hpp:40-43)."""
    m, n, k = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib.cgb_gemm_dims(ctypes.byref(ConvParams.of(cp).c()), ctypes.byref(m), ctypes.byref(n),
                             ctypes.byref(k)))
    return m.value, n.value, k.value


def im2col_workspace_bytes(cp) -> int:
    """k*n*4 bytes (im2col.hpp:36-39)."""
    v = lib.cgb_im2col_workspace_bytes(ctypes.byref(ConvParams.of(cp).c()))
    if v < 0:
        output_dims(cp)  # raises InvalidGeometry with the message
    return v


def convgemm_scratch_bytes(blocking: BlockingParams | None = None) -> int:
    """The reference's fused-path workspace formula (im2col.hpp:41-44), for API parity."""
    bp = blocking or BlockingParams()
    return (bp.mc * bp.kc + bp.kc * bp.nc) * 4


def conv_workspace_bytes(cp, algo: str = "fused", precision: str = "auto") -> int:
    """Device workspace one call takes (filter split + B-hat for the explicit path)."""
    return lib.cgb_conv_workspace_bytes(ALGOS[algo], PRECISIONS[precision], ctypes.byref(ConvParams.of(cp).c()))


def gemm_workspace_bytes(m: int, n: int, k: int, precision: str = "auto") -> int:
    """Device workspace one ``gemm`` call takes (cgb_gemm_workspace_bytes)."""
    return lib.cgb_gemm_workspace_bytes(PRECISIONS[precision], m, n, k)


def scratch_peak_bytes() -> int:
    return lib.cgb_scratch_peak_bytes()


def scratch_reset_peak() -> None:
    lib.cgb_scratch_reset_peak()


def scratch_set_limit(nbytes: int) -> None:
    lib.cgb_scratch_set_limit(nbytes)


def kernel_launch_count() -> int:
    return lib.cgb_kernel_launch_count()


def last_path() -> str:
    return PATHS.get(lib.cgb_last_path(), "?")


def set_tuning(key: str, value: int) -> None:
    """Dispatch-policy knob (include/convgemm_b200.h cgb_set_tuning); every setting is correct."""
    _check(lib.cgb_set_tuning(key.encode(), int(value)))


def get_tuning(key: str) -> int:
    v = ctypes.c_int64()
    _check(lib.cgb_get_tuning(key.encode(), ctypes.byref(v)))
    return v.value


class tuning:
    """Context manager: ``with tuning(sk=2, tail=0): ...`` sets knobs and restores them."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_tuning(k)
            set_tuning(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_tuning(k, v)
        return False


# ----------------------------------------------------------------------------- tensors
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def empty_tensor4(d0, d1, d2, d3, device="cuda", dtype=None):
    """A Fortran-ordered (leftmost-fastest) torch tensor of shape (d0, d1, d2, d3)."""
    import torch
    return torch.empty((d3, d2, d1, d0), device=device, dtype=dtype or torch.float32).permute(3, 2, 1, 0)


def _expect_shape(x, shape, name):
    if tuple(x.shape) != tuple(shape):
        raise InvalidGeometry(f"{name} tensor extents {tuple(x.shape)} disagree with ConvParams {tuple(shape)}")


def _torch_ptr(x, name, writable=False, dtype=None):
    import torch
    if not x.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (or a numpy array for the host path)")
    if x.dtype != (dtype or torch.float32):
        raise Unsupported(f"{name}: expected {dtype or torch.float32} on this path (got {x.dtype})")
    d = x.shape
    expect = (1, d[0], d[0] * d[1], d[0] * d[1] * d[2])
    if x.dim() != 4 or (x.numel() > 0 and tuple(x.stride()) != expect):
        raise ValueError(f"{name} must be a leftmost-fastest (Fortran-ordered) rank-4 tensor")
    return x.data_ptr()


def _shapes(cp: ConvParams):
    h_o, w_o = output_dims(cp)
    return ((cp.k_n, cp.k_h, cp.k_w, cp.c_i), (cp.h_i, cp.w_i, cp.c_i, cp.b), (cp.k_n, h_o, w_o, cp.b))


def conv(F, I, cp, algo: str = "fused", precision: str = "auto", out=None, stream=None, workspace=None,
         blocking: BlockingParams | None = None):
    """O = CONV(F, I). ``algo`` in {"fused", "explicit", "direct"} (bench.hpp:13-19:
    ConvGemm, Im2col, Direct). float32 runs the B200 operator (``precision``); float64
    (numpy or torch) runs the reference's f64 arithmetic bit for bit on the device's
    FP64 cores (``blocking.kc`` sets the accumulation blocks, as in the reference)."""
    cp = ConvParams.of(cp)
    fs, is_, os_ = _shapes(cp)
    a, p = ALGOS[algo], PRECISIONS[precision]
    bp = ctypes.byref(blocking.c()) if blocking is not None else None
    if _is_torch(F):
        import torch
        _expect_shape(F, fs, "filter")
        _expect_shape(I, is_, "input")
        f64 = F.dtype == torch.float64
        if f64 != (I.dtype == torch.float64):
            raise Unsupported("filter and input must have the same dtype")
        if out is None:
            out = empty_tensor4(*os_, device=F.device, dtype=F.dtype)
        _expect_shape(out, os_, "output")
        st = stream if stream is not None else torch.cuda.current_stream(F.device).cuda_stream
        if f64:
            _check(lib.cgb_conv_f64(a, _torch_ptr(F, "filter", dtype=torch.float64),
                                    _torch_ptr(I, "input", dtype=torch.float64), ctypes.byref(cp.c()), bp,
                                    _torch_ptr(out, "output", dtype=torch.float64), st))
            return out
        ws_ptr, ws_bytes = (workspace.data_ptr(), workspace.numel() * workspace.element_size()) \
            if workspace is not None else (None, 0)
        _check(lib.cgb_conv(a, p, _torch_ptr(F, "filter"), _torch_ptr(I, "input"), ctypes.byref(cp.c()),
                            _torch_ptr(out, "output"), ws_ptr, ws_bytes, st))
        return out
    # host path: numpy arrays (reference semantics, synchronous)
    dt = np.float64 if (np.asarray(F).dtype == np.float64 or np.asarray(I).dtype == np.float64) else np.float32
    F = np.asfortranarray(F, dtype=dt)
    I = np.asfortranarray(I, dtype=dt)
    _expect_shape(F, fs, "filter")
    _expect_shape(I, is_, "input")
    if out is None:
        out = np.empty(os_, dtype=dt, order="F")
    _expect_shape(out, os_, "output")
    if not out.flags.f_contiguous or out.dtype != dt:
        raise ValueError(f"output must be a Fortran-ordered {np.dtype(dt).name} array")
    if dt == np.float64:
        _check(lib.cgb_conv_host_f64(a, F.ctypes.data, I.ctypes.data, ctypes.byref(cp.c()), bp, out.ctypes.data))
        return out
    _check(lib.cgb_conv_host(a, p, F.ctypes.data, I.ctypes.data, ctypes.byref(cp.c()), out.ctypes.data, None))
    return out


def _validate_blocking(blocking):
    if blocking is not None:
        _check(lib.cgb_validate_blocking(ctypes.byref(blocking.c())))


def conv_gemm(F, I, cp, blocking: BlockingParams | None = None, threads: int = 1, precision: str = "auto",
              out=None):
    """Fused ConvGemm (conv.hpp:78-91): im2col happens inside the operand staging."""
    _validate_blocking(blocking)
    return conv(F, I, cp, "fused", precision, out, blocking=blocking)


def conv_im2col_gemm(F, I, cp, blocking: BlockingParams | None = None, threads: int = 1, precision: str = "auto",
                     out=None):
    """Explicit im2col + GEMM (conv.hpp:60-74): B-hat is materialised in HBM."""
    _validate_blocking(blocking)
    return conv(F, I, cp, "explicit", precision, out, blocking=blocking)


def conv_direct(F, I, cp, out=None):
    """The reference's seven-loop convolution (conv.hpp:24-55) on the device, bit-identical
    to the reference's conv_direct<float> / <double>: the checker of run_inference."""
    return conv(F, I, cp, "direct", "auto", out)


def gemm(A, B, blocking: BlockingParams | None = None, threads: int = 1, precision: str = "auto", out=None):
    """C = A @ B for column-major (Fortran-ordered) float32 matrices, the reference's
    ``gemm`` binding (bindings.cpp:200-210; gemm.hpp:46-105 over a MatrixSource). Runs as
    a 1x1 convolution over 1x1 images through ``cgb_gemm``: CUDA tensors on the current
    stream, numpy arrays synchronously (copied through the device)."""
    import torch
    _validate_blocking(blocking)
    host = not _is_torch(A)
    if host:
        An, Bn = np.asarray(A), np.asarray(B)
        if An.dtype == np.float64 or Bn.dtype == np.float64:
            # the reference's gemm<double> bit for bit on the device's FP64 cores
            An = np.asfortranarray(An, dtype=np.float64)
            Bn = np.asfortranarray(Bn, dtype=np.float64)
            if An.ndim != 2 or Bn.ndim != 2 or An.shape[1] != Bn.shape[0]:
                raise DimensionMismatch("gemm operand extents disagree")
            m, k = An.shape
            n = Bn.shape[1]
            C = np.zeros((m, n), dtype=np.float64, order="F")
            bp = ctypes.byref(blocking.c()) if blocking is not None else None
            _check(lib.cgb_gemm_host_f64(An.ctypes.data, m, Bn.ctypes.data, k, C.ctypes.data, m, m, n, k, bp, 0))
            return C
        A = torch.from_numpy(np.ascontiguousarray(An.astype(np.float32).T)).cuda().t()
        B = torch.from_numpy(np.ascontiguousarray(Bn.astype(np.float32).T)).cuda().t()
    if A.dim() != 2 or B.dim() != 2:
        raise DimensionMismatch("gemm operands must be matrices")
    m, k = A.shape
    k2, n = B.shape
    if k2 != k:
        raise DimensionMismatch(f"gemm inner dimensions disagree: {m}x{k} times {k2}x{n}")
    for x, nm in ((A, "a"), (B, "b")):
        if not x.is_cuda or x.dtype != torch.float32 or x.stride(0) != 1:
            raise ValueError(f"{nm} must be a column-major (Fortran-ordered) float32 CUDA matrix")
    if A.stride(1) != m:
        raise DimensionMismatch("a must be dense (leading dimension == rows)")
    C = out if out is not None else torch.empty((n, m), device=A.device, dtype=torch.float32).t()
    if tuple(C.shape) != (m, n) or C.stride(0) != 1 or C.stride(1) != m:
        raise DimensionMismatch("output must be a dense column-major m x n float32 matrix")
    st = torch.cuda.current_stream(A.device).cuda_stream
    _check(lib.cgb_gemm(PRECISIONS[precision], A.data_ptr(), m, B.data_ptr(), max(B.stride(1), k), C.data_ptr(), m,
                        m, n, k, None, 0, st))
    if host:
        return np.asfortranarray(C.cpu().numpy())
    return C


def im2col(I, cp, threads: int = 1, ldb: int | None = None, out=None):
    """Lowered matrix B (k x n, column-major) from the device kernel; bit-exact with im2col<float>
    (and im2col<double> for float64 input)."""
    import torch
    cp = ConvParams.of(cp)
    _, is_, _ = _shapes(cp)
    _, n, k = gemm_dims(cp)
    ldb = k if ldb is None else ldb
    host = not _is_torch(I)
    if host and np.asarray(I).dtype == np.float64:
        In = np.asfortranarray(I, dtype=np.float64)
        _expect_shape(In, is_, "input")
        B = np.zeros((ldb, n), dtype=np.float64, order="F")
        _check(lib.cgb_im2col_host_f64(In.ctypes.data, ctypes.byref(cp.c()), B.ctypes.data, ldb))
        return B[:k]
    if host:
        I = torch.from_numpy(np.asfortranarray(I, dtype=np.float32).reshape(-1, order="F")).cuda()
        I = I.view(cp.b, cp.c_i, cp.w_i, cp.h_i).permute(3, 2, 1, 0)
    _expect_shape(I, is_, "input")
    B = torch.empty((n, ldb), device=I.device, dtype=torch.float32) if out is None else out
    st = torch.cuda.current_stream(I.device).cuda_stream
    _check(lib.cgb_im2col(_torch_ptr(I, "input"), ctypes.byref(cp.c()), B.data_ptr(), ldb, st))
    Bt = B.t()[:k]  # (k, n) view with column stride ldb
    if host:
        return np.asfortranarray(Bt.cpu().numpy())
    return Bt


from .simulator import (  # noqa: E402  (the simulator builds on the entry points above)
    LayerResult, LayerSpec, ModelSpec, ParseError, UnknownLayerKind, model_workspace_bytes, parse_model,
    run_inference, write_csv)
