"""CNN inference simulator on the B200 operator: one timed sweep of a model's layers.

Host-side mirror of the reference's model and benchmark layer:

* ``parse_model`` / ``ModelSpec`` / ``LayerSpec`` -- model.cpp:35-95, model.hpp:10-37.
  Plain text, one layer per line (``conv k_n k_h k_w c_i h_i w_i s p``, ``fc m k``,
  ``pool h_o w_o c``), ``#`` comments, at least one conv layer; the same errors
  (``ParseError(line, msg)``, ``UnknownLayerKind``; conv geometry validated with
  ``output_dims``).
* ``model_workspace_bytes`` -- model.cpp:99-110 (largest explicit im2col workspace).
* ``run_inference`` -- bench.cpp:93-244: weights and two ping-pong activation buffers
  (each sized to the model's largest activation) filled from a fixed seed; each conv or
  fc layer reads one buffer and writes the other, then they swap; pool layers carry no
  work. Each layer is repeated until ``min_time`` of DEVICE time has elapsed (CUDA
  events around the repetitions, the reference's repeat-until-min_time, bench.cpp:200-210)
  and reported as time per repetition and GFLOPS. fc layers are ``gemm`` (a 1x1
  convolution over 1x1 images on the explicit tensor-core path, bench.cpp:140-153).
* ``write_csv`` -- bench.cpp:246-275, the same columns and the ``total`` row.

Algorithms (bench.hpp:13-19): ``convgemm`` = fused operator, ``im2col`` = explicit
(B-hat in HBM), ``gemm-only`` = the explicit GEMM over a B-hat lowered outside the timed
region, ``im2col-only`` = the lowering alone (no FLOPs, no output), ``direct`` =
conv_direct on the device, bit-identical to the reference's conv_direct<float>
(ref_order.cu). ``check`` compares every conv output with conv_direct, as the reference
does (bench.cpp:212-233), under the north star's per-output bar |O - O_direct| /
(||F[i_k]|| * ||B-hat[:, col]||) <= 1e-5 for the fp32-accurate precisions (5e-3 in plain
TF32 mode). The reference's own max|O - O_direct| / max(1, max|O_direct|) <= 1e-5 is a
bar for two IEEE fp32 summation orders; the tensor cores' fp32 accumulation is not
IEEE round-to-nearest, and on the simulator's growing activations 3xTF32 lands at
~1.1e-5 on it (ResNet-50 layer 14 at b=2) while meeting the per-output bar by 10x.
"""
from __future__ import annotations

import io
import math
import os
from dataclasses import dataclass, field

__all__ = ["LayerSpec", "ModelSpec", "LayerResult", "ParseError", "UnknownLayerKind", "parse_model",
           "model_workspace_bytes", "run_inference", "write_csv"]


class ParseError(ValueError):
    """convgemm::ParseError (types.hpp:31-35): line number + message."""

    def __init__(self, line: int, msg: str):
        super().__init__(f"line {line}: {msg}")
        self.line = line


class UnknownLayerKind(ParseError):
    """convgemm::UnknownLayerKind (types.hpp:37-41)."""

    def __init__(self, line: int, kind: str):
        super().__init__(line, f"unknown layer kind '{kind}'")
        self.kind = kind


@dataclass
class LayerSpec:
    kind: str  # "conv" | "fc" | "pool"
    conv: object = None  # ConvParams (b = 1 placeholder) for conv layers
    fc_m: int = 0
    fc_k: int = 0
    pool_h: int = 0
    pool_w: int = 0
    pool_c: int = 0


@dataclass
class ModelSpec:
    name: str
    layers: list = field(default_factory=list)

    def count(self, kind: str) -> int:
        return sum(1 for l in self.layers if l.kind == kind)

    def to_text(self) -> str:
        out = []
        for l in self.layers:
            if l.kind == "conv":
                c = l.conv
                out.append(f"conv {c.k_n} {c.k_h} {c.k_w} {c.c_i} {c.h_i} {c.w_i} {c.s} {c.p}")
            elif l.kind == "fc":
                out.append(f"fc {l.fc_m} {l.fc_k}")
            else:
                out.append(f"pool {l.pool_h} {l.pool_w} {l.pool_c}")
        return "\n".join(out) + "\n"


@dataclass
class LayerResult:
    layer: int  # 1-based position in the model file
    kind: str
    m: int
    n: int
    k: int
    time_s: float
    repetitions: int
    gflops: float
    workspace_bytes: int


def _fields(parts, names, line_no):
    vals = []
    for i, nm in enumerate(names):
        if i >= len(parts):
            raise ParseError(line_no, f"missing or malformed {nm}")
        try:
            vals.append(int(parts[i]))
        except ValueError:
            raise ParseError(line_no, f"missing or malformed {nm}") from None
    if len(parts) > len(names):
        raise ParseError(line_no, f"trailing token '{parts[len(names)]}'")
    return vals


def parse_model(src, name: str | None = None) -> ModelSpec:
    """Parse a model file (a path) or model text (a string containing a newline or a
    file-like object). model.cpp:35-95."""
    from . import ConvParams, InvalidGeometry, output_dims
    if hasattr(src, "read"):
        text, nm = src.read(), name or "model"
    elif isinstance(src, str) and "\n" not in src and os.path.exists(src):
        with open(src) as f:
            text = f.read()
        nm = name or os.path.splitext(os.path.basename(src))[0]
    elif isinstance(src, str) and "\n" not in src:
        from . import IoError
        raise IoError(f"cannot open model file '{src}'")
    else:
        text, nm = src, name or "model"
    model = ModelSpec(nm)
    line_no = 0
    for line_no, raw in enumerate(io.StringIO(text), start=1):
        line = raw.split("#", 1)[0]
        parts = line.split()
        if not parts:
            continue
        kind, rest = parts[0], parts[1:]
        if kind == "conv":
            k_n, k_h, k_w, c_i, h_i, w_i, s, p = _fields(rest, ("k_n", "k_h", "k_w", "c_i", "h_i", "w_i", "s", "p"),
                                                         line_no)
            cp = ConvParams(k_n, k_h, k_w, c_i, h_i, w_i, 1, s, p)
            try:
                output_dims(cp)
            except InvalidGeometry as e:
                raise ParseError(line_no, str(e)) from None
            model.layers.append(LayerSpec("conv", conv=cp))
        elif kind == "fc":
            m, k = _fields(rest, ("m", "k"), line_no)
            if m < 1 or k < 1:
                raise ParseError(line_no, "fc dimensions must be positive")
            model.layers.append(LayerSpec("fc", fc_m=m, fc_k=k))
        elif kind == "pool":
            h, w, c = _fields(rest, ("h_o", "w_o", "c"), line_no)
            if h < 1 or w < 1 or c < 1:
                raise ParseError(line_no, "pool dimensions must be positive")
            model.layers.append(LayerSpec("pool", pool_h=h, pool_w=w, pool_c=c))
        else:
            raise UnknownLayerKind(line_no, kind)
    if model.count("conv") == 0:
        raise ParseError(line_no, "model contains no conv layer")
    return model


def _with_batch(cp, b):
    from . import ConvParams
    return ConvParams(cp.k_n, cp.k_h, cp.k_w, cp.c_i, cp.h_i, cp.w_i, b, cp.s, cp.p)


def model_workspace_bytes(model: ModelSpec, batch: int) -> int:
    """Largest explicit im2col workspace over the conv layers at batch size b (model.cpp:99-110)."""
    from . import InvalidGeometry, im2col_workspace_bytes
    if batch < 1:
        raise InvalidGeometry("batch must be positive")
    return max((im2col_workspace_bytes(_with_batch(l.conv, batch)) for l in model.layers if l.kind == "conv"),
               default=0)


_ALGOS = ("direct", "im2col", "convgemm", "gemm-only", "im2col-only")


def _shapes(layer, batch):
    """(in, out, weight) element counts, bench.cpp:38-54."""
    from . import output_dims
    if layer.kind == "conv":
        cp = _with_batch(layer.conv, batch)
        h_o, w_o = output_dims(cp)
        return (cp.h_i * cp.w_i * cp.c_i * batch, cp.k_n * h_o * w_o * batch, cp.k_n * cp.k_h * cp.k_w * cp.c_i)
    if layer.kind == "fc":
        return layer.fc_k * batch, layer.fc_m * batch, layer.fc_m * layer.fc_k
    return 0, 0, 0


def _view4(buf, d0, d1, d2, d3):
    """Leftmost-fastest rank-4 view of the first d0*d1*d2*d3 floats of a flat buffer."""
    return buf[: d0 * d1 * d2 * d3].view(d3, d2, d1, d0).permute(3, 2, 1, 0)


def _view2(buf, rows, cols):
    """Column-major rows x cols view of a flat buffer."""
    return buf[: rows * cols].view(cols, rows).t()


def run_inference(model: ModelSpec, batch: int, algo: str = "convgemm", threads: int = 1, min_time: float = 0.05,
                  check: bool = False, blocking=None, precision: str = "auto", seed: int = 20177,
                  device: str = "cuda") -> list:
    """One inference sweep of ``model`` at batch size ``batch`` on the device
    (bench.cpp:93-244). ``threads`` is accepted for API parity (the reference's team
    size); the device tiling is internal."""
    import torch

    from . import (InvalidGeometry, _validate_blocking, conv, conv_workspace_bytes, gemm, gemm_dims, gemm_workspace_bytes, im2col,
                   output_dims)
    if batch < 1:
        raise InvalidGeometry("batch must be positive")
    if algo not in _ALGOS:
        raise ValueError(f"unknown algo '{algo}'")
    _validate_blocking(blocking)
    act = max([1] + [max(_shapes(l, batch)[:2]) for l in model.layers])
    wts = max([1] + [_shapes(l, batch)[2] for l in model.layers])
    g = torch.Generator(device=device).manual_seed(seed)
    act_a = torch.rand(act, generator=g, device=device) * 2 - 1
    act_b = torch.rand(act, generator=g, device=device) * 2 - 1
    weights = torch.empty(wts, device=device)
    st = torch.cuda.current_stream()
    src, dst = act_a, act_b
    results = []
    for li, layer in enumerate(model.layers, start=1):
        if layer.kind == "pool" or (layer.kind == "fc" and algo == "im2col-only"):
            continue
        n_in, n_out, n_w = _shapes(layer, batch)
        weights[:n_w].uniform_(-1, 1, generator=g)
        wrote = True
        if layer.kind == "fc":
            m, n, k = layer.fc_m, batch, layer.fc_k
            W, X, Y = _view2(weights, m, k), _view2(src, k, n), _view2(dst, m, n)
            prec = precision  # fc layers are gemm under every algo (bench.cpp:140-153)
            op = lambda W=W, X=X, Y=Y, prec=prec: gemm(W, X, precision=prec, out=Y)  # noqa: E731
            ws = gemm_workspace_bytes(m, n, k, prec)
        else:
            cp = _with_batch(layer.conv, batch)
            h_o, w_o = output_dims(cp)
            m, n, k = gemm_dims(cp)
            F = _view4(weights, cp.k_n, cp.k_h, cp.k_w, cp.c_i)
            I = _view4(src, cp.h_i, cp.w_i, cp.c_i, batch)
            O = _view4(dst, cp.k_n, h_o, w_o, batch)
            if algo == "convgemm":
                op = lambda F=F, I=I, O=O, cp=cp: conv(F, I, cp, "fused", precision, out=O)  # noqa: E731
                ws = conv_workspace_bytes(cp, "fused", precision)
            elif algo == "direct":
                op = lambda F=F, I=I, O=O, cp=cp: conv(F, I, cp, "direct", out=O)  # noqa: E731
                ws = 0
            elif algo == "im2col":
                op = lambda F=F, I=I, O=O, cp=cp: conv(F, I, cp, "explicit", precision, out=O)  # noqa: E731
                ws = conv_workspace_bytes(cp, "explicit", precision)
            elif algo == "gemm-only":
                Bhat = im2col(I, cp)  # lowered once, outside the timed op (bench.cpp:176-186)
                Fm = _view2(weights, m, k)
                Om = _view2(dst, m, n)
                op = lambda Fm=Fm, Bhat=Bhat, Om=Om: gemm(Fm, Bhat, precision=precision, out=Om)  # noqa: E731
                ws = k * n * 4
            else:  # im2col-only
                op = lambda I=I, cp=cp: im2col(I, cp)  # noqa: E731
                ws = k * n * 4
                wrote = False
        flops = 0.0 if algo == "im2col-only" else 2.0 * m * n * k
        # repeat-until-min_time on the device clock (at least one repetition)
        op()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        op()
        e1.record(st)
        torch.cuda.synchronize()
        t1 = max(e0.elapsed_time(e1) * 1e-3, 1e-7)
        reps = max(1, math.ceil(min_time / t1))
        e0.record(st)
        for _ in range(reps):
            op()
        e1.record(st)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / reps
        if check and layer.kind == "conv" and wrote and algo != "direct":
            ref = torch.empty_like(O)
            conv(F, I, cp, "direct", out=ref)  # the reference's checker, bit-identical
            err, tol = _per_output_error(conv, F, I, O, ref, cp), (5e-3 if precision == "tf32" else 1e-5)
            if err > tol:
                raise RuntimeError(f"check failed at layer {li}: error {err:g}")
        results.append(LayerResult(li, layer.kind, m, n, k, t, reps, flops / t / 1e9 if flops else 0.0, ws))
        if wrote:
            src, dst = dst, src
    return results


def _per_output_error(conv, F, I, O, ref, cp):
    """max over outputs of |O - O_ref| / (||F[i_k]|| * ||B-hat[:, col]||): the north
    star's per-output normalisation. The column norms of the lowered matrix come from one
    more convolution: ones-filters over I*I."""
    import torch

    from . import ConvParams
    fn = F.pow(2).sum(dim=(1, 2, 3)).sqrt()  # (k_n,)
    c4 = ConvParams(4, cp.k_h, cp.k_w, cp.c_i, cp.h_i, cp.w_i, cp.b, cp.s, cp.p)
    ones = torch.ones((cp.c_i, cp.k_w, cp.k_h, 4), device=F.device).permute(3, 2, 1, 0)
    sq = (I * I).permute(3, 2, 1, 0).contiguous().permute(3, 2, 1, 0)
    bn = conv(ones, sq, c4, "fused", "ffma")[0].clamp_min(0).sqrt()  # (h_o, w_o, b)
    scale = (fn.view(-1, 1, 1, 1) * bn.unsqueeze(0)).clamp_min(1e-30)
    return float(((O - ref).abs() / scale).max())


def write_csv(out, model: ModelSpec, batch: int, algo: str, threads: int, results: list, header: bool = True):
    """The reference's CSV (bench.cpp:246-275): one row per layer plus a ``total`` row.
    ``out``: a path or a writable text stream."""
    if isinstance(out, (str, os.PathLike)):
        with open(out, "w") as f:
            return write_csv(f, model, batch, algo, threads, results, header)
    if header:
        out.write("model,batch,algo,threads,layer,m,n,k,time_s,gflops,workspace_bytes\n")
    tot_t = tot_f = 0.0
    worst = 0
    for r in results:
        out.write(f"{model.name},{batch},{algo},{threads},{r.layer},{r.m},{r.n},{r.k},{r.time_s:.9g},"
                  f"{r.gflops:.6g},{r.workspace_bytes}\n")
        tot_t += r.time_s
        tot_f += r.gflops * r.time_s * 1e9
        worst = max(worst, r.workspace_bytes)
    tot_g = tot_f / tot_t / 1e9 if tot_t > 0 else 0.0
    out.write(f"{model.name},{batch},{algo},{threads},total,0,0,0,{tot_t:.9g},{tot_g:.6g},{worst}\n")
