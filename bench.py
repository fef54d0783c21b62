#!/usr/bin/env python
"""bench.py -- throughput of the B200 convolution operator on BASELINE.json configs[1].

Workload (one "step"): the seven ResNet-50 v1.5 3x3 convolutions of BASELINE.json
configs[1] at b=128 per GPU -- 56^2 64->64, 28^2 128->128, 14^2 256->256, 7^2 512->512
(stride 1, pad 1) and the stride-2 variants 56->28 c128, 28->14 c256, 14->7 c512 --
each run once through the fused operator (cgb_conv, CGB_ALGO_FUSED), FP32 tensors in
the reference layouts, synthetic uniform[-1,1] inputs from a fixed seed.

metric/unit: BASELINE.json's "conv GFLOPS (2*k_n*h_o*w_o*b*k_h*k_w*c_i/s)"; value =
whole-job FLOPs / max-over-ranks device time. The headline precision is TF32 (the mode
the north-star roofline target is stated in, tolerance 5e-3); the fp32-accurate 3xTF32
mode is measured in the same run and reported under "modes".

Launch: python bench.py [--gpus N --steps K --warmup W] (N>1 under torchrun, one rank
per GPU, batch sharded with no collective in the timed region; filters broadcast once).
--impl reference times the reference's own CPU conv_gemm (oracle/_ref) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _load_configs():
    # by file path: importing the package would load libconvgemm_b200.so into the
    # reference arm's process, which must run the reference alone
    import importlib.util
    spec = importlib.util.spec_from_file_location("cgb_configs", os.path.join(ROOT, "paper_2005_06410_b200", "configs.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


CONFIGS = _load_configs()
layer_seed = CONFIGS.layer_seed

METRIC = "conv GFLOPS (2·k_n·h_o·w_o·b·k_h·k_w·c_i/s) per layer & % TF32 TC roofline"
UNIT = "GFLOPS"
BATCH = 128

# (name, k_n, k, c_i, h_i, s, p)  -- BASELINE.json configs[1]
LAYERS = [
    ("r50_3x3_56_64", 64, 3, 64, 56, 1, 1),
    ("r50_3x3_28_128", 128, 3, 128, 28, 1, 1),
    ("r50_3x3_14_256", 256, 3, 256, 14, 1, 1),
    ("r50_3x3_7_512", 512, 3, 512, 7, 1, 1),
    ("r50_3x3_s2_56_128", 128, 3, 128, 56, 2, 1),
    ("r50_3x3_s2_28_256", 256, 3, 256, 28, 2, 1),
    ("r50_3x3_s2_14_512", 512, 3, 512, 14, 2, 1),
]


def layer_cp(layer, b):
    name, k_n, k, c_i, h_i, s, p = layer
    return dict(k_n=k_n, k_h=k, k_w=k, c_i=c_i, h_i=h_i, w_i=h_i, b=b, s=s, p=p)


def out_hw(cp):
    return (cp["h_i"] - cp["k_h"] + 2 * cp["p"]) // cp["s"] + 1, (cp["w_i"] - cp["k_w"] + 2 * cp["p"]) // cp["s"] + 1


def flops(cp):
    h_o, w_o = out_hw(cp)
    return 2 * cp["k_n"] * h_o * w_o * cp["b"] * cp["k_h"] * cp["k_w"] * cp["c_i"]


def nbytes(cp):
    h_o, w_o = out_hw(cp)
    return 4 * (cp["h_i"] * cp["w_i"] * cp["c_i"] * cp["b"] + cp["k_n"] * cp["k_h"] * cp["k_w"] * cp["c_i"]
                + cp["k_n"] * h_o * w_o * cp["b"])


def split_range(count, rank, nranks):
    """threads.hpp:20-25: contiguous static split, first count % nranks ranks get +1."""
    base, rem = divmod(count, nranks)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written on this pool). The
    TF32 tensor peak is bf16_tflops/2 (dense TF32 runs at half the bf16 rate on tcgen05;
    the burst figure, since each kernel is timed in a short burst); the HBM peak is
    hbm_gbs. The cuBLAS TF32 measurement (profiles/tf32_peak.json) is context only --
    our kernels exceed it, so it is not a peak."""
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p = {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m["bf16_tflops"]), "src": "MEASURED_PEAKS.json",
             "bf16_sustained": float(m.get("bf16_tflops_sustained") or 0) or None}
    except Exception:  # noqa: BLE001
        pass
    p["tf32_tflops"] = p["bf16_tflops"] / 2.0
    p["tf32_src"] = f"bf16_tflops/2 of {p['src']} (burst; dense TF32 = half the dense bf16 rate on tcgen05)"
    try:
        with open(os.path.join(ROOT, "profiles", "tf32_peak.json")) as f:
            p["cublas_tf32"] = float(json.load(f)["tf32_tflops"])
    except Exception:  # noqa: BLE001
        p["cublas_tf32"] = None
    return p


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled every
    2 ms on a thread (nvidia-smi -lms 100 as a fallback)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.stop_evt = threading.Event()
        self.t = None
        self.proc = None
        self.lines = []
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nvml = None

    def _poll(self):
        nv = self.nvml
        while not self.stop_evt.is_set():
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.nvml:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        try:
            fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                      "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=lambda: self.lines.extend(l.strip() for l in self.proc.stdout),
                                      daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def stop(self):
        if self.nvml:
            self.stop_evt.set()
            self.t.join(timeout=1)
            src = "nvml 2 ms"
        elif self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for ln in self.lines:
                parts = [x.strip() for x in ln.split(",")]
                try:
                    self.samples.append(float(parts[0]))
                    self.max_mhz = float(parts[1])
                except (ValueError, IndexError):
                    continue
                for nm, v in zip(names, parts[2:6]):
                    if v.lower() == "active":
                        self.reasons.add(nm)
            src = "nvidia-smi 100 ms"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": src}


# ----------------------------------------------------------------------------- distributed
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- CPU reference
def _ref_runner(threads):
    """The reference's own conv_gemm<float> (oracle/_ref, compiled from /root/reference);
    the plain-C port (oracle/) only where the reference build is absent."""
    from oracle.oracle import Reference, Restatement
    try:
        ref = Reference()
        return (lambda F, I, cp: ref.conv_gemm(F, I, cp, threads=threads)), "reference"
    except Exception:  # noqa: BLE001
        orc = Restatement()
        return (lambda F, I, cp: orc.conv_gemm(F, I, cp)), "port"


def host_tensors(layers, b, seed=20177):
    """Seeded host tensors (Fortran order, the reference layouts) for the CPU arms."""
    import numpy as np
    out = []
    for layer in layers:
        cp = layer_cp(layer, b)
        rng = np.random.default_rng(layer_seed(layer[0], seed))
        F = np.asfortranarray(rng.uniform(-1, 1, (cp["k_n"], 3, 3, cp["c_i"])).astype(np.float32))
        I = np.asfortranarray(rng.uniform(-1, 1, (cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])).astype(np.float32))
        out.append((layer, cp, F, I))
    return out


def run_reference_arm(args, world, rank):
    """The reference arm: the reference's CPU conv_gemm on the box's host cores, same
    metric/config as the GPU arm. Each step is the 7 layers at the full b=128 (the real
    config; ~4 s per step at ~50 GFLOPS on 16 cores) unless --ref-batch asks for a sample."""
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    run, kind = _ref_runner(threads)
    sample_b = args.ref_batch or BATCH
    data = host_tensors(LAYERS, sample_b)
    warm = host_tensors(LAYERS, 1)
    for _ in range(args.warmup):  # warm-up steps on one image (page-in, thread team)
        for layer, cp, F, I in warm:
            run(F, I, cp)
    step_t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for layer, cp, F, I in data:
            run(F, I, cp)
        step_t.append(time.perf_counter() - t0)
    step_flops = sum(flops(cp) for _, cp, _, _ in data)
    value = step_flops / statistics.mean(step_t) / 1e9
    # supplementary (SURVEY 8(d) times both CPU operators): the reference's explicit
    # conv_im2col_gemm<float>, one pass over the 7 layers at a b=8 sample
    explicit = None
    if kind == "reference" and not args.quick:
        from oracle.oracle import Reference
        ref = Reference()
        small = host_tensors(LAYERS, min(8, sample_b))
        t0 = time.perf_counter()
        for layer, cp, F, I in small:
            ref.conv_im2col_gemm(F, I, cp, threads=threads)
        dt = time.perf_counter() - t0
        explicit = {"value": sum(flops(cp) for _, cp, _, _ in small) / dt / 1e9, "unit": UNIT,
                    "algo": "conv_im2col_gemm (reference explicit im2col + gemm)",
                    "sample": f"one pass over the 7 layers at b={min(8, sample_b)}, threads={threads}"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(step_t),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (uniform[-1,1], seeded numpy)",
        "config": {"workload": "ResNet-50 v1.5 3x3 convs at b=128 (BASELINE configs[1])", "global_batch": BATCH,
                   "batch_per_step": sample_b, "same_config": sample_b == BATCH,
                   "layers": [l[0] for l in LAYERS], "algo": "conv_gemm (reference fused ConvGemm)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"each step = the 7 layers at b={sample_b} (of {BATCH}), "
                                   f"{step_flops / 1e9:.1f} GFLOP, conv_gemm<float> threads={threads}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "explicit": explicit,
    }
    print(json.dumps(line), flush=True)
    return 0


def host_image_batch(t, b0, b1):
    """Images [b0, b1) of a leftmost-fastest CUDA tensor as a Fortran numpy array."""
    import numpy as np
    x = t[..., b0:b1]
    flat = x.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy()
    return np.asfortranarray(flat.reshape(tuple(x.shape), order="F"))


def cpu_baseline_leg(tensors, nimg, min_time, threads):
    """cpu_baseline: the reference's conv_gemm on the first `nimg` images of the SAME
    inputs the GPU ran, repeat-until-min_time per layer (bench.cpp:200-210); its outputs
    double as a parity check of the GPU outputs of those images (returned per layer)."""
    from oracle.oracle import Restatement, per_output_error
    run, kind = _ref_runner(threads)
    orc = Restatement()
    total_flops, total_t, parity = 0, 0.0, {}
    for layer, cp, F, I, O in tensors:
        cpn = dict(cp, b=nimg)
        Fh = host_image_batch(F, 0, F.shape[3])
        Ih, Oh = host_image_batch(I, 0, nimg), host_image_batch(O, 0, nimg)
        reps, t0 = 0, time.perf_counter()
        while True:
            ref = run(Fh, Ih, cpn)
            reps += 1
            el = time.perf_counter() - t0
            if el >= min_time:
                break
        total_flops += flops(cpn) * reps
        total_t += el
        parity[layer[0]] = per_output_error(Oh, ref, orc.output_scale(Fh, Ih, cpn))
    return total_flops / total_t / 1e9, kind, total_t, parity


# ----------------------------------------------------------------------------- GPU arm
def make_layer_tensors(cg, torch, layers, b, rank, world, seed=20177):
    out = []
    for layer in layers:
        cp = layer_cp(layer, b)
        h_o, w_o = out_hw(cp)
        F = cg.empty_tensor4(cp["k_n"], 3, 3, cp["c_i"])
        gf = torch.Generator(device="cuda").manual_seed(layer_seed(layer[0], seed))  # stable (crc32) per layer
        F.copy_(torch.rand(F.shape, generator=gf, device="cuda") * 2 - 1)
        if world > 1:
            from paper_2005_06410_b200.shard import broadcast_filters
            broadcast_filters(F, src=0)  # filters broadcast once, outside the timed region
        gi = torch.Generator(device="cuda").manual_seed(layer_seed(layer[0], seed + 1 + rank))
        I = cg.empty_tensor4(cp["h_i"], cp["w_i"], cp["c_i"], b)
        I.copy_(torch.rand(I.shape, generator=gi, device="cuda") * 2 - 1)
        O = cg.empty_tensor4(cp["k_n"], h_o, w_o, b)
        out.append((layer, cp, F, I, O))
    return out


L2_NOTE = {
    "flush": "256 MiB L2 flush between timed steps (outside the CUDA events); per-step traffic > L2",
    "cycle": "no flush: inputs larger than L2 - the 7 layers' inputs (577 MB, 4.6x the 126 MB L2) are "
             "read in turn, so every layer's input was evicted by the other six since its last use",
}
TOL = {"tf32": 5e-3, "3xtf32": 1e-5, "auto": 1e-5}


def time_mode(cg, torch, tensors, precision, steps, warmup, flush, world, clocks=None):
    """Per-layer breakdown from an eager pass (CUDA events around each launch), then
    the step time from CUDA-graph replays of the 7 launches (host submission out of
    the device timeline; consecutive kernels overlap setup via programmatic dependent
    launch). L2 is flushed before every timed step, outside the events."""
    st = torch.cuda.current_stream()
    nl = len(tensors)

    def step():
        for layer, cp, F, I, O in tensors:
            cg.conv(F, I, cp, algo="fused", precision=precision, out=O)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    # eager per-layer pass
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nl)]
          for _ in range(steps)]
    for s in range(steps):
        if flush is not None:
            flush.zero_()
        for li, (layer, cp, F, I, O) in enumerate(tensors):
            ev[s][li][0].record(st)
            cg.conv(F, I, cp, algo="fused", precision=precision, out=O)
            ev[s][li][1].record(st)
    torch.cuda.synchronize()
    per_layer = [[ev[s][li][0].elapsed_time(ev[s][li][1]) for s in range(steps)] for li in range(nl)]
    # graph of one step
    side = torch.cuda.Stream()
    side.wait_stream(st)
    with torch.cuda.stream(side):
        step()
    st.wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    l0 = cg.kernel_launch_count()
    with torch.cuda.graph(g):
        step()
    launches_per_step = cg.kernel_launch_count() - l0
    for _ in range(warmup):
        g.replay()
    torch.cuda.synchronize()
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier(world)
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    for s in range(steps):
        if flush is not None:
            flush.zero_()  # L2 flush (256 MiB write) between timed steps, outside the events
        sev[s][0].record(st)
        g.replay()
        sev[s][1].record(st)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    barrier(world)
    step_ms = [a.elapsed_time(b) for a, b in sev]
    del g
    return per_layer, step_ms, launches_per_step * steps, clk


def time_concurrent(cg, torch, tensors, precision, steps, warmup, flush, world, nstreams):
    """Supplementary: the same 7 launches, but captured on `nstreams` forked streams
    (layer i on stream i mod nstreams, joined at the end of the step) -- the layers of
    this benchmark are independent operators, so a caller may issue them concurrently and
    the drain of one grid overlaps the ramp of the next. Same inputs, same launches, same
    L2 flush and event placement as the single-stream step; never the headline value."""
    st = torch.cuda.current_stream()
    side = [torch.cuda.Stream() for _ in range(nstreams)]

    def step():
        cur = torch.cuda.current_stream()
        for s in side:
            s.wait_stream(cur)
        for li, (layer, cp, F, I, O) in enumerate(tensors):
            with torch.cuda.stream(side[li % nstreams]):
                cg.conv(F, I, cp, algo="fused", precision=precision, out=O)
        for s in side:
            cur.wait_stream(s)

    warm = torch.cuda.Stream()
    warm.wait_stream(st)
    with torch.cuda.stream(warm):
        step()
    st.wait_stream(warm)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(warmup):
        g.replay()
    torch.cuda.synchronize()
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier(world)
    torch.cuda.synchronize()
    for s in range(steps):
        if flush is not None:
            flush.zero_()
        sev[s][0].record(st)
        g.replay()
        sev[s][1].record(st)
    torch.cuda.synchronize()
    barrier(world)
    ms = [a.elapsed_time(b) for a, b in sev]
    del g
    return ms


def time_e2e(cg, torch, tensors, precision, steps, warmup, world):
    """Public host-buffer API (cgb_conv_host via cg.conv on numpy arrays backed by
    pinned memory): H2D of F and I, the kernel, D2H of O, every step."""
    host = []
    h2d = d2h = 0
    for layer, cp, F, I, O in tensors:
        hF = torch.empty(F.numel(), dtype=torch.float32, pin_memory=True)
        hI = torch.empty(I.numel(), dtype=torch.float32, pin_memory=True)
        hO = torch.empty(O.numel(), dtype=torch.float32, pin_memory=True)
        hF.copy_(F.permute(3, 2, 1, 0).reshape(-1))
        hI.copy_(I.permute(3, 2, 1, 0).reshape(-1))
        npF = hF.numpy().reshape(F.shape, order="F")
        npI = hI.numpy().reshape(I.shape, order="F")
        npO = hO.numpy().reshape(O.shape, order="F")
        host.append((cp, npF, npI, npO, (hF, hI, hO)))
        h2d += 4 * (F.numel() + I.numel())
        d2h += 4 * O.numel()
    for _ in range(warmup):
        for cp, npF, npI, npO, _k in host:
            cg.conv(npF, npI, cp, algo="fused", precision=precision, out=npO)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    legacy = torch.cuda.default_stream()
    e0.record(legacy)
    for _ in range(steps):
        for cp, npF, npI, npO, _k in host:
            cg.conv(npF, npI, cp, algo="fused", precision=precision, out=npO)
    e1.record(legacy)
    torch.cuda.synchronize()
    barrier(world)
    return e0.elapsed_time(e1) / steps, h2d, d2h


def parity_fp64(torch, tensors):
    """Per layer: max north-star per-output error of the outputs just timed against an
    fp64 recomputation of EVERY output (tests/fp64ref.py; after the timed region)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from fp64ref import per_output_error_fp64
    return {layer[0]: per_output_error_fp64(torch, F, I, O, cp) for layer, cp, F, I, O in tensors}


def run_gpu_arm(args, world, rank, local):
    import torch

    import paper_2005_06410_b200 as cg
    torch.cuda.set_device(local)
    if args.tune:
        for k, v in json.loads(args.tune).items():
            cg.set_tuning(k, v)
    pk = peaks()
    from paper_2005_06410_b200.shard import split_range as shard_split
    b = BATCH  # weak scaling: b=128 per GPU (each rank an independent batch shard)
    if args.scaling == "strong":
        lo, hi = shard_split(BATCH, rank, world)  # threads.hpp:20-25 split of the global batch
        b = hi - lo
    if args.shard_of > 1:
        # analysis aid on a one-GPU box: time the shard rank 0 of an N-way strong-scaling run
        # would get (e.g. b=16 of 128 for N=8); the line is marked and is not a contract line
        assert world == 1, "--shard-of is a single-process measurement"
        lo, hi = shard_split(BATCH, 0, args.shard_of)
        b = hi - lo
    tensors = make_layer_tensors(cg, torch, LAYERS, b, rank, world)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.l2 == "flush" else None
    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    step_flops_local = sum(flops(cp) for _, cp, _, _, _ in tensors)
    total_flops = step_flops_local * world if args.scaling == "weak" else sum(flops(layer_cp(l, BATCH)) for l in LAYERS)
    if args.shard_of > 1:
        total_flops = step_flops_local

    modes = {}
    parity = {}
    cpu = None
    headline = args.precision
    order = [headline] + [m for m in ("3xtf32",) if m != headline and not args.quick]
    for prec in order:
        per_layer, step_ms, launches, c = time_mode(cg, torch, tensors, prec, args.steps, args.warmup, flush, world,
                                                    clocks if prec == headline else None)
        if prec == headline:
            clk = c
        ms_step = max_over_ranks(statistics.mean(step_ms), world)
        layers = []
        for li, (layer, cp, F, I, O) in enumerate(tensors):
            t = statistics.mean(per_layer[li]) * 1e-3
            fl, by = flops(cp), nbytes(cp)
            t_tc = fl / (pk["tf32_tflops"] * 1e12)
            t_hbm = by / (pk["hbm_gbs"] * 1e9)
            layers.append({"layer": layer[0], "ms": round(t * 1e3, 4), "gflops": round(fl / t / 1e9, 1),
                           "tflops": round(fl / t / 1e12, 1), "hbm_gbs": round(by / t / 1e9, 1),
                           "bound": "tensor" if t_tc >= t_hbm else "hbm",
                           "roofline_frac": round(max(t_tc, t_hbm) / t, 4)})
        modes[prec] = {"value": total_flops / (ms_step * 1e-3) / 1e9, "ms_per_step": ms_step,
                       "layers": layers, "gpu_launches": launches,
                       "achieved_tflops": step_flops_local / (ms_step * 1e-3) / 1e12}
        # parity of the outputs just timed (outside the timed region)
        if not args.no_parity:
            errs = parity_fp64(torch, tensors)
            parity[prec] = {"check": "fp64 recomputation of every output of every layer (cuDNN fp64 on the "
                                     "device, tests/fp64ref.py), per-output error normalised by "
                                     "||F[i_k]||*||B[:,col]||",
                            "tolerance": TOL[prec], "max_err": {k: float(f"{v:.3e}") for k, v in errs.items()},
                            "pass": all(v <= TOL[prec] for v in errs.values())}
        if prec == headline and world == 1 and rank == 0 and not args.no_cpu_baseline:
            v, kind, t, ref_err = cpu_baseline_leg(tensors, args.cpu_batch, args.cpu_min_time, os.cpu_count() or 1)
            cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": kind,
                   "sample": f"the 7 layers on images 0..{args.cpu_batch - 1} of the GPU inputs (b={args.cpu_batch} of "
                             f"{BATCH}), conv_gemm<float> repeated until >= {args.cpu_min_time}s per layer "
                             f"({t:.1f}s CPU total), threads=nproc"}
            parity["reference_sample"] = {
                "check": f"the reference's own conv_gemm output (cpu_baseline leg) vs the GPU {headline} output, "
                         f"images 0..{args.cpu_batch - 1} of the full-batch launch",
                "tolerance": TOL[headline], "max_err": {k: float(f"{e:.3e}") for k, e in ref_err.items()},
                "pass": all(e <= TOL[headline] for e in ref_err.values())}
    # supplementary: independent layers issued on forked streams (never the headline)
    concurrent = {}
    for ns in [int(x) for x in args.concurrent.split(",") if x]:
        try:
            ms = time_concurrent(cg, torch, tensors, headline, args.steps, args.warmup, flush, world, ns)
        except Exception as ex:  # noqa: BLE001  (supplementary leg: never takes the contract line down)
            if world > 1:
                raise
            concurrent[str(ns)] = {"streams": ns, "error": f"{type(ex).__name__}: {ex}"[:200]}
            continue
        ms_c = max_over_ranks(statistics.mean(ms), world)
        ach = step_flops_local / (ms_c * 1e-3) / 1e12
        concurrent[str(ns)] = {"streams": ns, "ms_per_step": ms_c, "value": total_flops / (ms_c * 1e-3) / 1e9,
                               "tf32_frac": ach / pk["tf32_tflops"]}
        if not args.no_parity:
            errs = parity_fp64(torch, tensors)
            concurrent[str(ns)]["parity_pass"] = all(v <= TOL[headline] for v in errs.values())
    # e2e through the host-buffer public API, every measured precision
    e2e = {}
    for prec in order:
        e2e_ms, h2d, d2h = time_e2e(cg, torch, tensors, prec, max(1, min(args.steps, 3)), 1, world)
        e2e_ms = max_over_ranks(e2e_ms, world)
        e2e[prec] = {"value": total_flops / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                     "api": "cgb_conv_host (host buffers, pinned)"}
    if rank != 0:
        return 0
    hm = modes[headline]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(headline)
        except Exception:  # noqa: BLE001
            traffic = None
    peak = pk["tf32_tflops"]
    line = {
        "metric": METRIC, "value": hm["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": hm["ms_per_step"], "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "tf32" if headline == "tf32" else "f32",
        "data": "synthetic (uniform[-1,1], seeded torch generator on device)",
        "config": {"workload": "ResNet-50 v1.5 3x3 convs at b=128 (BASELINE configs[1]), fused operator",
                   "global_batch": BATCH * world if args.scaling == "weak" else BATCH, "batch_per_gpu": b,
                   "layers": [l[0] for l in LAYERS], "precision": headline, "algo": "fused",
                   "l2": L2_NOTE[args.l2],
                   "launch": "one CUDA-graph replay of the 7 layer launches per step (programmatic dependent launch "
                             "between kernels); per-layer times from an eager pass",
                   "parallelism": f"batch-sharded dp{world} ({args.scaling} scaling), no collective in the timed "
                                  f"region",
                   **({"shard_of": args.shard_of,
                       "note": f"ANALYSIS LINE, not a contract run: the rank-0 shard (b={b}) of a "
                               f"{args.shard_of}-way strong-scaling split timed alone on one GPU; value = shard "
                               f"FLOPs / shard step time"} if args.shard_of > 1 else {})},
        "roofline": {"bound": "tensor", "achieved": hm["achieved_tflops"], "peak": peak,
                     "unit": "TFLOP/s", "frac": hm["achieved_tflops"] / peak, "traffic": traffic,
                     "peak_src": pk["tf32_src"],
                     "frac_vs_other_peaks": {
                         "MEASURED_PEAKS bf16_tflops_sustained/2 (the back-to-back figure; context only, `peak` is "
                         "the larger burst figure)":
                             hm["achieved_tflops"] / (pk["bf16_sustained"] / 2) if pk.get("bf16_sustained") else None,
                         "cuBLAS TF32 8192^3 burst on this pool (profiles/tf32_peak.json)":
                             hm["achieved_tflops"] / pk["cublas_tf32"] if pk.get("cublas_tf32") else None,
                         "tcgen05 kind::tf32 UMMA microbenchmark 1190 @1965 MHz (tools/umma_bench.cu, pair_bench.cu)":
                             hm["achieved_tflops"] / 1190.0},
                     "per_layer": hm["layers"]},
        "parity": parity,
        "concurrent": {"note": "SUPPLEMENTARY, not the headline: the same 7 launches captured on N forked streams "
                               "(layer i on stream i mod N, joined per step); the benchmark's layers are independent "
                               "operators, so the drain of one grid overlaps the ramp of the next. value/ms_per_step "
                               "above are the single-stream, dependency-safe step.",
                       "streams": concurrent} if concurrent else None,
        "cpu_baseline": cpu,
        "e2e": e2e[headline],
        "gpu_launches": hm["gpu_launches"],
        "clocks": clk,
        "modes": {m: {"value": v["value"], "ms_per_step": v["ms_per_step"],
                      "tf32_frac": v["achieved_tflops"] / peak,
                      # 3xTF32 issues three TF32 MMAs per product: its own roofline is P_TF32/3
                      "frac_of_own_roofline": v["achieved_tflops"] / (peak / (3 if m == "3xtf32" else 1)),
                      "e2e": e2e[m],
                      "per_layer_tflops": {l["layer"]: l["tflops"] for l in v["layers"]}} for m, v in modes.items()},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--concurrent", default="2",
                    help="comma list of stream counts for the supplementary forked-stream step ('' = skip)")
    ap.add_argument("--precision", default="tf32", choices=["tf32", "3xtf32", "auto"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the global b=128 split across ranks (threads.hpp:20-25); "
                         "weak: b=128 per rank")
    ap.add_argument("--quick", action="store_true", help="headline precision only")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l2", choices=sorted(L2_NOTE), default="flush",
                    help="flush: 256 MiB write before every timed step; cycle: no flush, the step's own "
                         "inputs (577 MB) are larger than L2")
    ap.add_argument("--cpu-batch", type=int, default=2)
    ap.add_argument("--cpu-min-time", type=float, default=2.0)
    ap.add_argument("--ref-batch", type=int, default=0, help="reference arm batch per step (0 = the full b=128)")
    ap.add_argument("--no-parity", action="store_true", help="skip the fp64 parity pass after timing")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="analysis: time only the rank-0 shard of an N-way strong-scaling split on this GPU")
    ap.add_argument("--tune", default="", help='dispatch knobs for A/B runs, JSON, e.g. {"tps": 1}')
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            return run_reference_arm(args, world, rank)
        return run_gpu_arm(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
