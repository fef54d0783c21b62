#!/usr/bin/env python
"""Per-layer throughput of the fused operator on ALL five BASELINE.json configs.

bench.py times configs[1] (the ResNet-50 3x3 step) under the driver's contract; this
tool covers the rest the same way, one layer at a time: seeded synthetic tensors with the
BASELINE shapes and distributions (uniform[-1,1]; the stem: I uniform[0,1], F N(0,0.05^2)),
CUDA events around each launch on the launching stream, a 256 MiB L2 flush before every
timed launch (outside the events), median of `--reps`. Reports GFLOPS, HBM GB/s of the
compulsory bytes 4*(|I|+|F|+|O|), the bound (tensor or HBM, max of FLOPs/P_TF32 and
bytes/BW_HBM) and the roofline fraction, per precision mode.

  python tools/bench_configs.py [--configs C1,C2,C3,C4,C5] [--precisions tf32,3xtf32] [--out FILE]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _prof  # noqa: E402,F401  (profiling build: CGB_* env knobs)
import paper_2005_06410_b200 as cg  # noqa: E402


def L(name, k_n, k, c_i, h_i, s, p, b, dist="uniform"):
    return dict(name=name, cp=dict(k_n=k_n, k_h=k, k_w=k, c_i=c_i, h_i=h_i, w_i=h_i, b=b, s=s, p=p), dist=dist)


CONFIGS = {
    "C1": [L("c1_3x3_56_64_b8", 64, 3, 64, 56, 1, 1, 8)],
    "C2": [L(n, k_n, k, c_i, h_i, s, p, 128) for (n, k_n, k, c_i, h_i, s, p) in bench.LAYERS],
    "C3": [L("c3_1x1_56_64_256", 256, 1, 64, 56, 1, 0, 256), L("c3_1x1_14_1024_256", 256, 1, 1024, 14, 1, 0, 256),
           L("c3_1x1_7_2048_512", 512, 1, 2048, 7, 1, 0, 256), L("c3_1x1_7_512_2048", 2048, 1, 512, 7, 1, 0, 256)],
    "C4": [L("c4_stem_7x7_s2_224_3_64", 64, 7, 3, 224, 2, 3, 256, dist="stem")],
    "C5": [L(f"c5_vgg{i + 1:02d}_{h}_{ci}_{kn}", kn, 3, ci, h, 1, 1, 64) for i, (h, ci, kn) in enumerate([
        (224, 3, 64), (224, 64, 64), (112, 64, 128), (112, 128, 128), (56, 128, 256), (56, 256, 256), (56, 256, 256),
        (28, 256, 512), (28, 512, 512), (28, 512, 512), (14, 512, 512), (14, 512, 512), (14, 512, 512)])],
}


def tensors(layer, seed=20177):
    cp = layer["cp"]
    h_o, w_o = bench.out_hw(cp)
    g = torch.Generator(device="cuda").manual_seed(seed)
    F = cg.empty_tensor4(cp["k_n"], cp["k_h"], cp["k_w"], cp["c_i"])
    I = cg.empty_tensor4(cp["h_i"], cp["w_i"], cp["c_i"], cp["b"])
    if layer["dist"] == "stem":
        F.copy_(torch.randn(F.shape, generator=g, device="cuda") * 0.05)
        I.copy_(torch.rand(I.shape, generator=g, device="cuda"))
    else:
        F.copy_(torch.rand(F.shape, generator=g, device="cuda") * 2 - 1)
        I.copy_(torch.rand(I.shape, generator=g, device="cuda") * 2 - 1)
    O = cg.empty_tensor4(cp["k_n"], h_o, w_o, cp["b"])
    return F, I, O


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--precisions", default="tf32,3xtf32")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--tune", default="{}", help="JSON of cgb_set_tuning knobs")
    a = ap.parse_args()
    for k, v in json.loads(a.tune).items():
        cg.set_tuning(k, v)
    pk = bench.peaks()
    P = pk["tf32_tflops"] * 1e12
    BW = pk["hbm_gbs"] * 1e9
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    rows = []
    for cname in a.configs.split(","):
        for layer in CONFIGS[cname]:
            cp = layer["cp"]
            F, I, O = tensors(layer)
            fl, by = bench.flops(cp), bench.nbytes(cp)
            for prec in a.precisions.split(","):
                peak = P / 3 if prec == "3xtf32" else P
                for _ in range(2):
                    cg.conv(F, I, cp, algo="fused", precision=prec, out=O)
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    cg.conv(F, I, cp, algo="fused", precision=prec, out=O)
                    e1.record(st)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e-3)
                t = statistics.median(ts)
                t_tc, t_hbm = fl / peak, by / BW
                r = dict(config=cname, layer=layer["name"], precision=prec, path=cg.last_path(), us=round(t * 1e6, 1),
                         gflops=round(fl / t / 1e9, 1), hbm_gbs=round(by / t / 1e9, 1),
                         bound="tensor" if t_tc >= t_hbm else "hbm", roofline_frac=round(max(t_tc, t_hbm) / t, 4),
                         tf32_frac=round(t_tc / t, 4), geometry=cp)
                rows.append(r)
                print(json.dumps(r), flush=True)
            del F, I, O
            torch.cuda.empty_cache()
    summ = {}
    for cname in a.configs.split(","):
        for prec in a.precisions.split(","):
            sel = [r for r in rows if r["config"] == cname and r["precision"] == prec]
            if sel:
                tot_f = sum(bench.flops(r["geometry"]) for r in sel)
                tot_t = sum(r["us"] for r in sel) * 1e-6
                summ[f"{cname}/{prec}"] = dict(layers=len(sel), gflops=round(tot_f / tot_t / 1e9, 1),
                                               us=round(tot_t * 1e6, 1))
    print(json.dumps({"summary": summ, "peaks": {"tf32_tflops": pk["tf32_tflops"], "hbm_gbs": pk["hbm_gbs"]}}))
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"rows": rows, "summary": summ, "peaks": pk,
                       "method": "eager launch per layer, CUDA events, L2 flushed before each timed launch, "
                                 f"median of {a.reps}"}, f, indent=1)


if __name__ == "__main__":
    main()
