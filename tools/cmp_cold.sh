#!/bin/bash
# Cold-L2 per-layer time (256 MiB flush before every launch), for an env setting A/B.
python - "$@" <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2005_06410_b200 as cg, bench
tensors = bench.make_layer_tensors(cg, torch, bench.LAYERS, 128, 0, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for layer, cp, F, I, O in tensors:
    cg.conv(F, I, cp, algo="fused", precision="tf32", out=O)
torch.cuda.synchronize()
tot = 0
for layer, cp, F, I, O in tensors:
    ts = []
    for r in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); cg.conv(F, I, cp, algo="fused", precision="tf32", out=O); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2]; tot += t
    print(f"{layer[0]:20s} {t * 1e3:7.1f} us (median, cold L2)")
print(f"sum {tot * 1e3:.1f} us")
PY
