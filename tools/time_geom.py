"""Time one geometry through the fused operator: python tools/time_geom.py k_n k c_i h s p b [precision]
(CUDA events around `reps` back-to-back launches after warm-up; for quick A/B of env knobs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _prof  # noqa: E402,F401  (profiling build: CGB_* env knobs)
import paper_2005_06410_b200 as cg  # noqa: E402

k_n, k, c_i, h, s, p, b = map(int, sys.argv[1:8])
prec = sys.argv[8] if len(sys.argv) > 8 else "tf32"
cp = dict(k_n=k_n, k_h=k, k_w=k, c_i=c_i, h_i=h, w_i=h, b=b, s=s, p=p)
h_o, w_o = cg.output_dims(cp)
F = cg.empty_tensor4(k_n, k, k, c_i).uniform_(-1, 1)
I = cg.empty_tensor4(h, h, c_i, b).uniform_(-1, 1)
O = cg.empty_tensor4(k_n, h_o, w_o, b)
for _ in range(3):
    cg.conv(F, I, cp, "fused", prec, out=O)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    cg.conv(F, I, cp, "fused", prec, out=O)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
fl = 2 * k_n * h_o * w_o * b * k * k * c_i
print(f"{sys.argv[1:8]} {prec} {cg.last_path()} {us:.1f} us {fl / us / 1e6:.1f} TFLOPS")
if int(os.environ.get("CGB_DEBUG_SW", "0")) & 64:
    import numpy as np
    buf = np.zeros((148, 16), dtype=np.uint64)
    cg.lib.cgb_debug_sw_stats(buf.ctypes.data, 148)
    lead = buf[:, 4] > 0  # CTAs whose MMA thread ran
    tot, wt, wa, wb, nt, ew, eb = [buf[:, i].astype(np.float64) for i in range(7)]
    print(f"  MMA thread cycles: total mean {tot[lead].mean():.0f}; wait t_empty {wt[lead].mean():.0f} a_full "
          f"{wa[lead].mean():.0f} b_full {wb[lead].mean():.0f}; segments {nt[lead].mean():.1f}; epilogue wait "
          f"{ew[lead].mean():.0f} busy {eb[lead].mean():.0f}")
