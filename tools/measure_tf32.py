"""Measured TF32 tensor-core peak on this box: fp32 torch.matmul
8192^3 with TF32 enabled (cuBLAS), best of 10 (burst) and back to back for 4 s
(sustained); writes profiles/tf32_peak.json, which bench.py uses as the roofline peak."""
import json, os, time
import torch
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda")
fl = 2 * n ** 3
for _ in range(3):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
    best = max(best, fl / (e0.elapsed_time(e1) * 1e-3) / 1e12)
t_end = time.time() + 4.0
cnt = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() < t_end:
    for _ in range(20):
        torch.matmul(a, b)
    cnt += 20
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sus = fl * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
out = {"tf32_tflops": round(best, 1), "tf32_tflops_sustained": round(sus, 1),
       "how": "torch.matmul fp32 8192^3, allow_tf32 (cuBLAS), best of 10 (burst) / back to back 4 s (sustained)",
       "gpu": torch.cuda.get_device_name(), "torch": torch.__version__}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs(os.path.join(root, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(root, "gpurun_out", "tf32_peak.json"), "w"), indent=1)
print(json.dumps(out))
