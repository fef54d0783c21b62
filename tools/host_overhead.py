"""Host cost of one cg.conv call (python + ctypes + cgb_conv host work) and the
back-to-back device time, for the BASELINE layers; plus CUDA-graph replay of the
7 launches (removes host submission from the device timeline)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_06410_b200 as cg
import bench

tensors = bench.make_layer_tensors(cg, torch, bench.LAYERS, 128, 0, 1)
st = torch.cuda.current_stream()
for layer, cp, F, I, O in tensors:
    cg.conv(F, I, cp, algo="fused", precision="tf32", out=O)
torch.cuda.synchronize()
# host-only cost: enqueue N calls of the smallest layer while the GPU is busy
big = torch.empty(1 << 28, device="cuda")
for layer, cp, F, I, O in tensors[:2]:
    n = 200
    big.zero_()
    t = time.perf_counter()
    for _ in range(n):
        cg.conv(F, I, cp, algo="fused", precision="tf32", out=O)
    dt = (time.perf_counter() - t) / n
    torch.cuda.synchronize()
    print(f"host per cg.conv call ({layer[0]}): {dt * 1e6:.1f} us")
lib = cg.lib
import ctypes
cpc = cg.ConvParams.of(tensors[0][1]).c()
F, I, O = tensors[0][2], tensors[0][3], tensors[0][4]
n = 200
t = time.perf_counter()
for _ in range(n):
    lib.cgb_conv(1, 2, F.data_ptr(), I.data_ptr(), ctypes.byref(cpc), O.data_ptr(), None, 0, st.cuda_stream)
dt = (time.perf_counter() - t) / n
torch.cuda.synchronize()
print(f"host per raw cgb_conv ctypes call: {dt * 1e6:.1f} us")

# stream timeline: 7 layers eager vs graph
def step():
    for layer, cp, F, I, O in tensors:
        cg.conv(F, I, cp, algo="fused", precision="tf32", out=O)
for mode in ("eager", "graph"):
    if mode == "graph":
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            step()
        torch.cuda.current_stream().wait_stream(s2)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            step()
        run = g.replay
    else:
        run = step
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = sum(bench.flops(cp) for _, cp, _, _, _ in tensors)
    print(f"{mode}: {ms * 1e3:.1f} us per 7-layer step  {fl / ms / 1e9:.1f} TFLOPS")
