"""Time the host-memory entry point (cgb_conv_host) per BASELINE layer: pinned vs
pageable caller buffers, sweeping the pipeline chunk size; plus raw PCIe copy rates."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2005_06410_b200 as cg
import bench

def raw_pcie(nbytes=256 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(f"raw {name} pinned {nbytes / dt / 1e9:.1f} GB/s")
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"raw bidirectional {2 * nbytes / dt / 1e9:.1f} GB/s total")
    hp = np.empty(nbytes, dtype=np.uint8); hp[:] = 1
    t = time.perf_counter(); d.copy_(torch.from_numpy(hp)); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"raw h2d pageable {nbytes / dt / 1e9:.1f} GB/s")

def host_memcpy(nbytes=512 << 20):
    from concurrent.futures import ThreadPoolExecutor
    a = np.ones(nbytes, np.uint8); b = np.ones(nbytes, np.uint8)
    for nt in (1, 2, 4, 8, 16):
        ex = ThreadPoolExecutor(nt)
        per = nbytes // nt
        def job(i):
            np.copyto(b[i * per:(i + 1) * per], a[i * per:(i + 1) * per])
        list(ex.map(job, range(nt)))
        t = time.perf_counter(); list(ex.map(job, range(nt))); dt = time.perf_counter() - t
        print(f"host memcpy {nt:2d} threads {nbytes / dt / 1e9:.1f} GB/s (copied bytes)")
        ex.shutdown()
    print("cpus", os.cpu_count())

if not os.environ.get("HB_SKIP_RAW"):
    raw_pcie()
    host_memcpy()
layers = bench.LAYERS if len(sys.argv) < 2 else [l for l in bench.LAYERS if l[0] in sys.argv[1:]]
tensors = bench.make_layer_tensors(cg, torch, layers, 128, 0, 1)
host = []
for layer, cp, F, I, O in tensors:
    hF = F.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy().reshape(F.shape, order="F")
    hI = I.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy().reshape(I.shape, order="F")
    host.append((layer, cp, hF, hI, O.shape))
def pinned(a):
    t = torch.empty(a.size, dtype=torch.float32, pin_memory=True)
    v = t.numpy(); v[:] = a.reshape(-1, order="F")
    return v.reshape(a.shape, order="F"), t
for mb in os.environ.get("HB_MB", "4,8,16,32").split(","):
    os.environ["CGB_HOST_CHUNK_MB"] = mb
    for kind in ("pinned", "pageable"):
        tot = 0.0
        keep = []
        for layer, cp, hF, hI, os_ in host:
            if kind == "pinned":
                F, k1 = pinned(hF); I, k2 = pinned(hI); O, k3 = pinned(np.zeros(os_, np.float32, order="F"))
                keep += [k1, k2, k3]
            else:
                F, I, O = hF, hI, np.zeros(os_, np.float32, order="F")
            cg.conv(F, I, cp, algo="fused", precision="tf32", out=O)
            reps = 3
            t = time.perf_counter()
            for _ in range(reps):
                cg.conv(F, I, cp, algo="fused", precision="tf32", out=O)
            dt = (time.perf_counter() - t) / reps
            tot += dt
        fl = sum(bench.flops(cp) for _, cp, _, _, _ in host)
        print(f"chunk {mb:>4} MB {kind:8s}: step {tot * 1e3:7.2f} ms  e2e {fl / tot / 1e12:6.2f} TFLOPS")
