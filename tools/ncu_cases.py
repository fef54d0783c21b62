"""One launch of a non-headline kernel for ncu (profiles/r02_*): python tools/ncu_cases.py CASE
  explicit  56x56 64->64 b=128 through the explicit path: K1 im2col_slab_kernel + K2 k2_gemm_kernel
  explicit3x  the same in 3xTF32 (filter_prep + K1 + K2 with the lo warps)
  ffma      VGG conv1 (224^2 3->64) b=64 on the FFMA kernel (K4)
  fc6       VGG fc6 (4096 x 25088) at b=64 through cgb_gemm (TF32)
  stem      the 7x7/s2 stem at b=256 (w-im2col mode of the shifted-window kernel)
  pw56      1x1 56^2 64->256 at b=256 (TMA-fed A)
  vgg56     VGG 56^2 256->256 at b=64 (the shifted-window kernel's best BASELINE layer, 860 TFLOP/s)
  direct    conv_direct (bit-exact reference order) on a small layer
  gather    AlexNet conv1 (11x11 stride 4, 3->64, 224^2) at b=64: outside the shifted-window
            domain (stride > 2), the tap-major gather kernel or the reference-order implicit GEMM
  tgather   3x3 stride 3, 64->128, 56^2, b=64: c_i >= 16 outside the shifted-window domain -> the
            tap-major gather kernel (tc_gather)
  alex5     AlexNet conv2 (5x5, 64->192, 55^2, unpadded) at b=64 on the shifted-window kernel (25 taps)
Runs the operation twice (the first launch warms allocations); profile with -s/-c."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2005_06410_b200 as cg  # noqa: E402
from paper_2005_06410_b200 import configs  # noqa: E402

case = sys.argv[1]
by = {l[0]: (c, l, cp, d) for c, l, cp, d in configs.all_layers()}


def layer(name, b=None, **kw):
    c, l, cp, d = by[name]
    if b:
        cp = dict(cp, b=b)
    F, I = configs.make_tensors(torch, cg.empty_tensor4, cp, d, 7)
    return cp, F, I


for _ in range(2):
    if case == "explicit":
        cp, F, I = layer("r50_3x3_56_64")
        cg.conv(F, I, cp, algo="explicit", precision="tf32")
    elif case == "explicit3x":
        cp, F, I = layer("r50_3x3_56_64")
        cg.conv(F, I, cp, algo="explicit", precision="3xtf32")
    elif case == "ffma":
        cp, F, I = layer("vgg_224_3_64")
        cg.conv(F, I, cp, precision="ffma")
    elif case == "fc6":
        g = torch.Generator(device="cuda").manual_seed(3)
        A = (torch.rand((25088, 4096), generator=g, device="cuda") * 2 - 1).t()  # 4096 x 25088, column-major
        B = (torch.rand((64, 25088), generator=g, device="cuda") * 2 - 1).t()    # 25088 x 64
        cg.gemm(A, B, precision="tf32")
    elif case == "stem":
        cp, F, I = layer("stem_7x7_s2_224")
        cg.conv(F, I, cp, precision="tf32")
    elif case == "vgg56":
        cp, F, I = layer("vgg_56_256_256a")
        cg.conv(F, I, cp, precision="tf32")
    elif case == "pw56":
        cp, F, I = layer("pw_56_64_256")
        cg.conv(F, I, cp, precision="tf32")
    elif case in ("gather", "alex5", "tgather"):
        cp = dict(k_n=128, k_h=3, k_w=3, c_i=64, h_i=56, w_i=56, b=64, s=3, p=1) if case == "tgather" else dict(k_n=64, k_h=11, k_w=11, c_i=3, h_i=224, w_i=224, b=64, s=4, p=0) if case == "gather" else \
            dict(k_n=192, k_h=5, k_w=5, c_i=64, h_i=55, w_i=55, b=64, s=1, p=0)
        F, I = configs.make_tensors(torch, cg.empty_tensor4, cp, "uniform", 11)
        cg.conv(F, I, cp, precision="tf32")
    elif case == "direct":
        cp, F, I = layer("r50_3x3_14_256", b=2)
        cg.conv(F, I, cp, algo="direct")
    torch.cuda.synchronize()
print(case, "ok", cg.last_path())
