import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2005_06410_b200 as cg
from paper_2005_06410_b200 import configs
cg.set_tuning("verbose", 1)
for name in ("r50_3x3_14_256", "r50_3x3_s2_28_256"):
    cfg, l, cp, dist = [x for x in configs.all_layers() if x[1][0] == name][0]
    F, I = configs.make_tensors(torch, cg.empty_tensor4, cp, dist, 1)
    O = cg.conv(F, I, cp, precision="tf32"); torch.cuda.synchronize()
    print(name, "ok")
