import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_2005_06410_b200 as cg
from oracle.oracle import Restatement, per_output_error
orc = Restatement()
def dev(a):
    a = np.asfortranarray(a, dtype=np.float32); d = a.shape
    return torch.from_numpy(a.reshape(-1, order='F').copy()).cuda().view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0)
def host(t):
    d = t.shape; return t.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy().reshape(d, order='F')
cases = [dict(k_n=64, k_h=1, k_w=1, c_i=32, h_i=16, w_i=16, b=2, s=1, p=0),
         dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=16, w_i=16, b=2, s=1, p=0),
         dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=8, w_i=8, b=1, s=1, p=1),
         dict(k_n=64, k_h=3, k_w=3, c_i=32, h_i=16, w_i=16, b=2, s=1, p=1),
         dict(k_n=64, k_h=3, k_w=3, c_i=64, h_i=56, w_i=56, b=2, s=1, p=1),
         dict(k_n=128, k_h=3, k_w=3, c_i=32, h_i=28, w_i=28, b=2, s=2, p=1)]
for cp in sys.argv[1:] and [cases[int(i)] for i in sys.argv[1:]] or cases:
    rng = np.random.default_rng(0)
    F = rng.uniform(-1, 1, (cp['k_n'], cp['k_h'], cp['k_w'], cp['c_i'])).astype(np.float32)
    I = rng.uniform(-1, 1, (cp['h_i'], cp['w_i'], cp['c_i'], cp['b'])).astype(np.float32)
    try:
        O = host(cg.conv(dev(F), dev(I), cp, precision='tf32'))
        torch.cuda.synchronize()
        err = per_output_error(O, orc.conv_gemm(np.asfortranarray(F), np.asfortranarray(I), cp), orc.output_scale(np.asfortranarray(F), np.asfortranarray(I), cp))
        print(cp, cg.last_path(), 'err', err, flush=True)
    except Exception as e:
        print(cp, 'EXC', str(e)[:200], flush=True); break
