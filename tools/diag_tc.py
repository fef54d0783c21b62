"""Diagnostics for the tcgen05 operand layouts: structured inputs reveal the K/M/N mappings."""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2005_06410_b200 as cg

def dev(a):
    a = np.asfortranarray(a, dtype=np.float32); d = a.shape
    return torch.from_numpy(a.reshape(-1, order='F').copy()).cuda().view(d[3], d[2], d[1], d[0]).permute(3, 2, 1, 0)
def host(t):
    d = t.shape; return t.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy().reshape(d, order='F')

rng = np.random.default_rng(0)
KN = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cp = dict(k_n=KN, k_h=1, k_w=1, c_i=32, h_i=8, w_i=16, b=1, s=1, p=0)  # n=128, K=32
F = np.asfortranarray(rng.integers(1, 100, (KN, 1, 1, 32)).astype(np.float32))
print("== K mapping: I nonzero only in channel j; expect O[n,pix] = F[n,j]")
for j in range(32):
    I = np.zeros((8, 16, 32, 1), np.float32, order='F'); I[:, :, j, 0] = 1.0
    O = host(cg.conv(dev(F), dev(I), cp, precision='tf32'))
    col = O[:, 0, 0, 0]
    match = [jj for jj in range(32) if np.allclose(col, F[:, 0, 0, jj])]
    uniform = np.allclose(O, O[:, :1, :1, :1])
    print(j, "->", match, "uniform over pixels" if uniform else "NONUNIFORM", col[:4])
print("== M mapping: I nonzero only at pixel q (all channels 1); expect O[:, q] = sum_j F[n,j]")
rs = F[:, 0, 0, :].sum(1)
for q in [0, 1, 2, 7, 8, 9, 31, 32, 33, 64, 127]:
    I = np.zeros((8, 16, 32, 1), np.float32, order='F'); I[q % 8, q // 8, :, 0] = 1.0
    O = host(cg.conv(dev(F), dev(I), cp, precision='tf32')).reshape(KN, 128, order='F')
    nz = np.nonzero(np.abs(O).sum(0))[0].tolist()
    print(q, "-> nonzero pixels", nz, "ok" if np.allclose(O[:, q], rs) else "BAD", O[:3, q] if nz else None, rs[:3])
