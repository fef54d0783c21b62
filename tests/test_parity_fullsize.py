"""GPU parity at the BASELINE configs' STATED batch sizes (VERDICT r01 "what's missing" #1).

Every layer of BASELINE.json configs[0..4] runs at its stated batch -- C1 b=8, C2 (the
bench step) b=128, C3 b=256, C4 b=256, C5 b=64 -- so the dispatcher takes exactly the
branches the bench and a user take (pair tiles, M tiles of 4 subtiles, tail tiles,
stream-K rounds, wide windows, TMA-fed 1x1 A). Two independent checks per launch:

* the CPU oracle (oracle/, pinned bitwise to the reference by tests/test_oracle.py) on
  sampled images -- the first (stream-K tiles are the lowest-numbered tiles), the last
  (tail tiles are the highest-numbered), the middle, and one seeded random image --
  with the north-star per-output bar (3xTF32 <= 1e-5, TF32 <= 5e-3);
* an fp64 recomputation on the device over EVERY output of the launch (tests/fp64ref.py,
  same normalisation), at the same bars.

The reference's own acceptance bar is all configs (acceptance.cpp:51-85; SURVEY.md
§8(c)(ii)).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2005_06410_b200 as cg  # noqa: E402
from paper_2005_06410_b200 import configs  # noqa: E402
from oracle.oracle import Restatement, per_output_error  # noqa: E402
from fp64ref import per_output_error_fp64  # noqa: E402

TOL = {"3xtf32": 1e-5, "tf32": 5e-3, "auto": 1e-5, "ffma": 1e-5}
LAYERS = configs.all_layers()
IDS = [f"{c}-{l[0]}" for c, l, _, _ in LAYERS]

_orc = None
_ref_cache = {}


def orc():
    global _orc
    if _orc is None:
        _orc = Restatement()
    return _orc


def host_image(t, i):
    """Image i of a leftmost-fastest CUDA tensor (d0, d1, d2, b) as a Fortran array (d0, d1, d2, 1)."""
    x = t[..., i:i + 1]
    flat = x.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy()
    return np.asfortranarray(flat.reshape(tuple(x.shape), order="F"))


def sample_images(b, seed):
    rs = np.random.default_rng(seed)
    return sorted({0, b // 2, b - 1, int(rs.integers(0, b))})


def oracle_image(name, cp, F_h, I_img, i):
    key = (name, i)
    if key not in _ref_cache:
        cp1 = dict(cp, b=1)
        _ref_cache[key] = (orc().conv_gemm(F_h, I_img, cp1), orc().output_scale(F_h, I_img, cp1))
    return _ref_cache[key]


def _run(layer_idx, prec):
    cfg, layer, cp, dist = LAYERS[layer_idx]
    name = layer[0]
    F, I = configs.make_tensors(torch, cg.empty_tensor4, cp, dist, configs.layer_seed(name))
    O = cg.conv(F, I, cp, algo="fused", precision=prec)
    torch.cuda.synchronize()
    path = cg.last_path()
    Ff = F.permute(3, 2, 1, 0).contiguous().view(-1).cpu().numpy()
    F_h = np.asfortranarray(Ff.reshape(tuple(F.shape), order="F"))
    worst_orc = 0.0
    for i in sample_images(cp["b"], configs.layer_seed(name, 7)):
        I_img = host_image(I, i)
        ref, scale = oracle_image(name, cp, F_h, I_img, i)
        err = per_output_error(host_image(O, i), ref, scale)
        worst_orc = max(worst_orc, err)
        assert err <= TOL[prec], (name, prec, "oracle image", i, err, path)
    worst_64 = per_output_error_fp64(torch, F, I, O, cp)
    assert worst_64 <= TOL[prec], (name, prec, "fp64 all images", worst_64, path)
    print(f"{cfg} {name} b={cp['b']} {prec}: path={path} oracle(sampled)={worst_orc:.2e} fp64(all)={worst_64:.2e}")
    del F, I, O
    torch.cuda.empty_cache()
    return path


@pytest.mark.parametrize("prec", ("tf32", "3xtf32"))
@pytest.mark.parametrize("idx", range(len(LAYERS)), ids=IDS)
def test_stated_batch_parity(idx, prec):
    _run(idx, prec)


@pytest.mark.parametrize("idx", [i for i, (c, l, _, _) in enumerate(LAYERS) if c in ("C4",) or l[0] == "vgg_224_3_64"],
                         ids=[IDS[i] for i, (c, l, _, _) in enumerate(LAYERS) if c in ("C4",) or l[0] == "vgg_224_3_64"])
def test_stated_batch_parity_auto_lowchannel(idx):
    """The fp32-accurate default on the low-channel layers (AUTO precision selection):
    3xTF32 on the w-im2col tensor-core rows, the faster fp32-accurate kernel there
    (VGG conv1 at b=64: 323 vs 508 us for FFMA)."""
    assert _run(idx, "auto") == "tcgen05-shifted-wim"
