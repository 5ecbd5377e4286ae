import sys, numpy as np
sys.path.insert(0, '.')
import paper_2410_06770_b200 as g
from tests.test_gpu_kr import _case, _strided
def err_of(pos, kw, c0):
    (ra, ext_a, inc_a, a, rb, ext_b, inc_b, b, _, _, _, _, inc_c, c) = pos
    A = _strided(a, ext_a, inc_a, 0).astype(np.float64); B = _strided(b, ext_b, inc_b, 0).astype(np.float64)
    ext_c = (ext_a[0], ext_a[1], ext_b[2])
    want = _strided(c0, ext_c, inc_c, kw["offset_c"]).astype(np.float64) + np.einsum("abjk,kjn->abn", A, B)
    got = _strided(c, ext_c, inc_c, kw["offset_c"]).astype(np.float64)
    d = np.abs(got - want)
    bad = np.argwhere(d > 1e-3)
    return d.max(), bad[:5].tolist(), len(bad)
for shape in [(2,64,16,30,40),(2,64,16,30,48),(2,64,16,30,96),(2,64,40,30,40),(6,16,40,24,96)]:
  for cm in (True, False):
    for split in (1, 0):
        for fused in (False, True):
            pos, kw = _case(*shape, cm, seed=7)
            c0 = pos[13].copy()
            g.set_split_k(split); g.set_kernel("tiled"); g.set_kr("force", fused)
            assert g.sgett(*pos, **kw) == []
            print(shape, "cm", cm, "split", split, "fused", fused, g.last_kernel(), err_of(pos, kw, c0))
