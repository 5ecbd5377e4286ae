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
    return float(d.max()), bad[:4].tolist(), len(bad)
if __name__ == "__main__":
    order = [(6,16,40,24,96),(3,50,8,64,128),(2,64,16,30,40)]
    if len(sys.argv) > 1: order = order[int(sys.argv[1]):]
    for shape in order:
        for fused in (True, False):
            pos, kw = _case(*shape, True, seed=sum(shape))
            c0 = pos[13].copy()
            g.set_split_k(0); g.set_kernel("tiled"); g.set_kr("force", fused)
            assert g.sgett(*pos, **kw) == []
            print(shape, "fused", fused, g.last_kernel(), err_of(pos, kw, c0), flush=True)
