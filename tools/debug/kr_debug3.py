import sys, numpy as np
sys.path.insert(0, '.')
import paper_2410_06770_b200 as g
from tests.test_gpu_kr import _case, _strided
from tools.debug.kr_debug2 import err_of
for shape in [(3,33,64,8,112),(3,33,64,8,48),(3,33,56,8,112),(3,33,48,16,112),(2,64,64,8,112)]:
    for split in (1, 2, 4):
        pos, kw = _case(*shape, True, seed=1)
        c0 = pos[13].copy()
        g.set_split_k(split); g.set_kernel("tiled"); g.set_kr("force", False)
        assert g.sgett(*pos, **kw) == []
        print(shape, "split", split, g.last_kernel(), err_of(pos, kw, c0), flush=True)
