import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2410_06770_b200 as g
from tests.golden_util import load_suite
g.set_kernel("tiled")
S = {c.id: c for c in load_suite()}
ids = ["Scalar contraction/1000026/d-int", "Scalar contraction/1000032/d-int",
       "Rank one tensor/1000007/d-int", "Rank one tensor/1000008/d-int"]
for rep in range(3):
    for k in ids:
        c = S[k]; a, b, cc = c.buffers()
        pos, kw = c.args(a, b, cc)
        g.dgett(*pos, **kw)
        print(rep, k, "got", cc, "want", c.want, g.last_kernel())
# synthetic dots
rng = np.random.default_rng(0)
bad = 0
for K in range(1, 40):
    for t in range(5):
        a = rng.integers(-4, 5, K).astype(float); b = rng.integers(-4, 5, K).astype(float)
        c0 = float(rng.integers(-4, 5)); c = np.array([c0])
        g.dgett(1, (K,), (1,), a, 1, (K,), (1,), b, 1, (0,), (0,), (), (), c)
        if c[0] != c0 + a @ b:
            bad += 1
            print("BAD K", K, "got", c[0], "want", c0 + a @ b, "c0", c0, "dot", a @ b)
print("bad", bad)
