import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2410_06770_b200 as g
from oracle import oracle
from paper_2410_06770_b200.workloads import C5
g.set_kernel("tiled")
for w in [C5.slice_free("A", 0, 0, 1).slice_free("A", 3, 0, 8), C5.slice_free("A", 0, 0, 2), C5]:
    a, b, c = w.buffers()
    want = c.copy(); pos, kw = w.args(a, b, want)
    oracle.oracle_sgett(*pos, **kw, threads=16)
    got = c.copy(); pos, kw = w.args(a, b, got)
    errs = g.sgett(*pos, **kw)
    err = np.max(np.abs(got.astype(np.float64) - want)) / (w.size_k)
    print(w.name, g.last_kernel(), errs, "errK", err, "maxdiff", np.max(np.abs(got.astype(np.float64) - want)), flush=True)
