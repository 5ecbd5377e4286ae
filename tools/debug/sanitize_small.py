"""Small xGETT calls through every kernel family, for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.workloads import C1, C3, C5  # noqa: E402

for mode in ("tiled", "ref", "ffma"):
    g.set_kernel(mode)
    for w in (C1, C3.slice_free("A", 0, 0, 2).slice_free("A", 2, 0, 20), C5.slice_free("A", 0, 0, 1)):
        a, b, c = w.buffers()
        pos, kw = w.args(a, b, c)
        assert (g.dgett if w.dtype == "d" else g.sgett)(*pos, **kw) == []
        print(mode, w.name, g.last_kernel(), flush=True)
    rng = np.random.default_rng(1)
    for dt, entry in ((np.complex128, g.zgett), (np.complex64, g.cgett)):
        A = (rng.uniform(-1, 1, 200 * 70) + 1j).astype(dt)
        B = (rng.uniform(-1, 1, 70 * 130) - 1j).astype(dt)
        C = np.zeros(200 * 130, dt)
        assert entry(2, (200, 70), (1, 200), A, 2, (70, 130), (1, 70), B, 1, (1,), (0,), (0, 1), (1, 200), C) == []
        print(mode, dt.__name__, g.last_kernel(), flush=True)
g.set_kernel("auto")
args = (2, (3, 4), (1, 3), np.ones(12), 2, (4, 5), (1, 4), np.ones(20), 1, (1,), (0,), (0, 1), (1, 1))
assert g.dgett(*args, np.zeros(10)) == []
print("serial", g.last_kernel())
g.zero_view(g.TensorView(2, (3, 3), (1, 5), 2, 20), np.ones(20))
print("ok")
