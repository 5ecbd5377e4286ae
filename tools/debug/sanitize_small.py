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
# the TMA SGETT (single CTA and the CTA pair), the staged dot kernel and the
# DGETT stream-K schedule below one wave, on small shapes
g.set_kernel("tiled")
rng = np.random.default_rng(2)
a = rng.uniform(-1, 1, 96 * 8 * 40 + 64).astype(np.float32)   # A (m 96, k 8x40) rows-major
b = rng.uniform(-1, 1, 300 * 320 + 64).astype(np.float32)     # B (n 300, k 8x40) K-major
for pair in (False, True):
    g.set_pair(pair)
    c = np.zeros(96 * 300 + 8, np.float32)
    assert g.sgett(3, (96, 8, 40), (1, 96, 768), a, 3, (300, 8, 40), (320, 40, 1), b, 2, (1, 2), (1, 2),
                   (0, 1), (1, 96), c) == []
    print("tiled", "tma pair" if pair else "tma", g.last_kernel(), flush=True)
g.set_pair(False)
g.set_kernel("dot")
a = rng.uniform(-1, 1, 24 * 1280)
b = rng.uniform(-1, 1, 1280 * 20)
c = np.zeros(24 * 20)
assert g.dgett(2, (24, 1280), (1280, 1), a, 2, (1280, 20), (20, 1), b, 1, (1,), (0,), (0, 1), (20, 1), c) == []
print("dot", g.last_kernel(), flush=True)
g.set_kernel("tiled")
a = rng.uniform(-1, 1, 640 * 256)
b = rng.uniform(-1, 1, 256 * 4096)
c = np.zeros(640 * 4096)
assert g.dgett(2, (640, 256), (256, 1), a, 2, (256, 4096), (4096, 1), b, 1, (1,), (0,), (0, 1), (4096, 1), c) == []
print("tiled", g.last_kernel(), flush=True)
g.set_kernel("auto")
args = (2, (3, 4), (1, 3), np.ones(12), 2, (4, 5), (1, 4), np.ones(20), 1, (1,), (0,), (0, 1), (1, 1))
assert g.dgett(*args, np.zeros(10)) == []
print("serial", g.last_kernel())
g.zero_view(g.TensorView(2, (3, 3), (1, 5), 2, 20), np.ones(20))
print("ok")
