"""DGETT below half a wave of tiles: device time per call for row-slabs of c2's
GEMM shape and small cubes (split-K vs stream-K: run with GETT_SK_SMALL=0/1)."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.device import dgett_device  # noqa: E402

for m, n, k in ((1024, 1024, 1024), (768, 768, 2048), (256, 4096, 4096), (128, 4096, 4096), (512, 2048, 4096)):
    a = torch.rand(m * k, dtype=torch.float64, device="cuda")
    b = torch.rand(k * n, dtype=torch.float64, device="cuda")
    c = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    args = (2, (m, k), (k, 1), a, 2, (k, n), (n, 1), b, 1, (1,), (0,), (0, 1), (n, 1), c)
    for _ in range(5):
        dgett_device(*args)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(30):
        dgett_device(*args)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / 30 * 1e3
    print(json.dumps({"m": m, "n": n, "k": k, "sk_small": os.environ.get("GETT_SK_SMALL", "0"), "ms": round(ms, 4),
                      "tflops": round(2 * m * n * k / ms / 1e9, 2), "kernel": g.last_kernel()}))
