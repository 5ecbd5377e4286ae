"""cgett / zgett device timing, embedded vs four real GETTs (one GPU)."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.device import cgett_device, sgett_device, zgett_device, dgett_device  # noqa: E402

for n in (1024, 2048):
    for dt, fn, name, mul in ((torch.complex64, cgett_device, "cgett", 8), (torch.float32, sgett_device, "sgett", 2),
                              (torch.complex128, zgett_device, "zgett", 8), (torch.float64, dgett_device, "dgett", 2)):
        a = torch.rand(n * n, dtype=dt, device="cuda")
        b = torch.rand(n * n, dtype=dt, device="cuda")
        c = torch.zeros(n * n, dtype=dt, device="cuda")
        args = (2, (n, n), (n, 1), a, 2, (n, n), (n, 1), b, 1, (1,), (0,), (0, 1), (n, 1), c)
        for embed in ((True, False) if dt.is_complex else (True,)):
            g.set_complex_embed(embed)
            for _ in range(3):
                fn(*args)
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(10):
                fn(*args)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t) / 10 * 1e3
            print(json.dumps({"op": name, "n": n, "ms": round(ms, 3), "tflops": round(mul * n ** 3 / ms / 1e9, 1),
                              "kernel": g.last_kernel()}))
g.set_complex_embed(True)
