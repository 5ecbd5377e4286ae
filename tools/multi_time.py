"""Host-buffer xGETT through one device vs the multi-device path on lanes of
the same GPU (devices=(0,)*n): the cost of the multi-device orchestration
(chunked upload + peer exchange of the replicated operand, per-lane slabs or
split-K + reduce).  On one GPU the lanes share one PCIe link and one set of
SMs, so this measures overhead, not scaling.

  python tools/multi_time.py [c2 c5 ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS  # noqa: E402


def timeit(fn, reps):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


def main(names):
    for name in names:
        w = CONFIGS[name]
        a, b, c = (torch.from_numpy(x).pin_memory().numpy() for x in w.buffers())
        pos, kw = w.args(a, b, c)
        entry = g.dgett if w.dtype == "d" else g.sgett
        reps = 5 if w.flops > 1e10 else 50
        row = {"config": name, "one_device_ms": 1e3 * timeit(lambda: entry(*pos, **kw), reps)}
        for n in (2, 4):
            t = timeit(lambda: entry(*pos, **kw, devices=(0,) * n), reps)
            row[f"lanes{n}_ms"] = 1e3 * t
            row[f"lanes{n}_sched"] = g.last_multi()
        row = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in row.items()}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4", "c5"])
