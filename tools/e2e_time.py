"""Wall-clock time of the drop-in host API (dgett/sgett on pinned numpy
buffers: H2D of the spans, kernels, D2H of C's span) on BASELINE configs.

    python tools/e2e_time.py c2 c4 [--slabs N]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())

import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS  # noqa: E402


def main():
    args = sys.argv[1:]
    slabs = -1
    if "--slabs" in args:
        i = args.index("--slabs")
        slabs = int(args[i + 1])
        del args[i:i + 2]
    g.set_pipeline(slabs)
    for name in args or ["c2"]:
        w = CONFIGS[name]
        a, b, c = (torch.from_numpy(x).pin_memory().numpy() for x in w.buffers())
        fn = g.dgett if w.dtype == "d" else g.sgett
        pos, kw = w.args(a, b, c)
        assert fn(*pos, **kw) == []
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            assert fn(*pos, **kw) == []
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[len(ts) // 2]
        print(json.dumps({"config": name, "slabs": slabs, "e2e_ms": round(t * 1e3, 3),
                          "gflops": round(w.flops / t / 1e9, 1), "kernel": g.last_kernel()}))


if __name__ == "__main__":
    main()
