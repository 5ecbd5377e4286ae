"""Time the device-resident xGETT on the BASELINE configs for one build of the
library (GETT_LIB_PATH selects a variant .so).  Prints one JSON line per
config: CUDA-event ms per call (median of reps) and TFLOP/s.

    GETT_LIB_PATH=build/variants/libgett_X.so python tools/tune.py c2 c3 c4 c5
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.device import dgett_device, sgett_device  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS  # noqa: E402


def main():
    names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    reps = int(os.environ.get("REPS", "7"))
    from dataclasses import replace

    extra = {
        # contiguous fp32 GEMM 4096^3 (row-major A[m,k], B[k,n]) as a tensor-core sanity point
        "sgemm": replace(CONFIGS["c2"], name="sgemm", dtype="s", ext_a=(4096, 4096),
                         inc_a=(4096, 1), len_a=4096 * 4096, ext_b=(4096, 4096), inc_b=(4096, 1),
                         len_b=4096 * 4096, inc_c=(4096, 1), len_c=4096 * 4096),
        "dgemm": replace(CONFIGS["c2"], name="dgemm", ext_a=(4096, 4096), inc_a=(4096, 1),
                         len_a=4096 * 4096, ext_b=(4096, 4096), inc_b=(4096, 1),
                         len_b=4096 * 4096, inc_c=(4096, 1), len_c=4096 * 4096),
    }
    for n in (2048, 4096):
        # row-major A[m,k], B[k,n]: A' K-major, B' rows-major (N fast)
        extra[f"sgemm{n}"] = replace(CONFIGS["c2"], name=f"sgemm{n}", dtype="s", ext_a=(n, n), inc_a=(n, 1),
                                     len_a=n * n, ext_b=(n, n), inc_b=(n, 1), len_b=n * n, inc_c=(n, 1),
                                     len_c=n * n)
        # the same product with the operands exchanged: the first operand is
        # B[k,n] (contracted mode 0), the second A[m,k]; perm puts m first in C
        extra[f"sgemm{n}_sw"] = replace(CONFIGS["c2"], name=f"sgemm{n}_sw", dtype="s", ext_a=(n, n),
                                        inc_a=(n, 1), len_a=n * n, ext_b=(n, n), inc_b=(n, 1), len_b=n * n,
                                        cont_a=(0,), cont_b=(1,), perm=(1, 0), inc_c=(n, 1), len_c=n * n)
    for name in names:
        w = extra[name] if name in extra else CONFIGS[name]
        a, b, c = w.buffers()
        ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
        fn = dgett_device if w.dtype == "d" else sgett_device
        pos, kw = w.args(ta, tb, tc)
        for _ in range(3):
            assert fn(*pos, **kw) == []
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(*pos, **kw)
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        # back-to-back calls keep the GPU queue full: device time per call
        # without the host-side call overhead (ctypes + plan lookup + launch)
        nq = max(4, min(50, int(20.0 / max(ms, 1e-3))))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(nq):
            fn(*pos, **kw)
        e1.record()
        e1.synchronize()
        msq = e0.elapsed_time(e1) / nq
        print(json.dumps({"lib": os.path.basename(os.environ.get("GETT_LIB_PATH", "default")),
                          "config": name, "ms": round(ms, 4),
                          "tflops": round(w.flops / ms / 1e9, 3), "kernel": g.last_kernel(),
                          "min_ms": round(min(times), 4), "ms_queued": round(msq, 4),
                          "tflops_queued": round(w.flops / msq / 1e9, 3)}), flush=True)
        del ta, tb, tc
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
