"""DGETT through the TMA-fed and the cp.async-fed warp-specialised kernels:
bitwise equality (same values, same DMMA order) and device time per call
(CUDA events, L2 flushed, median of 9).   python tools/dgett_tma_check.py [c2 c3 c4]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200 import _native  # noqa: E402
from paper_2410_06770_b200.device import dgett_device  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS, colmajor  # noqa: E402


def main(names):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for name in names:
        w = CONFIGS[name.split(":")[0]]
        if name.endswith(":col"):
            w = colmajor(w)
        a, b, c = w.buffers()
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        res = {}
        for tma in (1, 0):
            os.environ["GETT_DGETT_TMA"] = str(tma)
            _native.LIB.gett_set_tma(1)
            g.set_tma(True)
            # (GETT_DGETT_TMA is read once per process: toggle through the SGETT
            # switch instead when it is off)
            if not tma:
                g.set_tma(False)
            tc = torch.from_numpy(c).cuda()
            pos, kw = w.args(ta, tb, tc)
            assert dgett_device(*pos, **kw) == []
            kname = g.last_kernel()
            out = tc.cpu().numpy()
            times = []
            for _ in range(9):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dgett_device(*pos, **kw)
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            ms = float(np.median(times))
            res[tma] = out
            print(json.dumps({"config": name, "tma": tma, "kernel": kname, "ms": round(ms, 4),
                              "tflops": round(w.flops / ms / 1e9, 2)}), flush=True)
        g.set_tma(True)
        print(json.dumps({"config": name, "bitwise_equal": res[0].tobytes() == res[1].tobytes()}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4", "c3:col", "c4:col"])
