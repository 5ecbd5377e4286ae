"""c5-class SGETT on the k-run kernel vs the tiled tcgen05 kernel: accuracy vs
fp64 (K-normalised), fused vs separate split-K reduce (bitwise), device time
(CUDA events, L2 flushed, median of 21).

  python tools/kr_check.py [c5 ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2410_06770_b200.device import sgett_device  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS  # noqa: E402

MODES = [("tiled", dict(kr="off")), ("kr_fused", dict(kr="force", fused=True)), ("kr_pair", dict(kr="force")),
         ("kr_single", dict(kr="force", pair=False))]


def main(names):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for name in names:
        w = CONFIGS[name]
        a, b, c = w.buffers()
        ref = oracle.einsum_check(w.ext_a, w.inc_a, a, w.off_a, w.ext_b, w.inc_b, b, w.off_b,
                                  w.conts, w.cont_a, w.cont_b, w.perm)
        ref = ref + oracle.strided(c, w.ext_c, w.inc_c, w.off_c).astype(np.float64)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        outs = {}
        for mode, kw in MODES:
            g.set_kr(kw["kr"], kw.get("fused", False), kw.get("pair", True))
            tc = torch.from_numpy(c).cuda()
            pos, kwa = w.args(ta, tb, tc)
            assert sgett_device(*pos, **kwa) == []
            kname = g.last_kernel()
            got = tc.cpu().numpy()
            outs[mode] = got
            err = np.max(np.abs(oracle.strided(got, w.ext_c, w.inc_c, w.off_c) - ref)) / (
                w.size_k * np.abs(a).max() * np.abs(b).max())
            times = []
            for _ in range(21):
                tc2 = torch.from_numpy(c).cuda()
                pos, kwa = w.args(ta, tb, tc2)
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sgett_device(*pos, **kwa)
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            ms = float(np.median(times))
            print(json.dumps({"config": name, "mode": mode, "kernel": kname, "err_k": err, "ms": round(ms, 4),
                              "gflops": round(w.flops / ms / 1e6, 1),
                              "hbm_frac": round(w.alg_bytes / (ms * 1e-3) / 6546.2e9, 3)}), flush=True)
        if "kr_fused" in outs:
            print(json.dumps({"config": name, "fused_eq_sep": outs["kr_fused"].tobytes() == outs["kr_pair"].tobytes()}))
        g.set_kr("auto")


if __name__ == "__main__":
    main(sys.argv[1:] or ["c5"])
