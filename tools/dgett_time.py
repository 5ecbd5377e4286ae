"""Device time of one DGETT/SGETT config per call (CUDA events, L2 flushed,
median of 15), bitwise checksum of the output; env knobs (GETT_*) apply.
    python tools/dgett_time.py c2 c3 c4"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200.device import dgett_device, sgett_device  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS  # noqa: E402


def main(names):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for name in names:
        w = CONFIGS[name]
        entry = dgett_device if w.dtype == "d" else sgett_device
        a, b, c = w.buffers()
        ta, tb, tc0 = (torch.from_numpy(x).cuda() for x in (a, b, c))
        tc = tc0.clone()
        pos, kw = w.args(ta, tb, tc)
        assert entry(*pos, **kw) == []
        digest = hashlib.sha1(tc.cpu().numpy().tobytes()).hexdigest()[:12]
        times = []
        for _ in range(15):
            flush.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            entry(*pos, **kw)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        times.sort()
        ms = times[len(times) // 2]
        print(json.dumps({"config": name, "kernel": g.last_kernel(), "ms": round(ms, 4),
                          "tflops": round(w.flops / ms / 1e9, 2),
                          "out_sha": digest, "env": {k: v for k, v in os.environ.items() if k.startswith("GETT_")}}))


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4"])
