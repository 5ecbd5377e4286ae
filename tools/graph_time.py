"""Per-call time of a device xGETT issued directly vs replayed from a CUDA
graph (graph.py), back to back on one stream.

    python tools/graph_time.py c1 c5
"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2410_06770_b200.device import dgett_device, sgett_device  # noqa: E402
from paper_2410_06770_b200.graph import GettGraph  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS  # noqa: E402


def per_call(f, n=200):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


for name in sys.argv[1:] or ["c1"]:
    w = CONFIGS[name]
    ta, tb, tc = (torch.from_numpy(x).cuda() for x in w.buffers())
    fn = dgett_device if w.dtype == "d" else sgett_device
    pos, kw = w.args(ta, tb, tc)
    direct = per_call(lambda: fn(*pos, **kw))
    gg = GettGraph(fn, *pos, **kw)
    replay = per_call(gg.replay)
    print(json.dumps({"config": name, "us_per_call_direct": round(direct, 2),
                      "us_per_call_graph_replay": round(replay, 2)}))
