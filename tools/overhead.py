"""Host-side cost of one device-entry xGETT call (no synchronisation): the
full Python entry point vs the bare native call with pre-built arguments.

    python tools/overhead.py [config ...]
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())

import torch  # noqa: E402

import paper_2410_06770_b200 as g  # noqa: E402
from paper_2410_06770_b200 import _native  # noqa: E402
from paper_2410_06770_b200.device import dgett_device, sgett_device  # noqa: E402
from paper_2410_06770_b200.plan import prepare  # noqa: E402
from paper_2410_06770_b200.workloads import CONFIGS  # noqa: E402


def per_call(fn, n):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    dt = time.perf_counter() - t
    torch.cuda.synchronize()
    return dt / n * 1e6


def main():
    names = sys.argv[1:] or ["c1", "c5"]
    for name in names:
        w = CONFIGS[name]
        a, b, c = w.buffers()
        ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
        fn = dgett_device if w.dtype == "d" else sgett_device
        pos, kw = w.args(ta, tb, tc)
        for _ in range(3):
            fn(*pos, **kw)
        n = 200
        full = per_call(lambda: fn(*pos, **kw), n)
        pr = prepare(len(w.ext_a), w.ext_a, w.inc_a, w.off_a, len(a), len(w.ext_b), w.ext_b,
                     w.inc_b, w.off_b, len(b), w.conts, w.cont_a, w.cont_b, w.perm, w.inc_c)
        cap = pr.cap
        codes = (ctypes.c_int32 * cap)()
        info = (ctypes.c_int64 * (cap * _native.ERR_INFO_WORDS))()
        nat = getattr(_native.LIB, f"gett_{w.dtype}gett_device")
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        args = (*pr.args_a, ta.data_ptr(), w.off_a, len(a), *pr.args_b, tb.data_ptr(), w.off_b,
                len(b), *pr.args_spec, tc.data_ptr(), w.off_c, len(c), stream, codes, info, cap)
        native = per_call(lambda: nat(*args), n)
        g.set_kernel("ref")
        ref = per_call(lambda: nat(*args), n)
        g.set_kernel("auto")
        empty = per_call(lambda: torch.cuda.current_stream(), n)
        # plan handle: device tensors (stream-ordered) and the bare execute
        plan = (g.dgett_plan if w.dtype == "d" else g.sgett_plan)(
            *w.args(a, b, c)[0], **w.args(a, b, c)[1])
        pdev = per_call(lambda: plan.device(ta, tb, tc), n)
        h, ex = plan._h, _native.LIB.gett_execute_device
        pa, pb, pc = ta.data_ptr(), tb.data_ptr(), tc.data_ptr()
        pnat = per_call(lambda: ex(h, pa, pb, pc, stream), n)
        # host buffers, synchronous end to end (pinned): dgett vs the plan
        ha, hb, hc = (torch.from_numpy(x).pin_memory().numpy() for x in (a, b, c))
        hpos, hkw = w.args(ha, hb, hc)
        entry = g.dgett if w.dtype == "d" else g.sgett
        host_full = per_call(lambda: entry(*hpos, **hkw), n)
        host_plan = per_call(lambda: plan(ha, hb, hc), n)
        plan.close()
        print(json.dumps({"config": name, "us_per_call_python_entry": round(full, 2),
                          "us_per_call_native": round(native, 2),
                          "us_per_call_native_ref_kernel": round(ref, 2),
                          "us_per_call_plan_device": round(pdev, 2),
                          "us_per_call_plan_native_execute": round(pnat, 2),
                          "us_per_call_host_dgett_sync": round(host_full, 2),
                          "us_per_call_host_plan_sync": round(host_plan, 2),
                          "us_current_stream": round(empty, 2), "kernel": g.last_kernel()}),
              flush=True)


if __name__ == "__main__":
    main()
