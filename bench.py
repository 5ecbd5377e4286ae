"""bench.py — xGETT GFLOP/s on the BASELINE headline config (c2 = configs[1]).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one xGETT over the c2 workload: A = 4096x4096 view of a [4100,4224]
f64 parent, B = 4096x4096 view of a [4096,4160] parent, C += A·B into a
[4096,4200] parent, seeded synthetic uniform[-1,1] data.
  * value: device-resident operands (torch CUDA tensors as plumbing) through
    the zero-copy C ABI entry gett_dgett_device; CUDA events around exactly K
    steps, max over ranks; inputs (410 MB) exceed the 126 MB L2.
  * e2e: the same metric through the drop-in host API (dgett on pinned numpy
    buffers): H2D of the addressed spans + kernel + D2H of C's span per step.
  * N > 1 (torchrun): the free mode A0 (= C mode 0) is split into N row
    slabs, one per rank, no collective -> total work fixed.
  * --impl reference: the reference algorithm's CPU implementation (the C
    restatement in oracle/, all host threads) on a bounded row sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2410_06770_b200.workloads import C2  # noqa: E402

METRIC = "xGETT GFLOP/s (2·|C|·|K|/s), DGETT c2 4096^3 strided GEMM-shaped subtensor"
WORKLOAD = ("c2: DGETT A[4096,4096] view of f64 [4100,4224], B[4096,4096] view of [4096,4160], "
            "contract A1-B0, identity PERM, C += into [4096,4200] parent (BASELINE configs[1])")
FP64_PEAK_TFLOPS = 37.151  # measured DMMA m16n8k4 loop, profiles/peaks_r01.jsonl
FP64_PEAK_SRC = ("measured FP64 DMMA peak (tools/peaks.cu, profiles/peaks_r01.jsonl); "
                 "MEASURED_PEAKS.json has no FP64 figure")


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def shard(world, rank):
    rows = C2.ext_a[0]
    lo, hi = rows * rank // world, rows * (rank + 1) // world
    return C2.slice_free("A", 0, lo, hi), hi - lo


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def traffic_from_profiles():
    """dram bytes per launch of the DGETT kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_dgett_c2.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    return None


def cpu_sample(rows, threads):
    """Oracle port (reference loop restated in C) on `rows` rows of c2."""
    from oracle import oracle

    w = C2.slice_free("A", 0, 0, rows)
    a, b, c = w.buffers() if not hasattr(cpu_sample, "bufs") else cpu_sample.bufs
    cpu_sample.bufs = (a, b, c)
    pos, kw = w.args(a, b, c)
    t0 = time.perf_counter()
    oracle.oracle_dgett(*pos, **kw, threads=threads)
    return time.perf_counter() - t0, w.flops


def calibrate_rows(threads, target_s):
    dt, fl = cpu_sample(threads, threads)  # one row per thread
    rate = fl / max(dt, 1e-6)
    rows = int(target_s * rate / (2 * 4096 * 4096))
    return max(threads, min(4096, rows))


def run_reference(args):
    rank, _, world = env_rank()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    rows = calibrate_rows(threads, 3.0)
    for _ in range(args.warmup):
        cpu_sample(rows, threads)
    total_t, total_f = 0.0, 0
    for _ in range(args.steps):
        dt, fl = cpu_sample(rows, threads)
        total_t += dt
        total_f += fl
    value = total_f / total_t / 1e9
    sample = (f"{rows} of 4096 rows of c2 per step (free-mode slice of A0, bitwise equal to "
              f"the same rows of a full run), {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total_t / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "parallelism": f"rank 0 only, {threads} host threads"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def run_ours(args):
    import torch

    import paper_2410_06770_b200 as g
    from paper_2410_06770_b200.device import dgett_device

    rank, local, world = env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w, rows = shard(world, rank)
    a, b, c = C2.buffers()
    dev = torch.device("cuda", local)
    ta, tb, tc = (torch.from_numpy(x).to(dev) for x in (a, b, c))
    stream = torch.cuda.current_stream()
    pos, kw = w.args(ta, tb, tc)

    def step():
        errs = dgett_device(*pos, **kw)
        assert errs == [], errs

    for _ in range(max(3, args.warmup)):
        step()
    kname = g.last_kernel()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = g.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = g.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    # per-launch kernel time (one tiled launch per step at this size)
    k_ms = ms / args.steps
    # e2e through the host API, pinned host buffers
    pa, pb, pc = (torch.from_numpy(x).pin_memory().numpy() for x in (a, b, c))
    hpos, hkw = w.args(pa, pb, pc)
    g.dgett(*hpos, **hkw)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e2e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        assert g.dgett(*hpos, **hkw) == []
    e2e_s = (time.perf_counter() - t0) / e2e_steps

    def spans(ext, inc):
        lo = sum(i * (e - 1) for e, i in zip(ext, inc) if i < 0)
        hi = sum(i * (e - 1) for e, i in zip(ext, inc) if i > 0)
        return hi - lo + 1

    h2d = 8 * (spans(w.ext_a, w.inc_a) + spans(w.ext_b, w.inc_b) + spans(w.ext_c, w.inc_c))
    d2h = 8 * spans(w.ext_c, w.inc_c)

    if dist:
        t = torch.tensor([ms, e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1])
    total_flops = C2.flops  # all ranks together process the whole c2 per step
    value = total_flops * args.steps / (ms * 1e-3) / 1e9
    e2e_value = total_flops / e2e_s / 1e9
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    achieved = w.flops / (k_ms * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform[-1,1], SURVEY §8d)",
        "config": {"workload": WORKLOAD, "global_flops_per_step": total_flops,
                   "parallelism": f"free-mode A0 split into {world} row slab(s), no collective",
                   "l2": "inputs larger than L2 (A+B+C spans 410 MB > 126 MB)",
                   "kernel": kname},
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "achieved": round(achieved, 3),
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                     "traffic": traffic_from_profiles(), "peak_source": FP64_PEAK_SRC,
                     "kernel": kname},
        "clocks": clocks.summary(),
        "e2e": {"value": round(e2e_value, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "how": "dgett() on pinned numpy buffers: H2D spans + kernel + D2H C span, wall clock"},
    }
    if world == 1 and not args.no_configs:
        line["other_configs"] = other_configs(dev)
    if world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        rows = calibrate_rows(threads, 10.0)
        dt, fl = cpu_sample(rows, threads)
        line["cpu_baseline"] = {
            "value": round(fl / dt / 1e9, 4), "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": f"{rows} of 4096 rows of c2 ({dt:.1f} s), oracle/gett_oracle.c, {threads} threads"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# fp32 via 3xTF32: a third of the tf32 MMA rate measured by tools/mma_rate.cu
# (2046 MAC/clk/SM x 148 SMs x 1.965 GHz)
TF32X3_PEAK_TFLOPS = 2 * 2046 * 148 * 1.965e9 / 3 / 1e12


def hbm_gbs():
    """HBM GB/s: MEASURED_PEAKS.json (driver-written) when present, else the
    value it held on this pool's B200s."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6538.6


def other_configs(dev):
    """The other BASELINE configs (parity cases, not the headline): device time
    per call, each call timed alone with CUDA events after an L2 flush (a 256 MB
    write, > 126 MB L2), median of 7.  Reported for context only."""
    import torch

    import paper_2410_06770_b200 as g
    from paper_2410_06770_b200.device import dgett_device, sgett_device
    from paper_2410_06770_b200.workloads import CONFIGS

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    out = {}
    for name in ("c1", "c3", "c4", "c5"):
        w = CONFIGS[name]
        a, b, c = w.buffers()
        ta, tb, tc = (torch.from_numpy(x).to(dev) for x in (a, b, c))
        fn = dgett_device if w.dtype == "d" else sgett_device
        pos, kw = w.args(ta, tb, tc)
        for _ in range(3):
            assert fn(*pos, **kw) == []
        times = []
        for _ in range(7):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(*pos, **kw)
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        # roofline of the config: the larger of the HBM time for its algorithmic
        # bytes and the tensor time for its FLOPs (FP64 DMMA peak; fp32 at a
        # third of the measured tf32 MMA issue rate, 3xTF32)
        t_hbm = w.alg_bytes / (hbm_gbs() * 1e9)
        t_tc = w.flops / ((FP64_PEAK_TFLOPS if w.dtype == "d" else TF32X3_PEAK_TFLOPS) * 1e12)
        bound = "hbm" if t_hbm > t_tc else "tensor"
        out[name] = {"gflops": round(w.flops / (ms * 1e-3) / 1e9, 2), "ms": round(ms, 4),
                     "dtype": "f64" if w.dtype == "d" else "f32", "kernel": g.last_kernel(),
                     "l2": "flushed before each call",
                     "roofline": {"bound": bound, "floor_ms": round(max(t_hbm, t_tc) * 1e3, 4),
                                  "frac": round(max(t_hbm, t_tc) / (ms * 1e-3), 4)}}
        del ta, tb, tc
    del flush
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other_configs timings")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
