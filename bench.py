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
  * N > 1: one process per GPU.  Launched by torchrun (the driver), or — when
    WORLD_SIZE is unset — bench.py re-executes itself under
    torch.distributed.run with N ranks.  The free mode A0 (= C mode 0) is split
    into N row slabs, one per rank, no collective -> total work
    fixed.  N > 1 also times c5 as split-K across the ranks with one NCCL
    reduce (``splitk_c5``).
  * --impl reference: the reference's own implementation — the unmodified
    numba ``gett.kernel.dgett`` from baseline/_ref, through its public API —
    on the box's host cores: one process per core, each a disjoint row slab of
    c2 (a free-mode slice, bitwise equal to the same rows of a full run).  This
    process never imports the package (libgett_b200.so is not mapped).
"""
from __future__ import annotations

import argparse
import hashlib
import importlib.util
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
# the pip --target install puts the package at baseline/_ref/gett; a copied
# source tree has it at baseline/_ref/pkg/src/gett
REF_SRC = next((d for d in (os.path.join(ROOT, "baseline", "_ref"),
                            os.path.join(ROOT, "baseline", "_ref", "pkg", "src"))
                if os.path.isdir(os.path.join(d, "gett"))),
               os.path.join(ROOT, "baseline", "_ref"))
LIB_PATH = os.path.join(ROOT, "paper_2410_06770_b200", "libgett_b200.so")


def _load_workloads():
    """paper_2410_06770_b200/workloads.py by path, WITHOUT importing the
    package (whose __init__ maps libgett_b200.so): the reference arm must
    not load our library."""
    name = "_gett_bench_workloads"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(
        name, os.path.join(ROOT, "paper_2410_06770_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


W = _load_workloads()
C2 = W.C2

METRIC = "xGETT GFLOP/s (2·|C|·|K|/s), DGETT c2 4096^3 strided GEMM-shaped subtensor"
WORKLOAD = ("c2: DGETT A[4096,4096] view of f64 [4100,4224], B[4096,4096] view of [4096,4160], "
            "contract A1-B0, identity PERM, C += into [4096,4200] parent (BASELINE configs[1])")
FP64_PEAK_TFLOPS = 37.116  # best DMMA loop, profiles/r02/peaks/peaks.jsonl (SM clock 1965 MHz: clocks.csv)
FP64_PEAK_SRC = ("measured FP64 DMMA peak (tools/peaks.cu via tools/peaks_with_clocks.sh, "
                 "profiles/r02/peaks/{peaks.jsonl,clocks.csv}); MEASURED_PEAKS.json has no FP64 figure")


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def config_obj(n):
    """The `config` object — identical in both arms for the same N."""
    return {"workload": WORKLOAD, "global_flops_per_step": C2.flops,
            "parallelism": (f"free-mode A0 split into {n} row slab(s), one per GPU, no collective"
                            if n > 1 else "1 GPU"),
            "l2": "inputs larger than L2 (A+B+C spans 410 MB > 126 MB)"}


def shard(world, rank):
    """This rank's slab of c2 on the native multi-device schedule
    (gett_multi_schedule: the partition one gett_dgett_multi call runs)."""
    if world == 1:
        return C2, C2.ext_a[0]
    from paper_2410_06770_b200.shard import schedule

    class _Len:
        def __init__(self, n):
            self.n = n

        def __len__(self):
            return self.n

    pos, kw = C2.args(_Len(C2.len_a), _Len(C2.len_b), _Len(C2.len_c))
    s = schedule(pos, kw, world)
    assert s.strategy == "slabs", s
    lo, hi = s.range(rank)
    return C2.slice_free(s.owner, s.dim, lo, hi), hi - lo


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


def lib_sha16():
    try:
        with open(LIB_PATH, "rb") as f:
            return hashlib.sha256(f.read()).hexdigest()[:16]
    except OSError:
        return None


def src_sha16():
    """sha256 prefix of the native sources the library is built from (nvcc's
    output bytes differ between identical builds, so a capture is matched to
    a build by its sources when the binary hash differs)."""
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2410_06770_b200", "csrc")
    files = sorted(os.path.join(csrc, f) for f in os.listdir(csrc)
                   if f.endswith((".cu", ".cuh", ".hpp", ".cpp")) or f == "Makefile")
    files.append(os.path.join(ROOT, "include", "gett_b200.h"))
    for fn in files:
        h.update(os.path.basename(fn).encode())
        with open(fn, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def traffic_from_profiles():
    """dram bytes per launch of the DGETT kernel from the committed ncu capture
    — only when the capture was taken on THIS build of libgett_b200.so (the
    capture records the library's sha256 prefix, and the sha256 prefix of its
    sources); else None."""
    p = os.path.join(ROOT, "profiles", "ncu_dgett_c2.json")
    if not os.path.exists(p):
        return None, "no capture"
    with open(p) as f:
        d = json.load(f)
    if d.get("so_sha16") and d["so_sha16"] == lib_sha16():
        return d.get("dram_bytes_per_launch"), f"profiles/ncu_dgett_c2.json (same binary, so_sha16 {d['so_sha16']})"
    if d.get("src_sha16") and d["src_sha16"] == src_sha16():
        return d.get("dram_bytes_per_launch"), (f"profiles/ncu_dgett_c2.json (same sources, src_sha16 "
                                                f"{d['src_sha16']}; binary rebuilt)")
    return None, f"capture so/src {d.get('so_sha16')}/{d.get('src_sha16')} != this build {lib_sha16()}/{src_sha16()}"


# ---------------------------------------------------------------------------
# The reference arm: the unmodified numba reference, fanned out over cores
# ---------------------------------------------------------------------------

_REF = {}


def _ref_init():
    """Import the reference from baseline/_ref and warm its JIT with one tiny
    call (bench_sweep.py:61 warms the same way)."""
    if "dgett" in _REF:
        return _REF["dgett"]
    if not os.path.isdir(os.path.join(REF_SRC, "gett")):
        raise FileNotFoundError(f"{REF_SRC}/gett is missing (baseline/_ref not installed)")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "gett_ref_numba_cache"))
    sys.path.insert(0, REF_SRC)
    from gett.kernel import dgett  # the reference's public entry (kernel.py:166-184)

    a = np.ones(8)
    c = np.zeros(1)
    assert dgett(1, (8,), (1,), a, 1, (8,), (1,), a, 1, (0,), (0,), (), (), c) == []
    _REF["dgett"] = dgett
    return dgett


def _ref_rows(job):
    """Worker: rows [lo, hi) of c2 through the reference dgett; seconds."""
    lo, hi = job
    dgett = _REF["dgett"]
    a, b, c = _REF["bufs"]
    w = C2.slice_free("A", 0, lo, hi)
    pos, kw = w.args(a, b, c)
    t0 = time.perf_counter()
    errs = dgett(*pos, **kw)
    dt = time.perf_counter() - t0
    assert errs == [], errs
    return dt


class RefPool:
    """One forked process per host core, each holding the reference's JIT'd
    kernel; a step gives every process its own row slab of c2 and takes the
    wall time until the last one finishes."""

    def __init__(self, procs):
        import multiprocessing as mp

        _ref_init()
        _REF["bufs"] = C2.buffers()  # shared copy-on-write with the forked workers
        self.procs = procs
        self.pool = mp.get_context("fork").Pool(procs)
        self.pool.map(_ref_rows, [(0, 1)] * procs)  # fault the pages in

    def step(self, rows_per_proc):
        jobs = []
        row = 0
        for _ in range(self.procs):
            jobs.append((row % 4096, row % 4096 + rows_per_proc))
            row += rows_per_proc
        t0 = time.perf_counter()
        self.pool.map(_ref_rows, jobs, chunksize=1)
        dt = time.perf_counter() - t0
        return dt, self.procs * rows_per_proc * 2 * 4096 * 4096

    def close(self):
        self.pool.close()
        self.pool.join()


def reference_measure(steps, warmup, target_s):
    """(GFLOP/s, seconds per step, rows per step, processes) of the reference
    fanned out over every host core."""
    procs = len(os.sched_getaffinity(0))
    pool = RefPool(procs)
    try:
        dt, _ = pool.step(1)
        rows = max(1, min(4096 // procs, int(target_s / max(dt, 1e-3))))
        for _ in range(warmup):
            pool.step(rows)
        tt, fl = 0.0, 0
        for _ in range(steps):
            dt, f = pool.step(rows)
            tt += dt
            fl += f
    finally:
        pool.close()
    return fl / tt / 1e9, tt / steps, rows * procs, procs


def ref_single_core(rows):
    """The reference as shipped: one process, one core (SURVEY §8d plan)."""
    _ref_init()
    if "bufs" not in _REF:
        _REF["bufs"] = C2.buffers()
    dt = _ref_rows((0, rows))
    return rows * 2 * 4096 * 4096 / dt / 1e9, dt


def run_reference(args):
    rank, _, world = env_rank()
    if rank != 0:
        return
    n = max(args.gpus, world)
    kind = "reference"
    try:
        _ref_init()  # raises when baseline/_ref is not installed
        gfl, s_step, rows, procs = reference_measure(args.steps, args.warmup, args.ref_step_s)
        sample = (f"{rows} of 4096 rows of c2 per step ({rows // procs} per process; free-mode slices "
                  f"of A0, bitwise equal to the same rows of a full run), unmodified numba "
                  f"gett.kernel.dgett from baseline/_ref, {procs} processes x 1 thread")
    except (FileNotFoundError, ImportError) as exc:
        # the installed reference did not travel: time the oracle port (the
        # reference loop restated in C, oracle/) on all host threads instead
        print(f"bench.py: reference not importable ({exc}); timing the oracle port", file=sys.stderr)
        kind = "port"
        procs = len(os.sched_getaffinity(0))
        rows = calibrate_port_rows(procs, args.ref_step_s)
        for _ in range(args.warmup):
            port_sample(rows, procs)
        t_all, f_all = 0.0, 0
        for _ in range(args.steps):
            dt, fl = port_sample(rows, procs)
            t_all, f_all = t_all + dt, f_all + fl
        gfl, s_step = f_all / t_all / 1e9, t_all / args.steps
        sample = (f"{rows} of 4096 rows of c2 per step, oracle/gett_oracle.c (the reference loop restated "
                  f"in C; baseline/_ref missing), {procs} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gfl, 4), "unit": "GFLOP/s",
        "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * s_step, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_obj(n),
        "cpu_baseline": {"value": round(gfl, 4), "unit": "GFLOP/s", "cores": procs,
                         "kind": kind, "sample": sample},
        "e2e": {"value": round(gfl, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if args.json_out:
        with open(args.json_out, "w") as f:
            json.dump(line, f)
    print(json.dumps(line), flush=True)


def cpu_baselines():
    """Our arm's cpu_baseline: the reference fan-out (a fresh process, so this
    CUDA process never forks), plus the single-core reference and the C port
    of the oracle beside it."""
    out = {}
    tmp = os.path.join("/tmp", f"gett_ref_{os.getpid()}.json")
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "MASTER_ADDR",
                        "MASTER_PORT", "TORCHELASTIC_RUN_ID", "GROUP_RANK")}
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference",
                        "--steps", "3", "--warmup", "1", "--ref-step-s", "3", "--json-out", tmp],
                       env=env, capture_output=True, text=True, timeout=900)
    if r.returncode == 0 and os.path.exists(tmp):
        with open(tmp) as f:
            out["cpu_baseline"] = json.load(f)["cpu_baseline"]
        os.unlink(tmp)
    else:
        out["cpu_baseline"] = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                               "sample": "failed: " + (r.stderr or "")[-300:]}
    extra = []
    try:
        code = ("import sys, json; sys.argv=['bench.py']; import bench; "
                "print(json.dumps(bench.ref_single_core(8)))")
        r1 = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                            text=True, timeout=600)
        g1, dt1 = json.loads(r1.stdout.strip().splitlines()[-1])
        extra.append({"value": round(g1, 4), "unit": "GFLOP/s", "cores": 1, "kind": "reference",
                      "sample": f"8 of 4096 rows of c2 ({dt1:.1f} s), the reference as shipped "
                                "(numba, single-threaded), 1 process"})
    except Exception as e:  # noqa: BLE001 — a missing figure is reported, not fatal
        extra.append({"kind": "reference", "cores": 1, "value": None, "sample": f"failed: {e}"})
    threads = len(os.sched_getaffinity(0))
    rows = calibrate_port_rows(threads, 5.0)
    dt, fl = port_sample(rows, threads)
    extra.append({"value": round(fl / dt / 1e9, 4), "unit": "GFLOP/s", "cores": threads,
                  "kind": "port", "sample": f"{rows} of 4096 rows of c2 ({dt:.1f} s), "
                                            f"oracle/gett_oracle.c (C restatement), {threads} threads"})
    out["cpu_baseline_more"] = extra
    return out


def port_sample(rows, threads):
    """Oracle port (reference loop restated in C) on `rows` rows of c2."""
    from oracle import oracle

    w = C2.slice_free("A", 0, 0, rows)
    if not hasattr(port_sample, "bufs"):
        port_sample.bufs = C2.buffers()
    a, b, c = port_sample.bufs
    pos, kw = w.args(a, b, c)
    t0 = time.perf_counter()
    oracle.oracle_dgett(*pos, **kw, threads=threads)
    return time.perf_counter() - t0, w.flops


def calibrate_port_rows(threads, target_s):
    dt, fl = port_sample(threads, threads)  # one row per thread
    rate = fl / max(dt, 1e-6)
    rows = int(target_s * rate / (2 * 4096 * 4096))
    return max(threads, min(4096, rows))


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch

    sys.path.insert(0, ROOT)
    import paper_2410_06770_b200 as g
    from paper_2410_06770_b200.device import dgett_device

    rank, local, world = env_rank()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # host-side barriers for the sections where one rank drives every GPU:
        # an NCCL barrier would leave a spinning kernel on the waiting ranks'
        # GPUs, time-slicing against rank 0's work there
        try:
            cpu_group = dist.new_group(backend="gloo")
        except Exception as exc:  # noqa: BLE001  (no gloo transport: fall back to NCCL barriers)
            print(f"bench.py: gloo side group unavailable ({exc}); NCCL barriers", file=sys.stderr)
            cpu_group = None
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
    k_ms = ms / args.steps  # one DGETT launch per step at this size
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
    del pa, pb, pc

    splitk = None
    e2e_ranks = None
    if dist:
        t = torch.tensor([ms, e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1])
        t = torch.tensor([launches, h2d, d2h], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        launches, h2d, d2h = (int(x) for x in t.tolist())
        del ta, tb, tc
        torch.cuda.empty_cache()
        splitk = splitk_c5(dist, dev, args)
        # e2e of the whole job through ONE drop-in call driving all N GPUs
        # (gett_dgett_multi: slabs per GPU, B exchanged over NVLink); rank 0
        # calls, the other ranks wait
        e2e_ranks = e2e_s
        torch.cuda.synchronize()
        dist.barrier(group=cpu_group)
        if rank == 0:
            fa, fb, fc = (torch.from_numpy(x).pin_memory().numpy() for x in (a, b, c))
            fpos, fkw = C2.args(fa, fb, fc)
            devs = list(range(world))
            assert g.dgett(*fpos, **fkw, devices=devs) == []
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                assert g.dgett(*fpos, **fkw, devices=devs) == []
            e2e_s = (time.perf_counter() - t0) / e2e_steps
            multi_sched = g.last_multi()
            del fa, fb, fc
        dist.barrier(group=cpu_group)
    total_flops = C2.flops  # all ranks together process the whole c2 per step
    value = total_flops * args.steps / (ms * 1e-3) / 1e9
    e2e_value = total_flops / e2e_s / 1e9
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    if dist:
        h2d = 8 * (spans(C2.ext_a, C2.inc_a) + spans(C2.ext_b, C2.inc_b) + spans(C2.ext_c, C2.inc_c))
        d2h = 8 * spans(C2.ext_c, C2.inc_c)
        e2e_value = total_flops / e2e_s / 1e9
    achieved = w.flops / (k_ms * 1e-3) / 1e12
    traffic, traffic_src = traffic_from_profiles()
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform[-1,1], SURVEY §8d)",
        "config": config_obj(world),
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "achieved": round(achieved, 3),
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": FP64_PEAK_SRC, "kernel": kname, "so_sha16": lib_sha16(),
                     "src_sha16": src_sha16()},
        "clocks": clocks.summary(),
        "e2e": {"value": round(e2e_value, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "how": ("dgett() on pinned numpy buffers: H2D spans + kernel + D2H C span, wall "
                        "clock" + (f"; ONE call with devices=range({world}) from rank 0 "
                                   f"({multi_sched})" if world > 1 else ""))},
    }
    if splitk:
        line["splitk_c5"] = splitk
    if e2e_ranks is not None:
        line["e2e_per_rank_slabs"] = {
            "value": round(total_flops / e2e_ranks / 1e9, 2), "unit": "GFLOP/s",
            "how": f"each of {world} ranks dgett() on its own slab from its own host buffers, max over ranks"}
    if world == 1 and not args.no_configs:
        line["other_configs"] = other_configs(dev)
    if world == 1 and not args.no_cpu_baseline:
        line.update(cpu_baselines())
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def splitk_c5(dist, dev, args):
    """c5 (SGETT, 73,728 outputs — too few to split by output) as split-K across
    the ranks: each rank contracts its K slice on its GPU, one NCCL reduce lands
    the partial sums on rank 0, which adds them into C (shard.splitk_device).
    Device-timed with CUDA events, max over ranks."""
    import torch

    from paper_2410_06770_b200.shard import splitk_device

    w = W.C5
    a, b, c = w.buffers()
    ta, tb, tc = (torch.from_numpy(x).to(dev) for x in (a, b, c))
    pos, kw = w.args(ta, tb, tc)
    for _ in range(3):
        assert splitk_device("s", pos, kw) == []
    torch.cuda.synchronize()
    dist.barrier()
    n = max(5, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        splitk_device("s", pos, kw)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / n], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    return {"gflops": round(w.flops / (ms * 1e-3) / 1e9, 2), "ms": round(ms, 4),
            "how": "K split over ranks, ncclReduce(sum) of the 73,728-float partial to rank 0, "
                   "owner adds into C; CUDA events, max over ranks, L2 not flushed"}


# fp32 via 3xTF32: a third of the tf32 MMA rate measured by tools/mma_rate.cu
# (2046 MAC/clk/SM x 148 SMs x 1.965 GHz; profiles/r02/peaks/mma_rate.jsonl)
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
    per call with CUDA events.  Configs whose operands exceed the 126 MB L2
    (c3, c4) run back to back; c5 (107 MB) rotates over enough copies of its
    operands to exceed twice the L2, back to back (a single short call timed
    alone after an L2 flush is quantised by the event clock); c1 (0.7 MB,
    latency-bound) is timed alone after a 256 MB L2 flush, median of 21.
    Reported for context only."""
    import torch

    import paper_2410_06770_b200 as g
    from paper_2410_06770_b200.device import dgett_device, sgett_device

    L2 = 126 << 20
    out = {}
    for name in ("c1", "c3", "c4", "c5"):
        w = W.CONFIGS[name]
        a, b, c = w.buffers()
        fn = dgett_device if w.dtype == "d" else sgett_device
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if w.alg_bytes < (1 << 20):
            ta, tb, tc = (torch.from_numpy(x).to(dev) for x in (a, b, c))
            pos, kw = w.args(ta, tb, tc)
            for _ in range(3):
                assert fn(*pos, **kw) == []
            flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
            times = []
            for _ in range(21):
                flush.zero_()
                e0.record()
                fn(*pos, **kw)
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            ms = float(np.median(times))
            how = "timed alone after an L2 flush (256 MB write), median of 21"
            del flush
        else:
            copies = 1 if w.alg_bytes > L2 else -(-2 * L2 // w.alg_bytes)
            sets = []
            for _ in range(copies):
                ta, tb, tc = (torch.from_numpy(x).to(dev) for x in (a, b, c))
                sets.append(w.args(ta, tb, tc))
            for pos, kw in sets:
                assert fn(*pos, **kw) == []
            # (c4: 5 calls of 6.4 ms; c3: 20 calls of 0.76 ms; c5: 60 per operand copy)
            n = max(5, 3 * copies) if w.flops > 1e11 else (20 * copies if w.flops > 1e10 else 60 * copies)
            torch.cuda.synchronize()
            e0.record()
            for i in range(n):
                pos, kw = sets[i % copies]
                fn(*pos, **kw)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / n
            how = ("back to back, operands larger than L2" if copies == 1 else
                   f"back to back over {copies} copies of the operands (> 2x L2), {n} calls")
            del sets
        # roofline of the config: the larger of the HBM time for its algorithmic
        # bytes and the tensor time for its FLOPs (FP64 DMMA peak; fp32 at a
        # third of the measured tf32 MMA issue rate, 3xTF32)
        t_hbm = w.alg_bytes / (hbm_gbs() * 1e9)
        t_tc = w.flops / ((FP64_PEAK_TFLOPS if w.dtype == "d" else TF32X3_PEAK_TFLOPS) * 1e12)
        bound = "hbm" if t_hbm > t_tc else "tensor"
        out[name] = {"gflops": round(w.flops / (ms * 1e-3) / 1e9, 2), "ms": round(ms, 4),
                     "dtype": "f64" if w.dtype == "d" else "f32", "kernel": g.last_kernel(),
                     "l2": how,
                     "roofline": {"bound": bound, "floor_ms": round(max(t_hbm, t_tc) * 1e3, 4),
                                  "frac": round(max(t_hbm, t_tc) / (ms * 1e-3), 4)}}
    torch.cuda.empty_cache()
    return out


def launch_ranks(args):
    """--gpus N without a torchrun environment: re-execute this script under
    torch.distributed.run with N ranks (one per GPU) and return its status.
    Fails loudly when the node has fewer than N GPUs."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, found {have}",
              file=sys.stderr, flush=True)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other_configs timings")
    ap.add_argument("--ref-step-s", type=float, default=1.5,
                    help="reference arm: target seconds of CPU work per step")
    ap.add_argument("--json-out", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        run_reference(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args)
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
