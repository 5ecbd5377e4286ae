"""Summarise one kernel of an ncu report (--page raw) into a small JSON file
for profiles/.  Usage:
    python tools/ncu_summary.py REPORT.ncu-rep OUT.json [note...]
The summary records the sha256 prefix of the libgett_b200.so in the tree
(the build the capture must have been taken on; bench.py reports the capture's
traffic only when it matches the library it runs) and algorithmic figures when
GETT_ALG_BYTES / GETT_ALG_FLOPS are set.
"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2410_06770_b200",
                   "libgett_b200.so")

KEYS = {
    "gpu__time_duration.sum": "gpu_time",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_active_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "s": 1.0}


def main():
    args = sys.argv[1:]
    kfilter = []
    if args and args[0].startswith("--kernel="):
        kfilter = ["-k", "regex:" + args.pop(0).split("=", 1)[1]]
    rep, out = args[0], args[1]
    note = " ".join(args[2:])
    raw = subprocess.run(["ncu", "-i", rep] + kfilter + ["--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {"report": rep.split("/")[-1], "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None,
         "note": note}
    stalls = {}
    for i, name in enumerate(h):
        try:
            x = float(v[i].replace(",", ""))
        except ValueError:
            continue
        if name in KEYS:
            key = KEYS[name]
            if u[i] in SCALE:
                x *= SCALE[u[i]]
                key += "_s" if u[i] in ("ms", "us", "ns", "s") else ""
            d[key] = x
        if name.startswith("smsp__average_warps_issue_stalled_") and x > 0.1:
            stalls[name.split("stalled_")[1].split("_per")[0]] = round(x, 3)
    if "dram_bytes_read" in d:
        d["dram_bytes_per_launch"] = d["dram_bytes_read"] + d.get("dram_bytes_write", 0.0)
    with open(LIB, "rb") as f:
        d["so_sha16"] = hashlib.sha256(f.read()).hexdigest()[:16]
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.argv = sys.argv[:1]
    import bench  # noqa: E402  (only for src_sha16; bench imports no GPU code at import time)

    d["src_sha16"] = bench.src_sha16()
    for env, key in (("GETT_ALG_BYTES", "algorithmic_bytes_per_launch"), ("GETT_ALG_FLOPS", "algorithmic_flops_per_launch")):
        if os.environ.get(env):
            d[key] = float(os.environ[env])
    if d.get("algorithmic_bytes_per_launch") and d.get("dram_bytes_per_launch"):
        d["traffic_over_algorithmic"] = round(d["dram_bytes_per_launch"] / d["algorithmic_bytes_per_launch"], 3)
    d["top_stalls_per_issue"] = stalls
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
