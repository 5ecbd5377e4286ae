"""Generate the .tns golden fixtures by running the REFERENCE's tensorfile and
CLI (gett.tensorfile / gett.cli, /root/reference/pkg/src) in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_tns_golden.py

Outputs (small, committed) under tests/golden/tns/:
  <name>.tns       files written by the reference writer (s/d/c/z, ranks 0-3,
                   negative increments, offsets, special values)
  values.npz       the buffers those files were written from
  malformed.json   malformed file texts and the reference reader's error
                   message for each (path shown as "{path}")
  cli_run.json     `gett run` invocations on reference-written inputs, with the
                   reference CLI's exit code, stderr and output file text
/root/reference is never read at test time.
"""
from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "tns")

from gett import cli  # noqa: E402  (the reference)
from gett.layout import TensorView  # noqa: E402
from gett.tensorfile import TensorFile, TensorFileError, read_tensor, write_tensor  # noqa: E402

DT = {"s": np.float32, "d": np.float64, "c": np.complex64, "z": np.complex128}


def buffers():
    rng = np.random.default_rng(11)
    cases = {}
    for tag in "sdcz":
        n = 13
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-30, 30, n)
        if tag in "cz":
            x = x + 1j * rng.standard_normal(n) * 1e-5
        x = x.astype(DT[tag])
        cases[f"r2_{tag}"] = (tag, TensorView(2, (3, 4), (1, 3), 1, n), x)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-310, 5e-324, 1.7976931348623157e308,
                        0.1, 1 / 3.0], dtype=np.float64)
    cases["special_d"] = ("d", TensorView(1, (10,), (1,), 0, 10), special)
    cases["special_s"] = ("s", TensorView(1, (10,), (1,), 0, 10), special.astype(np.float32))
    cases["rank0_d"] = ("d", TensorView(0, (), (), 2, 3), np.array([1.5, -2.25, 3e100]))
    cases["neg_inc_z"] = ("z", TensorView(2, (2, 3), (-1, -2), 5, 6),
                          (np.arange(6) + 1j * np.arange(6, 0, -1)).astype(np.complex128))
    cases["empty_d"] = ("d", TensorView(2, (0, 4), (1, 1), 0, 0), np.zeros(0))
    cases["int3_d"] = ("d", TensorView(3, (2, 3, 2), (6, 2, 1), 0, 12),
                       rng.integers(-9, 9, 12).astype(np.float64))
    return cases


MALFORMED = {
    "bad_magic": "GETT-TENSOR 2\ndtype: d\nrank: 0\nextents:\nincrements:\noffset: 0\nbuffer: 1\n1\n",
    "empty_file": "",
    "bad_dtype": "GETT-TENSOR 1\ndtype: q\nrank: 0\nextents:\nincrements:\noffset: 0\nbuffer: 1\n1\n",
    "missing_key": "GETT-TENSOR 1\ndtype: d\nrank: 1\n",
    "wrong_key": "GETT-TENSOR 1\ndtype: d\nrnak: 1\nextents: 2\nincrements: 1\noffset: 0\nbuffer: 2\n1 2\n",
    "rank_not_int": "GETT-TENSOR 1\ndtype: d\nrank: x\nextents: 2\nincrements: 1\noffset: 0\nbuffer: 2\n1 2\n",
    "rank_two_ints": "GETT-TENSOR 1\ndtype: d\nrank: 1 2\nextents: 2\nincrements: 1\noffset: 0\nbuffer: 2\n1 2\n",
    "extent_count": "GETT-TENSOR 1\ndtype: d\nrank: 2\nextents: 2\nincrements: 1 2\noffset: 0\nbuffer: 4\n1 2 3 4\n",
    "inc_count": "GETT-TENSOR 1\ndtype: d\nrank: 2\nextents: 2 2\nincrements: 1\noffset: 0\nbuffer: 4\n1 2 3 4\n",
    "neg_offset": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 2\nincrements: 1\noffset: -1\nbuffer: 2\n1 2\n",
    "neg_rank": "GETT-TENSOR 1\ndtype: d\nrank: -1\nextents:\nincrements:\noffset: 0\nbuffer: 2\n1 2\n",
    "bad_value": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 3\nincrements: 1\noffset: 0\nbuffer: 3\n1 2\nthree\n",
    "too_many": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 2\nincrements: 1\noffset: 0\nbuffer: 2\n1\n2 3\n4\n",
    "too_few": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 3\nincrements: 1\noffset: 0\nbuffer: 3\n1 2\n\n",
    "complex_odd": "GETT-TENSOR 1\ndtype: z\nrank: 1\nextents: 1\nincrements: 1\noffset: 0\nbuffer: 1\n1\n",
    "neg_extent": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: -2\nincrements: 1\noffset: 0\nbuffer: 2\n1 2\n",
    "out_of_bounds": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 3\nincrements: 1\noffset: 0\nbuffer: 2\n1 2\n",
    "neg_stride_oob": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 3\nincrements: -1\noffset: 1\nbuffer: 3\n1 2 3\n",
    "underscore_ok": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 2\nincrements: 1\noffset: 0\nbuffer: 2\n1_0 2\n",
    "bad_then_surplus": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 1\nincrements: 1\noffset: 0\nbuffer: 1\nx 2\n",
    "surplus_then_bad": "GETT-TENSOR 1\ndtype: d\nrank: 1\nextents: 1\nincrements: 1\noffset: 0\nbuffer: 1\n1 x\n",
}

RUNS = [
    # name, a dims/incs, b dims/incs, dtype, extra CLI args
    ("matmul_d", ((3, 4), (1, 3)), ((4, 2), (1, 4)), "d",
     ["--conts", "1", "--cont-a", "1", "--cont-b", "0", "--perm", "0,1"]),
    ("perm_out_inc_d", ((2, 3, 4), (1, 2, 6)), ((4, 5), (5, 1)), "d",
     ["--conts", "1", "--cont-a", "2", "--cont-b", "0", "--perm", "2,0,1", "--out-inc", "1,5,10"]),
    ("outer_s", ((3,), (1,)), ((2,), (1,)), "s", ["--perm", "1,0"]),
    ("complex_z", ((2, 2), (1, 2)), ((2, 3), (1, 2)), "z",
     ["--conts", "1", "--cont-a", "1", "--cont-b", "0", "--perm", "0,1"]),
    ("bad_spec", ((3, 4), (1, 3)), ((4, 2), (1, 4)), "d",
     ["--conts", "1", "--cont-a", "5", "--cont-b", "0", "--perm", "0,1"]),
    ("extent_mismatch", ((3, 4), (1, 3)), ((5, 2), (1, 5)), "d",
     ["--conts", "1", "--cont-a", "1", "--cont-b", "0", "--perm", "0,1"]),
    ("out_ext_check", ((3, 4), (1, 3)), ((4, 2), (1, 4)), "d",
     ["--conts", "1", "--cont-a", "1", "--cont-b", "0", "--perm", "0,1", "--out-ext", "3,3"]),
    ("pairs_mismatch", ((3, 4), (1, 3)), ((4, 2), (1, 4)), "d",
     ["--conts", "2", "--cont-a", "1", "--cont-b", "0", "--perm", "0,1"]),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    vals = {}
    for name, (tag, view, data) in buffers().items():
        write_tensor(os.path.join(OUT, name + ".tns"), TensorFile(tag, view, data))
        vals[name] = data
    np.savez(os.path.join(OUT, "values.npz"), **vals)

    bad = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in MALFORMED.items():
            p = os.path.join(tmp, name + ".tns")
            with open(p, "w") as f:
                f.write(text)
            try:
                t = read_tensor(p)
                bad[name] = {"text": text, "error": None, "data": [repr(float(v)) for v in
                                                                   np.asarray(t.data).ravel()]}
            except TensorFileError as e:
                bad[name] = {"text": text, "error": str(e).replace(p, "{path}"), "line": e.line}
    with open(os.path.join(OUT, "malformed.json"), "w") as f:
        json.dump(bad, f, indent=1, sort_keys=True)

    runs = {}
    rng = np.random.default_rng(5)
    with tempfile.TemporaryDirectory() as tmp:
        for name, (ea, ia), (eb, ib), tag, extra in RUNS:
            def mk(ext, inc):
                n = 1 + sum((e - 1) * abs(i) for e, i in zip(ext, inc))
                x = rng.integers(-5, 6, n).astype(np.float64)
                if tag in "cz":
                    x = x + 1j * rng.integers(-5, 6, n)
                return TensorFile(tag, TensorView(len(ext), ext, inc, 0, n), x.astype(DT[tag]))
            ta, tb = mk(ea, ia), mk(eb, ib)
            pa, pb, pc = (os.path.join(tmp, f"{name}_{x}.tns") for x in "abc")
            write_tensor(pa, ta)
            write_tensor(pb, tb)
            err = io.StringIO()
            with contextlib.redirect_stderr(err):
                rc = cli.main(["run", pa, pb, pc] + extra)
            out = open(pc).read() if os.path.exists(pc) else None
            runs[name] = {"a": open(pa).read(), "b": open(pb).read(), "args": extra, "rc": rc,
                          "stderr": err.getvalue().replace(tmp + "/", "{dir}/"), "out": out}
    with open(os.path.join(OUT, "cli_run.json"), "w") as f:
        json.dump(runs, f, indent=1, sort_keys=True)
    print(f"{len(vals)} files, {len(bad)} malformed cases, {len(runs)} CLI runs -> {OUT}")


if __name__ == "__main__":
    main()
