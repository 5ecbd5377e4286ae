"""Loaders for the golden fixtures made by tests/golden/make_golden.py from
the reference implementation.  Inputs are regenerated from the stored seeds."""
from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def view_offsets(ext, inc, off):
    """Absolute offsets of a view, dimension 0 fastest (layout.py:128-140)."""
    if any(e == 0 for e in ext):
        return np.empty(0, np.int64)
    offs = np.full(1, off, dtype=np.int64)
    for e, i in zip(ext, inc):
        steps = np.int64(i) * np.arange(e, dtype=np.int64)
        offs = (offs[np.newaxis, :] + steps[:, np.newaxis]).ravel()
    return offs


class SuiteCase:
    def __init__(self, d, want):
        self.__dict__.update(d)
        self.want = want

    @property
    def np_dtype(self):
        return {"d": np.float64, "s": np.float32, "z": np.complex128, "c": np.complex64}[self.dtype]

    def buffers(self):
        rng = np.random.default_rng(self.data_seed)
        dt = self.np_dtype

        def draw(n):
            if self.dtype in "cz":
                if self.data == "int":
                    re, im = rng.integers(-4, 5, n), rng.integers(-4, 5, n)
                else:
                    re, im = rng.uniform(-1.0, 1.0, n), rng.uniform(-1.0, 1.0, n)
                return (re + 1j * im).astype(dt)
            if self.data == "int":
                return rng.integers(-4, 5, n).astype(dt)
            return rng.uniform(-1.0, 1.0, n).astype(dt)

        return draw(self.a["len"]), draw(self.b["len"]), draw(self.c["len"])

    def args(self, a, b, c):
        pos = (self.a["rank"], tuple(self.a["ext"]), tuple(self.a["inc"]), a,
               self.b["rank"], tuple(self.b["ext"]), tuple(self.b["inc"]), b,
               self.conts, tuple(self.cont_a), tuple(self.cont_b), tuple(self.perm),
               tuple(self.c["inc"]), c)
        kw = dict(offset_a=self.a["off"], offset_b=self.b["off"], offset_c=self.c["off"])
        return pos, kw

    def c_offsets(self):
        return view_offsets(self.c["ext"], self.c["inc"], self.c["off"])

    @property
    def id(self):
        return f"{self.category}/{self.seed}/{self.dtype}-{self.data}"


def load_suite():
    z = np.load(os.path.join(GOLDEN, "suite.npz"))
    cases = json.loads(str(z["cases"]))
    out = []
    for d in cases:
        arr = z[d["store"]][d["out_start"]:d["out_start"] + d["out_len"]]
        real = {"d": np.float64, "s": np.float32, "z": np.float64, "c": np.float32}[d["dtype"]]
        want = np.ascontiguousarray(arr.astype(real))
        if d["dtype"] in "cz":
            want = want.view(np.complex128 if d["dtype"] == "z" else np.complex64)
        out.append(SuiteCase(d, want))
    return out


def load_configs():
    z = np.load(os.path.join(GOLDEN, "configs.npz"))
    meta = json.loads(str(z["meta"]))
    return {k: (v, z[k]) for k, v in meta.items()}


def load_validation():
    with open(os.path.join(GOLDEN, "validation.json")) as f:
        cases = json.load(f)
    for c in cases:
        args = list(c["args"])
        for i in (3, 7, 13):
            args[i] = np.zeros(args[i]["zeros"])
        for i in (1, 2, 5, 6, 9, 10, 11, 12):
            args[i] = tuple(args[i])
        c["args"] = tuple(args)
    return cases


def load_zero_view():
    with open(os.path.join(GOLDEN, "zero_view.json")) as f:
        return json.load(f)


def sliced_workload(meta):
    """The Workload slice a configs.npz entry was computed on."""
    from dataclasses import replace

    from paper_2410_06770_b200.workloads import CONFIGS

    w = CONFIGS[meta["workload"]]
    return replace(w, ext_a=tuple(meta["ext_a"]), off_a=meta["off_a"], ext_b=tuple(meta["ext_b"]),
                   off_b=meta["off_b"], off_c=meta["off_c"])
