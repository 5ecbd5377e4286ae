"""The BASELINE.json configurations c1..c5 as concrete, seeded xGETT calls.

Each workload is the literal argument list of one reference xGETT call
(kernel.py:158-184 order) over synthetic parent buffers.  The concrete
extents/increments/parents follow SURVEY.md §8d (BASELINE.json configs[0..4]);
c5 uses the reference PERM (1,2,0) that yields C [96,48,16] under the
free-index -> output-position rule (plan.py:10-12).

Data: np.random.default_rng(seed) over the whole parent buffers, drawn in the
order A parent, B parent, C parent; fp32 values are drawn in f64 then cast
(the reference's refill_uniform convention, testkit.py:453-459).  C's parent
is drawn from the same distribution, so β = 1 accumulation and the padding
sentinels are both exercised.

Slicing: ``Workload.slice_free(owner, dim, lo, hi)`` restricts one free mode to
[lo, hi) by shifting the owning operand's and C's offsets — the reference
result of a slice is bitwise equal to the same elements of the full run
(SURVEY §8e), which is how large configs are checked and how the CPU baseline
samples them.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    dtype: str            # "d" or "s"
    ext_a: tuple
    inc_a: tuple
    len_a: int
    ext_b: tuple
    inc_b: tuple
    len_b: int
    conts: int
    cont_a: tuple
    cont_b: tuple
    perm: tuple
    inc_c: tuple
    len_c: int
    dist: str             # "uniform" | "normal"
    seed: int
    off_a: int = 0
    off_b: int = 0
    off_c: int = 0
    note: str = field(default="", compare=False)

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == "d" else np.float32

    @property
    def free_a(self):
        return [d for d in range(len(self.ext_a)) if d not in self.cont_a]

    @property
    def free_b(self):
        return [d for d in range(len(self.ext_b)) if d not in self.cont_b]

    @property
    def ext_c(self):
        src = [self.ext_a[d] for d in self.free_a] + [self.ext_b[d] for d in self.free_b]
        out = [0] * len(src)
        for i, e in enumerate(src):
            out[self.perm[i]] = e
        return tuple(out)

    @property
    def size_c(self):
        return int(np.prod(self.ext_c, dtype=np.int64)) if self.ext_c else 1

    @property
    def size_k(self):
        return int(np.prod([self.ext_a[d] for d in self.cont_a], dtype=np.int64)) if self.conts else 1

    @property
    def flops(self):
        """Algorithmic FLOPs 2·|C|·|K| (cli.py:175 counts |C|·|K| MACs)."""
        return 2 * self.size_c * self.size_k

    @property
    def alg_bytes(self):
        """elt·(|A_view| + |B_view| + 2·|C_view|): addressed elements only,
        C read and written."""
        elt = 8 if self.dtype == "d" else 4
        na = int(np.prod(self.ext_a, dtype=np.int64))
        nb = int(np.prod(self.ext_b, dtype=np.int64))
        return elt * (na + nb + 2 * self.size_c)

    def buffers(self):
        """Fresh seeded parent buffers (a, b, c) as numpy arrays."""
        rng = np.random.default_rng(self.seed)
        if self.dist == "uniform":
            draw = lambda n: rng.uniform(-1.0, 1.0, n)
        elif self.dist == "normal":
            draw = lambda n: rng.standard_normal(n)
        else:
            raise ValueError(self.dist)
        a = draw(self.len_a).astype(self.np_dtype)
        b = draw(self.len_b).astype(self.np_dtype)
        c = draw(self.len_c).astype(self.np_dtype)
        return a, b, c

    def args(self, a, b, c):
        """Positional + keyword arguments of the xGETT call."""
        pos = (len(self.ext_a), self.ext_a, self.inc_a, a, len(self.ext_b), self.ext_b, self.inc_b,
               b, self.conts, self.cont_a, self.cont_b, self.perm, self.inc_c, c)
        kw = dict(offset_a=self.off_a, offset_b=self.off_b, offset_c=self.off_c)
        return pos, kw

    def slice_free(self, owner: str, dim: int, lo: int, hi: int) -> "Workload":
        """Restrict free mode `dim` of operand `owner` ("A"/"B") to [lo, hi)."""
        if owner == "A":
            fi = self.free_a.index(dim)
            ext, inc = list(self.ext_a), self.inc_a
        else:
            fi = len(self.free_a) + self.free_b.index(dim)
            ext, inc = list(self.ext_b), self.inc_b
        assert 0 <= lo < hi <= ext[dim]
        ext[dim] = hi - lo
        q = self.perm[fi]
        kw = dict(off_c=self.off_c + lo * self.inc_c[q], name=f"{self.name}[{owner}{dim}:{lo}:{hi}]")
        if owner == "A":
            kw.update(ext_a=tuple(ext), off_a=self.off_a + lo * inc[dim])
        else:
            kw.update(ext_b=tuple(ext), off_b=self.off_b + lo * inc[dim])
        return replace(self, **kw)


def colmajor(w: "Workload") -> "Workload":
    """The same contraction with every tensor packed first-dimension-fastest
    (the reference's canonical layout, layout.py:10-11; SURVEY §8d asks for a
    column-major variant of c3/c4 in parity tests)."""
    def packed(ext):
        inc, step = [], 1
        for e in ext:
            inc.append(step)
            step *= int(e)
        return tuple(inc), step

    inc_a, len_a = packed(w.ext_a)
    inc_b, len_b = packed(w.ext_b)
    inc_c, len_c = packed(w.ext_c)
    return replace(w, name=w.name + "_colmajor", inc_a=inc_a, len_a=len_a, inc_b=inc_b,
                   len_b=len_b, inc_c=inc_c, len_c=len_c, off_a=0, off_b=0, off_c=0)


def _rowmajor(ext):
    inc = [1] * len(ext)
    for i in range(len(ext) - 2, -1, -1):
        inc[i] = inc[i + 1] * ext[i + 1]
    return tuple(inc)


C1 = Workload(
    "c1", "d",
    (48, 32, 40), _rowmajor((48, 32, 40)), 48 * 32 * 40,
    (40, 20, 32), _rowmajor((40, 20, 32)), 40 * 20 * 32,
    2, (1, 2), (2, 0), (1, 0), (48, 1), 960, "uniform", 0,
    note="DGETT small rank-3 x rank-3 (BASELINE configs[0])")

C2 = Workload(
    "c2", "d",
    (4096, 4096), (4224, 1), 4100 * 4224,
    (4096, 4096), (4160, 1), 4096 * 4160,
    1, (1,), (0,), (0, 1), (4200, 1), 4096 * 4200, "uniform", 1,
    note="DGETT GEMM-shaped strided subtensor (BASELINE configs[1])")

C3 = Workload(
    "c3", "d",
    (256, 512, 256), (131072, 256, 1), 256 * 512 * 256,
    (512, 384), (384, 1), 512 * 384,
    1, (1,), (0,), (0, 2, 1), (98304, 256, 1), 256 * 384 * 256, "normal", 2,
    note="DGETT tensor-times-matrix mode-2 (BASELINE configs[2])")

C4 = Workload(
    "c4", "d",
    (72, 72, 64, 64), (294912, 4096, 64, 1), 72 * 72 * 64 * 64,
    (64, 64, 72, 72), (331776, 5184, 72, 1), 64 * 64 * 72 * 72,
    2, (2, 3), (0, 1), (0, 2, 1, 3), (373248, 5184, 72, 1), 72 ** 4, "uniform", 3,
    note="DGETT rank-4 x rank-4 coupled-cluster-like (BASELINE configs[3])")

C5 = Workload(
    "c5", "s",
    (48, 24, 32, 16, 40), (983040, 40960, 1280, 40, 1), 48 * 24 * 64 * 16 * 40,
    (40, 32, 24, 96), (73728, 2304, 96, 1), 40 * 32 * 24 * 96,
    3, (1, 2, 4), (2, 1, 0), (1, 2, 0), (960, 20, 1), 96 * 48 * 20, "uniform", 4,
    note="SGETT high-rank mixed strides (BASELINE configs[4])")

CONFIGS = {w.name: w for w in (C1, C2, C3, C4, C5)}
