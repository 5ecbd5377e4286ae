"""CPU oracle for the xGETT hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (the cpu_baseline leg and
--impl reference) may import this module.  It is the checker, never the thing
measured as the product, and the product package never imports it.

Contents
--------
* ``oracle_dgett`` / ``oracle_sgett``: ctypes bindings to gett_oracle.c, the C
  restatement of the reference loop (kernel.py:48-78, plan.py:258-289).  Same
  argument order as the reference xGETT (kernel.py:158-184), plus a free-range
  [free_lo, free_hi) for bounded samples and a thread count.
* ``validate_codes``: a pure-Python restatement of plan.py:162-234 (and the
  phase-2 C footprint check, kernel.py:149-153) returning the ordered error
  code names, used to fuzz the native planner.
* ``einsum_check``: fp64 numpy cross-check on as_strided views.

Parity: pinned against the reference's own outputs (tests/golden/, generated
by tests/golden/make_golden.py from the reference gett package).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    """Compile liboracle.so from gett_oracle.c (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "gett_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(path)
        i64p = ctypes.POINTER(ctypes.c_int64)
        for name in ("oracle_dgett", "oracle_sgett", "oracle_zgett", "oracle_cgett"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_int, i64p, i64p, ctypes.c_void_p, ctypes.c_int64,
                          ctypes.c_int, i64p, i64p, ctypes.c_void_p, ctypes.c_int64,
                          ctypes.c_int, i64p, i64p, i64p, i64p, ctypes.c_void_p, ctypes.c_int64,
                          ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
        _LIB = L
    return _LIB


def _i64(seq):
    arr = (ctypes.c_int64 * max(1, len(seq)))(*[int(x) for x in seq])
    return arr


def _call(name, dtype, rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b,
          perm, inc_c, c, offset_a=0, offset_b=0, offset_c=0, free_lo=0, free_hi=-1, threads=1):
    a = np.ascontiguousarray(a, dtype=dtype)
    b = np.ascontiguousarray(b, dtype=dtype)
    assert isinstance(c, np.ndarray) and c.dtype == dtype and c.flags.c_contiguous
    rc = getattr(lib(), name)(
        int(rank_a), _i64(ext_a), _i64(inc_a), a.ctypes.data, int(offset_a),
        int(rank_b), _i64(ext_b), _i64(inc_b), b.ctypes.data, int(offset_b),
        int(conts), _i64(cont_a), _i64(cont_b), _i64(perm), _i64(inc_c), c.ctypes.data,
        int(offset_c), int(free_lo), int(free_hi), int(threads))
    if rc != 0:
        raise ValueError(f"{name}: unsupported descriptor (rc={rc})")


def oracle_dgett(*args, **kw):
    """Reference-order float64 contraction into c (in place).  Mirrors
    dgett's argument order (kernel.py:166-184)."""
    _call("oracle_dgett", np.float64, *args, **kw)


def oracle_sgett(*args, **kw):
    """Reference-order float32 contraction into c (in place)."""
    _call("oracle_sgett", np.float32, *args, **kw)


def oracle_zgett(*args, **kw):
    """Reference-order complex128 contraction into c (kernel.py:195-200)."""
    _call("oracle_zgett", np.complex128, *args, **kw)


def oracle_cgett(*args, **kw):
    """Reference-order complex64 contraction into c (kernel.py:187-192)."""
    _call("oracle_cgett", np.complex64, *args, **kw)


ORACLE = {"d": oracle_dgett, "s": oracle_sgett, "z": oracle_zgett, "c": oracle_cgett}


# ---------------------------------------------------------------------------
# validation restatement (plan.py:130-241)


def _footprint(ext, inc):
    lo = hi = 0
    for e, i in zip(ext, inc):
        if e <= 0:
            continue
        span = i * (e - 1)
        if span < 0:
            lo += span
        else:
            hi += span
    return lo, hi


def _fp_bad(ext, inc, off, n):
    if any(e == 0 for e in ext):
        return False
    lo, hi = _footprint(ext, inc)
    return off + lo < 0 or off + hi >= n


def validate_codes(rank_a, ext_a, inc_a, len_a, off_a, rank_b, ext_b, inc_b, len_b, off_b,
                   conts, cont_a, cont_b, perm, inc_c, len_c=None, off_c=0):
    """Ordered list of error-code names, as gett.plan.validate then the
    kernel's phase-2 output footprint check would produce (plan.py:179-232,
    kernel.py:146-153)."""
    errs = []
    for ext in (ext_a, ext_b):
        for e in ext:
            if e < 0:
                errs.append("NegativeExtent")

    def cont_ok(idx, rank):
        ok = True
        seen = set()
        for d in idx:
            if not 0 <= d < rank:
                errs.append("ContIndexOutOfRange")
                ok = False
            elif d in seen:
                errs.append("ContIndexDuplicate")
                ok = False
            seen.add(d)
        return ok

    a_ok = cont_ok(cont_a, rank_a)
    b_ok = cont_ok(cont_b, rank_b)
    if a_ok and b_ok:
        for da, db in zip(cont_a, cont_b):
            if ext_a[da] != ext_b[db]:
                errs.append("ExtentMismatch")
    rank_c = rank_a + rank_b - 2 * conts
    perm_ok = True
    if len(perm) != rank_c:
        errs.append("PermLengthWrong")
        perm_ok = False
    elif sorted(perm) != list(range(rank_c)):
        errs.append("PermNotBijection")
        perm_ok = False
    inc_ok = True
    if len(inc_c) != rank_c:
        errs.append("IncCLengthWrong")
        inc_ok = False
    ext_c = None
    if a_ok and b_ok and perm_ok and inc_ok:
        srcs = [ext_a[d] for d in range(rank_a) if d not in set(cont_a)]
        srcs += [ext_b[d] for d in range(rank_b) if d not in set(cont_b)]
        ext_c = [0] * rank_c
        for i, e in enumerate(srcs):
            ext_c[perm[i]] = e
        for e, i in zip(ext_c, inc_c):
            if i == 0 and e > 1:
                errs.append("OutputWriteAliasing")
    if _fp_bad(ext_a, inc_a, off_a, len_a):
        errs.append("FootprintOutOfBounds")
    if _fp_bad(ext_b, inc_b, off_b, len_b):
        errs.append("FootprintOutOfBounds")
    if errs or len_c is None:
        return errs
    if _fp_bad(ext_c, inc_c, off_c, len_c):
        errs.append("FootprintOutOfBounds")
    return errs


# ---------------------------------------------------------------------------
# fp64 numpy cross-check


def strided(buf, ext, inc, off):
    """An ndarray view of the xGETT view (ext, inc, off) over a 1-D buffer
    (negative increments allowed)."""
    item = buf.itemsize
    base = buf[off:] if off < len(buf) else buf[len(buf):]
    return np.lib.stride_tricks.as_strided(base, shape=tuple(ext),
                                           strides=tuple(i * item for i in inc))


def einsum_check(ext_a, inc_a, a, off_a, ext_b, inc_b, b, off_b, conts, cont_a, cont_b, perm,
                 out_dtype=np.float64):
    """C = contract(A, B) in fp64 via numpy.einsum, returned as an ndarray with
    output extents (the accumulate-free value)."""
    ra, rb = len(ext_a), len(ext_b)
    letters = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ"
    la = [None] * ra
    lb = [None] * rb
    nxt = 0
    for da, db in zip(cont_a, cont_b):
        la[da] = lb[db] = letters[nxt]
        nxt += 1
    free = []
    for d in range(ra):
        if la[d] is None:
            la[d] = letters[nxt]
            free.append(letters[nxt])
            nxt += 1
    for d in range(rb):
        if lb[d] is None:
            lb[d] = letters[nxt]
            free.append(letters[nxt])
            nxt += 1
    out = [None] * len(free)
    for i, p in enumerate(perm):
        out[p] = free[i]
    A = strided(a, ext_a, inc_a, off_a).astype(np.float64)
    B = strided(b, ext_b, inc_b, off_b).astype(np.float64)
    expr = "".join(la) + "," + "".join(lb) + "->" + "".join(out)
    return np.einsum(expr, A, B, optimize=True).astype(out_dtype)
