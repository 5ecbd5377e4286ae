"""Validation and spec types — the host-side mirror of gett.plan.

The checks themselves run natively (csrc/planner.cpp, a restatement of
/root/reference/pkg/src/gett/plan.py:162-234); this module keeps the
reference's Python surface: ``ErrorCode`` (:23-32), ``ValidationError``
(:35-41), ``ContractionError`` (:44-49), ``ContractionSpec`` (:52-72, same
structural ValueErrors), ``output_rank`` (:109-110), ``free_dims``
(:113-116), ``derive_output_extents`` (:119-127), ``validate`` (:162-234) and
the error-message texts, rebuilt from the native codes + info words.
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass

from . import _native
from .layout import TensorView


class ErrorCode(enum.Enum):
    ExtentMismatch = "ExtentMismatch"
    ContIndexOutOfRange = "ContIndexOutOfRange"
    ContIndexDuplicate = "ContIndexDuplicate"
    PermLengthWrong = "PermLengthWrong"
    PermNotBijection = "PermNotBijection"
    IncCLengthWrong = "IncCLengthWrong"
    OutputWriteAliasing = "OutputWriteAliasing"
    FootprintOutOfBounds = "FootprintOutOfBounds"
    NegativeExtent = "NegativeExtent"


# native enum gett_error_code (include/gett_b200.h) -> ErrorCode
_CODE = {
    1: ErrorCode.ExtentMismatch,
    2: ErrorCode.ContIndexOutOfRange,
    3: ErrorCode.ContIndexDuplicate,
    4: ErrorCode.PermLengthWrong,
    5: ErrorCode.PermNotBijection,
    6: ErrorCode.IncCLengthWrong,
    7: ErrorCode.OutputWriteAliasing,
    8: ErrorCode.FootprintOutOfBounds,
    9: ErrorCode.NegativeExtent,
}
_NAME = {0: "A", 1: "B", 2: "C"}


@dataclass(frozen=True)
class ValidationError:
    code: ErrorCode
    message: str

    def __str__(self) -> str:
        return f"{self.code.value}: {self.message}"


class ContractionError(ValueError):
    """Carries a validation error list."""

    def __init__(self, errors):
        self.errors = list(errors)
        super().__init__("; ".join(str(e) for e in self.errors))


@dataclass(frozen=True)
class ContractionSpec:
    """Pair count, paired dimensions of A and B, and the free-index ->
    output-position permutation."""

    conts: int
    cont_a: tuple
    cont_b: tuple
    perm: tuple

    def __post_init__(self):
        object.__setattr__(self, "cont_a", tuple(int(i) for i in self.cont_a))
        object.__setattr__(self, "cont_b", tuple(int(i) for i in self.cont_b))
        object.__setattr__(self, "perm", tuple(int(p) for p in self.perm))
        if self.conts < 0:
            raise ValueError(f"conts must be non-negative, got {self.conts}")
        if len(self.cont_a) != self.conts or len(self.cont_b) != self.conts:
            raise ValueError(
                f"cont_a and cont_b must each list {self.conts} dimensions, "
                f"got {len(self.cont_a)} and {len(self.cont_b)}")


def output_rank(rank_a: int, rank_b: int, conts: int) -> int:
    return rank_a + rank_b - 2 * conts


def free_dims(rank: int, contracted) -> list:
    dropped = set(contracted)
    return [d for d in range(rank) if d not in dropped]


def derive_output_extents(a: TensorView, b: TensorView, spec: ContractionSpec) -> tuple:
    """Output extents by output dimension (requires a valid spec)."""
    rank_c = output_rank(a.rank, b.rank, spec.conts)
    out = (ctypes.c_int64 * max(1, rank_c))()
    rc = _native.LIB.gett_derive_output_extents(
        a.rank, _native.i64(a.extents), b.rank, _native.i64(b.extents), spec.conts,
        _native.i64(spec.cont_a), _native.i64(spec.cont_b), _native.i64(spec.perm), out)
    _native.check(rc, "derive_output_extents")
    return tuple(int(out[i]) for i in range(rank_c))


def error_capacity(rank_a: int, rank_b: int, conts: int) -> int:
    """Upper bound on the number of errors one validation can report."""
    return 2 * (rank_a + rank_b) + 3 * conts + 3 * max(0, rank_a + rank_b) + 16


def decode_errors(n, codes, info, rank_a, ext_a, rank_b, ext_b, spec, inc_c) -> list:
    """Rebuild the reference's ValidationError list (messages per plan.py)."""
    errs = []
    for i in range(n):
        code = _CODE[int(codes[i])]
        w = [int(info[i * _native.ERR_INFO_WORDS + j]) for j in range(_native.ERR_INFO_WORDS)]
        name = _NAME.get(w[0], "?")
        if code is ErrorCode.NegativeExtent:
            msg = f"{name} has extent {w[2]} at dimension {w[1]}"
        elif code is ErrorCode.ContIndexOutOfRange:
            msg = (f"cont_{name.lower()}[{w[1]}] = {w[2]} is outside dimensions "
                   f"0..{w[3] - 1} of {name}")
        elif code is ErrorCode.ContIndexDuplicate:
            msg = f"cont_{name.lower()}[{w[1]}] = {w[2]} repeats a contracted dimension of {name}"
        elif code is ErrorCode.ExtentMismatch:
            msg = (f"contracted pair {w[1]} has extent {w[2]} in A (dimension {w[3]}) "
                   f"but {w[4]} in B (dimension {w[5]})")
        elif code is ErrorCode.PermLengthWrong:
            msg = f"perm has {w[1]} entries, output rank is {w[2]}"
        elif code is ErrorCode.PermNotBijection:
            msg = f"perm {tuple(spec.perm)} is not a bijection on 0..{w[1] - 1}"
        elif code is ErrorCode.IncCLengthWrong:
            msg = f"inc_c has {w[1]} entries, output rank is {w[2]}"
        elif code is ErrorCode.OutputWriteAliasing:
            msg = f"inc_c[{w[1]}] = 0 would alias writes across extent {w[2]}"
        else:  # FootprintOutOfBounds
            msg = f"{name} addresses offsets {w[1]}..{w[2]} but its buffer holds {w[3]} elements"
        errs.append(ValidationError(code, msg))
    return errs


def validate(a: TensorView, b: TensorView, spec: ContractionSpec, inc_c,
             c_view: TensorView | None = None) -> list:
    """Every violation in the arguments, in the reference's order; an empty
    list means valid.  Never raises on bad values (plan.py:162-234)."""
    inc_c = tuple(int(i) for i in inc_c)
    cap = error_capacity(a.rank, b.rank, spec.conts) + (2 * c_view.rank if c_view else 0)
    codes = (ctypes.c_int32 * cap)()
    info = (ctypes.c_int64 * (cap * _native.ERR_INFO_WORDS))()
    if c_view is not None:
        mode, rcv, ecv, icv, off_c, len_c = (2, c_view.rank, c_view.extents, c_view.increments,
                                              c_view.base_offset, c_view.buffer_len)
    else:
        mode, rcv, ecv, icv, off_c, len_c = (0, 0, (), (), 0, 0)
    n = _native.LIB.gett_validate(
        a.rank, _native.i64(a.extents), _native.i64(a.increments), a.base_offset, a.buffer_len,
        b.rank, _native.i64(b.extents), _native.i64(b.increments), b.base_offset, b.buffer_len,
        spec.conts, _native.i64(spec.cont_a), _native.i64(spec.cont_b),
        len(spec.perm), _native.i64(spec.perm), len(inc_c), _native.i64(inc_c),
        mode, rcv, _native.i64(ecv), _native.i64(icv), off_c, len_c, codes, info, cap)
    _native.check(n, "validate")
    return decode_errors(min(n, cap), codes, info, a.rank, a.extents, b.rank, b.extents, spec, inc_c)


# ---------------------------------------------------------------------------
# Per-call descriptor cache.  Building the views/spec (structural checks) and
# the ctypes argument arrays costs ~15 µs of Python per call — more than the
# device time of small contractions.  The result is a pure function of the
# descriptor values, so repeated calls with an equal descriptor reuse it.
# Scalars are keyed with their types (ctypes rejects e.g. float offsets, and
# a hit must not mask that); tuple elements go through int() either way.

class Prepared:
    __slots__ = ("a_view", "b_view", "spec", "inc_c", "cap", "args_a", "args_b", "args_spec")

    def __init__(self, a_view, b_view, spec, inc_c):
        self.a_view, self.b_view, self.spec, self.inc_c = a_view, b_view, spec, inc_c
        self.cap = error_capacity(a_view.rank, b_view.rank, spec.conts)
        self.args_a = (a_view.rank, _native.i64(a_view.extents), _native.i64(a_view.increments))
        self.args_b = (b_view.rank, _native.i64(b_view.extents), _native.i64(b_view.increments))
        self.args_spec = (spec.conts, _native.i64(spec.cont_a), _native.i64(spec.cont_b),
                          len(spec.perm), _native.i64(spec.perm), len(inc_c), _native.i64(inc_c))


_PREP: dict = {}
_PREP_CAP = 1024


def prepare(rank_a, ext_a, inc_a, offset_a, len_a, rank_b, ext_b, inc_b, offset_b, len_b,
            conts, cont_a, cont_b, perm, inc_c) -> Prepared:
    """Views, spec and native argument arrays for one call (cached).  Raises
    exactly what TensorView / ContractionSpec construction raises."""
    try:
        key = (rank_a, type(rank_a), tuple(ext_a), tuple(inc_a), offset_a, type(offset_a), len_a,
               rank_b, type(rank_b), tuple(ext_b), tuple(inc_b), offset_b, type(offset_b), len_b,
               conts, type(conts), tuple(cont_a), tuple(cont_b), tuple(perm), tuple(inc_c))
        hit = _PREP.get(key)
    except TypeError:  # unhashable or non-iterable descriptor: no caching
        key = hit = None
    if hit is not None:
        return hit
    p = Prepared(TensorView(rank_a, ext_a, inc_a, offset_a, len_a),
                 TensorView(rank_b, ext_b, inc_b, offset_b, len_b),
                 ContractionSpec(conts, cont_a, cont_b, perm),
                 tuple(int(i) for i in inc_c))
    if key is not None:
        if len(_PREP) >= _PREP_CAP:
            _PREP.pop(next(iter(_PREP)))
        _PREP[key] = p
    return p


_TLS = threading.local()


def err_buffers(cap):
    """Per-thread error-report buffers (the native side writes them only on a
    validation failure, and the caller decodes them before returning)."""
    bufs = getattr(_TLS, "bufs", None)
    if bufs is None:
        bufs = _TLS.bufs = {}
    pair = bufs.get(cap)
    if pair is None:
        pair = bufs[cap] = ((ctypes.c_int32 * cap)(), (ctypes.c_int64 * (cap * _native.ERR_INFO_WORDS))())
    return pair
