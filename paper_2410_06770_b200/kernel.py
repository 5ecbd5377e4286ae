"""xGETT entry points — the drop-in for gett.kernel (host numpy buffers).

``sgett`` / ``dgett`` keep the reference signature, keyword offsets, raises
and return values (/root/reference/pkg/src/gett/kernel.py:124-184):

* TypeError unless c is an ndarray; a, b go through np.asarray; every buffer
  must be 1-D with exactly the entry point's dtype (kernel.py:132-140).
* ValueError for structural problems (TensorView / ContractionSpec).
* Value problems come back as the reference's ValidationError list, in the
  reference's order, with c untouched (kernel.py:146-153).
* Otherwise C += contract(A, B) runs on the GPU and [] is returned.

The call crosses the C ABI (include/gett_b200.h) with plain pointers; the
native side validates, plans, copies the addressed spans to the device,
launches the sm_100a kernel and copies C's span back.  There is no CPU path.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .layout import TensorView
from .plan import decode_errors, err_buffers, prepare

_PREFIX_DTYPE = {
    "s": np.dtype(np.float32),
    "d": np.dtype(np.float64),
    "c": np.dtype(np.complex64),
    "z": np.dtype(np.complex128),
}
_ENTRY = {"s": "gett_sgett", "d": "gett_dgett", "c": "gett_cgett", "z": "gett_zgett"}


_MULTI = {"s": "gett_sgett_multi", "d": "gett_dgett_multi"}


def _gett(prefix, rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm,
          inc_c, c, offset_a, offset_b, offset_c, devices=None):
    dtype = _PREFIX_DTYPE[prefix]
    if not isinstance(c, np.ndarray):
        raise TypeError("c must be a numpy array (results are written in place)")
    a = np.asarray(a)
    b = np.asarray(b)
    for name, buf in (("a", a), ("b", b), ("c", c)):
        if buf.ndim != 1:
            raise TypeError(f"{name} must be a flat 1-D buffer, got shape {buf.shape}")
        if buf.dtype != dtype:
            raise TypeError(f"{name} has dtype {buf.dtype}, this entry point needs {dtype}")
    pr = prepare(rank_a, ext_a, inc_a, offset_a, a.shape[0], rank_b, ext_b, inc_b, offset_b,
                 b.shape[0], conts, cont_a, cont_b, perm, inc_c)
    a_view, b_view, spec, inc_c = pr.a_view, pr.b_view, pr.spec, pr.inc_c
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    cw = c if c.flags.c_contiguous else np.ascontiguousarray(c)
    empty = a_view.is_empty or b_view.is_empty
    if not c.flags.writeable and not empty:
        # the reference fails at its first store into c, after both validation
        # phases (kernel.py:146-153): return their errors, else fail before any work
        from .plan import derive_output_extents, validate
        errs = validate(a_view, b_view, spec, inc_c)
        if not errs:
            ext_c = derive_output_extents(a_view, b_view, spec)
            c_view = TensorView(len(ext_c), ext_c, tuple(inc_c), int(offset_c), c.shape[0])
            errs = validate(a_view, b_view, spec, inc_c, c_view=c_view)
        if errs:
            return errs
        raise ValueError("assignment destination is read-only")
    cap = pr.cap
    codes, info = err_buffers(cap)
    args = (*pr.args_a, a.ctypes.data, a_view.base_offset, a_view.buffer_len,
            *pr.args_b, b.ctypes.data, b_view.base_offset, b_view.buffer_len,
            *pr.args_spec, cw.ctypes.data, int(offset_c), cw.shape[0])
    if devices is not None:
        if prefix not in _MULTI:
            raise TypeError(f"{prefix}gett has no multi-device form")
        devs = [int(d) for d in devices]
        if not devs:
            raise ValueError("devices must list at least one CUDA device")
        rc = getattr(_native.LIB, _MULTI[prefix])(*args, len(devs), _native.i32(devs), codes, info, cap)
    else:
        rc = getattr(_native.LIB, _ENTRY[prefix])(*args, codes, info, cap)
    n = _native.check(rc, prefix + "gett")
    if n:
        return decode_errors(min(n, cap), codes, info, a_view.rank, a_view.extents, b_view.rank,
                             b_view.extents, spec, inc_c)
    if cw is not c:
        c[...] = cw
    return []


def sgett(rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
          conts, cont_a, cont_b, perm, inc_c, c,
          offset_a=0, offset_b=0, offset_c=0, *, devices=None):
    """32-bit real contraction; see dgett for the parameter contract."""
    return _gett("s", rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
                 conts, cont_a, cont_b, perm, inc_c, c, offset_a, offset_b, offset_c, devices)


def dgett(rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
          conts, cont_a, cont_b, perm, inc_c, c,
          offset_a=0, offset_b=0, offset_c=0, *, devices=None):
    """64-bit real binary tensor contraction, accumulating into c.

    Arguments follow the xGETT interface order: A's rank,
    extents, increments and buffer; the same for B; the pair count, paired
    dimensions of A and of B, the free-index -> output-position permutation;
    the output increments and buffer.  offset_* locate each view's first used
    element.  Returns [] when the contraction ran, else the validation error
    list (c untouched).  C is accumulated: clear the view first (zero_view)
    for a plain contraction.

    devices (keyword, beyond the reference signature): run the call across
    these CUDA devices — C's outermost free mode split into one slab per
    device, or the largest contracted pair split with one reduce on
    devices[0] when the free extents are too small (include/gett_b200.h,
    gett_dgett_multi).  set_devices() makes a list the default.
    """
    return _gett("d", rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
                 conts, cont_a, cont_b, perm, inc_c, c, offset_a, offset_b, offset_c, devices)


def cgett(rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
          conts, cont_a, cont_b, perm, inc_c, c,
          offset_a=0, offset_b=0, offset_c=0):
    """64-bit complex (2x32-bit) contraction; see dgett for the parameter contract."""
    return _gett("c", rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
                 conts, cont_a, cont_b, perm, inc_c, c, offset_a, offset_b, offset_c)


def zgett(rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
          conts, cont_a, cont_b, perm, inc_c, c,
          offset_a=0, offset_b=0, offset_c=0):
    """128-bit complex (2x64-bit) contraction; see dgett for the parameter contract."""
    return _gett("z", rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
                 conts, cont_a, cont_b, perm, inc_c, c, offset_a, offset_b, offset_c)


def zero_view(view: TensorView, buf: np.ndarray) -> None:
    """Set every element addressed by the view to zero, touching nothing else
    (kernel.py:111-113), on the GPU."""
    if not isinstance(buf, np.ndarray) or buf.ndim != 1:
        raise TypeError("buf must be a flat 1-D numpy array")
    prefix = dtype_prefix(buf.dtype)
    if view.is_empty or any(e < 0 for e in view.extents):
        return
    lo = hi = 0
    for e, i in zip(view.extents, view.increments):
        span = i * (e - 1)
        lo, hi = (lo + span, hi) if span < 0 else (lo, hi + span)
    if view.base_offset + lo < 0 or view.base_offset + hi >= buf.shape[0]:
        raise IndexError(f"view addresses offsets {view.base_offset + lo}..{view.base_offset + hi} "
                         f"outside a buffer of {buf.shape[0]} elements")
    if not buf.flags.writeable:
        raise ValueError("assignment destination is read-only")
    w = buf if buf.flags.c_contiguous else np.ascontiguousarray(buf)
    f = _native.LIB.gett_zero_view_d if prefix in "dz" else _native.LIB.gett_zero_view_s
    if prefix in "cz":
        # complex: the real and imaginary parts are two real views with
        # doubled increments over the interleaved (re, im) buffer
        inc2 = [2 * i for i in view.increments]
        for part in (0, 1):
            _native.check(f(view.rank, _native.i64(view.extents), _native.i64(inc2),
                            2 * view.base_offset + part, 2 * w.shape[0], w.ctypes.data),
                          "zero_view")
    else:
        _native.check(f(view.rank, _native.i64(view.extents), _native.i64(view.increments),
                        view.base_offset, w.shape[0], w.ctypes.data), "zero_view")
    if w is not buf:
        buf[...] = w


def pack(view: TensorView, buf) -> np.ndarray:
    """The elements the view addresses, in canonical packed order (dimension
    0 fastest) — testkit.pack's data (/root/reference/pkg/src/gett/testkit.py:101-103,
    ``buf[view_offsets(view)]``), gathered on the GPU bit for bit."""
    buf = np.asarray(buf)
    if buf.ndim != 1:
        raise TypeError("buf must be a flat 1-D buffer")
    dtype_prefix(buf.dtype)  # s/d/c/z element types only
    n = 1
    for e in view.extents:
        n *= max(int(e), 0)
    out = np.empty(n, dtype=buf.dtype)
    if n == 0:
        return out
    lo = hi = 0
    for e, i in zip(view.extents, view.increments):
        span = i * (e - 1)
        lo, hi = (lo + span, hi) if span < 0 else (lo, hi + span)
    if view.base_offset + lo < 0 or view.base_offset + hi >= buf.shape[0]:
        raise IndexError(f"view addresses offsets {view.base_offset + lo}..{view.base_offset + hi} "
                         f"outside a buffer of {buf.shape[0]} elements")
    src = np.ascontiguousarray(buf)
    _native.check(_native.LIB.gett_pack(view.rank, _native.i64(view.extents),
                                        _native.i64(view.increments), view.base_offset,
                                        src.shape[0], src.itemsize, src.ctypes.data,
                                        out.ctypes.data), "pack")
    return out


def dtype_prefix(dtype) -> str:
    """The s/d/c/z tag for a numpy element type (kernel.py:203-209)."""
    dtype = np.dtype(dtype)
    for prefix, dt in _PREFIX_DTYPE.items():
        if dt == dtype:
            return prefix
    raise TypeError(f"no entry point for dtype {dtype}")


def gett_for_dtype(dtype):
    """The entry point matching a numpy dtype."""
    return globals()[dtype_prefix(dtype) + "gett"]
