"""Plan once, execute many: the per-call host cost of small contractions.

``dgett(...)`` re-derives everything from its arguments on every call
(kernel.py:124-155 does the same in the reference: type checks, views, spec,
two-phase validation, plan).  For a call repeated on buffers of the same
shape, ``dgett_plan`` does that work once — with the reference's exact
signature — and returns a ``GettPlan`` whose ``__call__(a, b, c)`` (numpy,
synchronous) or ``device(a, b, c)`` (CUDA tensors, stream-ordered) run
C += contract(A, B) through gett_execute / gett_execute_device
(include/gett_b200.h): one ctypes call, no validation or plan lookup.

    p = dgett_plan(rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b,
                   conts, cont_a, cont_b, perm, inc_c, c, offset_a=0, ...)
    if p.errors: ...            # the list dgett would return, C untouched
    p(a, b, c)                  # == dgett(... same arguments ...)

Buffers passed to a plan must have the planned dtype and lengths (checked)
and be contiguous; their contents may change freely between calls.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .plan import decode_errors, err_buffers, prepare

_DT = {"d": np.dtype(np.float64), "s": np.dtype(np.float32)}


class GettPlan:
    """A validated, planned xGETT (see the module docstring)."""

    __slots__ = ("prefix", "errors", "_h", "_lens", "_dtype", "_exec", "_exec_dev", "_last_dev",
                 "__weakref__")

    def __init__(self, prefix, rank_a, ext_a, inc_a, len_a, rank_b, ext_b, inc_b, len_b, conts, cont_a,
                 cont_b, perm, inc_c, len_c, offset_a=0, offset_b=0, offset_c=0, devices=None):
        if prefix not in _DT:
            raise TypeError(f"{prefix}gett has no plan form (d and s only)")
        self.prefix = prefix
        self._h = None
        self._dtype = _DT[prefix]
        self._lens = (int(len_a), int(len_b), int(len_c))
        pr = prepare(rank_a, ext_a, inc_a, offset_a, len_a, rank_b, ext_b, inc_b, offset_b, len_b,
                     conts, cont_a, cont_b, perm, inc_c)
        codes, info = err_buffers(pr.cap)
        devs = [] if devices is None else [int(d) for d in devices]
        h = ctypes.c_void_p()
        rc = _native.LIB.gett_plan_create(
            prefix.encode(), *pr.args_a, pr.a_view.base_offset, pr.a_view.buffer_len,
            *pr.args_b, pr.b_view.base_offset, pr.b_view.buffer_len, *pr.args_spec,
            int(offset_c), int(len_c), len(devs), _native.i32(devs), ctypes.byref(h), codes, info,
            pr.cap)
        n = _native.check(rc, prefix + "gett_plan")
        self.errors = (decode_errors(min(n, pr.cap), codes, info, pr.a_view.rank, pr.a_view.extents,
                                     pr.b_view.rank, pr.b_view.extents, pr.spec, pr.inc_c) if n else [])
        self._h = h.value
        self._last_dev = None  # the tensors of the last device() call (checks done)
        self._exec = _native.LIB.gett_execute
        self._exec_dev = _native.LIB.gett_execute_device

    def _check(self, a, b, c):
        for name, buf, n in (("a", a, self._lens[0]), ("b", b, self._lens[1]), ("c", c, self._lens[2])):
            if buf.dtype != self._dtype or buf.shape != (n,):
                raise TypeError(f"{name} must be a flat {self._dtype} buffer of {n} elements (the planned length)")

    def __call__(self, a, b, c):
        """C += contract(A, B) on host numpy buffers (synchronous); returns
        the plan's validation errors (then nothing runs), else []."""
        if self.errors:
            return self.errors
        if not (isinstance(a, np.ndarray) and isinstance(b, np.ndarray) and isinstance(c, np.ndarray)):
            raise TypeError("a, b and c must be numpy arrays")
        self._check(a, b, c)
        if not (a.flags.c_contiguous and b.flags.c_contiguous and c.flags.c_contiguous):
            raise TypeError("plan buffers must be contiguous")
        if not c.flags.writeable:
            raise ValueError("assignment destination is read-only")
        if self._h is not None:
            _native.check(self._exec(self._h, a.ctypes.data, b.ctypes.data, c.ctypes.data),
                          self.prefix + "gett_execute")
        return []

    def device(self, a, b, c, stream=None):
        """C += contract(A, B) on CUDA tensors, on the current (or given)
        stream of c's device; no host synchronisation."""
        if self.errors:
            return self.errors
        import torch

        from .device import _raw_stream

        last = self._last_dev
        if last is None or last[0] is not a or last[1] is not b or last[2] is not c:
            if not (a.is_cuda and b.is_cuda and c.is_cuda):
                raise TypeError("a, b and c must be CUDA tensors")
            want = torch.float64 if self.prefix == "d" else torch.float32
            for name, t, n in (("a", a, self._lens[0]), ("b", b, self._lens[1]), ("c", c, self._lens[2])):
                if t.dtype != want or t.dim() != 1 or t.shape[0] != n or t.stride(0) != 1:
                    raise TypeError(f"{name} must be a contiguous 1-D {want} tensor of {n} elements")
            self._last_dev = (a, b, c)
        elif a.shape[0] != self._lens[0] or b.shape[0] != self._lens[1] or c.shape[0] != self._lens[2]:
            raise TypeError("a buffer was resized since it was planned")
        handle = _raw_stream(c.device.index) if stream is None else stream.cuda_stream
        if self._h is not None:
            _native.check(self._exec_dev(self._h, a.data_ptr(), b.data_ptr(), c.data_ptr(),
                                         ctypes.c_void_p(handle)), self.prefix + "gett_execute_device")
        return []

    def close(self):
        self._last_dev = None
        if self._h is not None:
            _native.LIB.gett_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass


def _plan(prefix, rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c,
          c, offset_a=0, offset_b=0, offset_c=0, *, devices=None):
    return GettPlan(prefix, rank_a, ext_a, inc_a, len(a), rank_b, ext_b, inc_b, len(b), conts, cont_a,
                    cont_b, perm, inc_c, len(c), offset_a, offset_b, offset_c, devices)


def dgett_plan(rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c,
               offset_a=0, offset_b=0, offset_c=0, *, devices=None) -> GettPlan:
    """A GettPlan for dgett's arguments (the buffers give the lengths)."""
    return _plan("d", rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm,
                 inc_c, c, offset_a, offset_b, offset_c, devices=devices)


def sgett_plan(rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c,
               offset_a=0, offset_b=0, offset_c=0, *, devices=None) -> GettPlan:
    """A GettPlan for sgett's arguments (the buffers give the lengths)."""
    return _plan("s", rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm,
                 inc_c, c, offset_a, offset_b, offset_c, devices=devices)
