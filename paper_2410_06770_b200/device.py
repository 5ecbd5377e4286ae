"""Zero-copy xGETT on device-resident buffers (torch CUDA tensors as plumbing).

``dgett_device`` / ``sgett_device`` take the reference argument list with
1-D CUDA tensors in place of numpy buffers and launch on the tensors' device
and the current torch stream (stream-ordered, no host synchronisation).  They
call gett_dgett_device / gett_sgett_device (include/gett_b200.h): the same
native validation, planner and sm_100a kernels as the host entry points, but
no host<->device copies.  Validation errors come back as ValidationError
lists exactly like dgett's.
"""
from __future__ import annotations

import ctypes

from . import _native
from .layout import TensorView
from .plan import ContractionSpec, decode_errors, error_capacity

_DT = {"s": "float32", "d": "float64", "c": "complex64", "z": "complex128"}


def _buf(t, name, prefix):
    import torch

    want = getattr(torch, _DT[prefix])
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dim() != 1:
        raise TypeError(f"{name} must be a flat 1-D buffer, got shape {tuple(t.shape)}")
    if t.dtype != want:
        raise TypeError(f"{name} has dtype {t.dtype}, this entry point needs {want}")
    if t.stride(0) != 1:
        raise TypeError(f"{name} must be contiguous")
    return t


def _gett_device(prefix, rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b,
                 perm, inc_c, c, offset_a=0, offset_b=0, offset_c=0, stream=None):
    import torch

    a = _buf(a, "a", prefix)
    b = _buf(b, "b", prefix)
    c = _buf(c, "c", prefix)
    if not (a.device == b.device == c.device):
        raise ValueError("a, b and c must live on one device")
    a_view = TensorView(rank_a, ext_a, inc_a, offset_a, a.shape[0])
    b_view = TensorView(rank_b, ext_b, inc_b, offset_b, b.shape[0])
    spec = ContractionSpec(conts, cont_a, cont_b, perm)
    inc_c = tuple(int(i) for i in inc_c)
    cap = error_capacity(a_view.rank, b_view.rank, spec.conts)
    codes = (ctypes.c_int32 * cap)()
    info = (ctypes.c_int64 * (cap * _native.ERR_INFO_WORDS))()
    if stream is None:
        stream = torch.cuda.current_stream(c.device)
    fn = getattr(_native.LIB, f"gett_{prefix}gett_device")
    with torch.cuda.device(c.device):
        rc = fn(a_view.rank, _native.i64(a_view.extents), _native.i64(a_view.increments),
                a.data_ptr(), a_view.base_offset, a_view.buffer_len,
                b_view.rank, _native.i64(b_view.extents), _native.i64(b_view.increments),
                b.data_ptr(), b_view.base_offset, b_view.buffer_len,
                spec.conts, _native.i64(spec.cont_a), _native.i64(spec.cont_b),
                len(spec.perm), _native.i64(spec.perm), len(inc_c), _native.i64(inc_c),
                c.data_ptr(), int(offset_c), c.shape[0], ctypes.c_void_p(stream.cuda_stream),
                codes, info, cap)
    n = _native.check(rc, prefix + "gett_device")
    if n:
        return decode_errors(min(n, cap), codes, info, a_view.rank, a_view.extents, b_view.rank,
                             b_view.extents, spec, inc_c)
    return []


def dgett_device(*args, **kw):
    """float64 xGETT on CUDA tensors (stream-ordered); see kernel.dgett."""
    return _gett_device("d", *args, **kw)


def sgett_device(*args, **kw):
    """float32 xGETT on CUDA tensors (stream-ordered); see kernel.sgett."""
    return _gett_device("s", *args, **kw)


def zero_view_device(view: TensorView, buf, stream=None) -> None:
    """zero_view on a CUDA tensor (stream-ordered)."""
    import torch

    prefix = "d" if buf.dtype == torch.float64 else "s"
    _buf(buf, "buf", prefix)
    if stream is None:
        stream = torch.cuda.current_stream(buf.device)
    fn = _native.LIB.gett_zero_view_d_device if prefix == "d" else _native.LIB.gett_zero_view_s_device
    with torch.cuda.device(buf.device):
        _native.check(fn(view.rank, _native.i64(view.extents), _native.i64(view.increments),
                         view.base_offset, buf.shape[0], buf.data_ptr(),
                         ctypes.c_void_p(stream.cuda_stream)), "zero_view_device")


def cgett_device(*args, **kw):
    """complex64 xGETT on CUDA tensors (stream-ordered); see kernel.cgett."""
    return _gett_device("c", *args, **kw)


def zgett_device(*args, **kw):
    """complex128 xGETT on CUDA tensors (stream-ordered); see kernel.zgett."""
    return _gett_device("z", *args, **kw)
