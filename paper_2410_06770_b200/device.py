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
from .plan import decode_errors, err_buffers, prepare

_DT = {"s": "float32", "d": "float64", "c": "complex64", "z": "complex128"}


_WANT = {}


def _buf(t, name, prefix):
    import torch

    want = _WANT.get(prefix)
    if want is None:
        want = _WANT[prefix] = getattr(torch, _DT[prefix])
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dim() != 1:
        raise TypeError(f"{name} must be a flat 1-D buffer, got shape {tuple(t.shape)}")
    if t.dtype != want:
        raise TypeError(f"{name} has dtype {t.dtype}, this entry point needs {want}")
    if t.stride(0) != 1:
        raise TypeError(f"{name} must be contiguous")
    return t


def _raw_stream(dev_index):
    """Handle of the current torch stream on a device.  The private raw-stream
    query avoids building a torch.cuda.Stream object (several µs per call)."""
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(dev_index)
    return torch.cuda.current_stream(dev_index).cuda_stream


def _gett_device(prefix, rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b,
                 perm, inc_c, c, offset_a=0, offset_b=0, offset_c=0, stream=None):
    import torch

    a = _buf(a, "a", prefix)
    b = _buf(b, "b", prefix)
    c = _buf(c, "c", prefix)
    dev = c.device
    if not (a.device == b.device == dev):
        raise ValueError("a, b and c must live on one device")
    pr = prepare(rank_a, ext_a, inc_a, offset_a, a.shape[0], rank_b, ext_b, inc_b, offset_b,
                 b.shape[0], conts, cont_a, cont_b, perm, inc_c)
    cap = pr.cap
    codes, info = err_buffers(cap)
    handle = _raw_stream(dev.index) if stream is None else stream.cuda_stream
    fn = _FN[prefix]
    args = (*pr.args_a, a.data_ptr(), pr.a_view.base_offset, pr.a_view.buffer_len,
            *pr.args_b, b.data_ptr(), pr.b_view.base_offset, pr.b_view.buffer_len,
            *pr.args_spec, c.data_ptr(), int(offset_c), c.shape[0],
            ctypes.c_void_p(handle), codes, info, cap)
    if torch.cuda.current_device() == dev.index:
        rc = fn(*args)
    else:
        with torch.cuda.device(dev):
            rc = fn(*args)
    n = _native.check(rc, prefix + "gett_device")
    if n:
        return decode_errors(min(n, cap), codes, info, pr.a_view.rank, pr.a_view.extents,
                             pr.b_view.rank, pr.b_view.extents, pr.spec, pr.inc_c)
    return []


_FN = {p: getattr(_native.LIB, f"gett_{p}gett_device") for p in "sdcz"}


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


def pack_device(view: TensorView, buf, stream=None):
    """pack (kernel.pack) of a CUDA tensor: a new 1-D tensor of the view's
    elements in canonical order (dimension 0 fastest), stream-ordered."""
    import torch

    if not isinstance(buf, torch.Tensor) or not buf.is_cuda or buf.dim() != 1 or buf.stride(0) != 1:
        raise TypeError("buf must be a contiguous 1-D CUDA tensor")
    n = 1
    for e in view.extents:
        n *= max(int(e), 0)
    out = torch.empty(n, dtype=buf.dtype, device=buf.device)
    if n == 0:
        return out
    if stream is None:
        stream = torch.cuda.current_stream(buf.device)
    with torch.cuda.device(buf.device):
        _native.check(_native.LIB.gett_pack_device(
            view.rank, _native.i64(view.extents), _native.i64(view.increments), view.base_offset,
            buf.shape[0], buf.element_size(), buf.data_ptr(), out.data_ptr(),
            ctypes.c_void_p(stream.cuda_stream)), "pack_device")
    return out
