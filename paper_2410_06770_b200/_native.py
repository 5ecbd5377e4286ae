"""ctypes binding of libgett_b200.so — the C ABI declared in include/gett_b200.h.

There is no Python or CPU fallback: if the library is missing this module
raises at import, and any CUDA failure inside a call is raised as
GettRuntimeError.  Only plain pointers and sizes cross the boundary.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GETT_LIB_PATH") or os.path.join(_HERE, "libgett_b200.so")

# every symbol include/gett_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "gett_dgett", "gett_sgett", "gett_dgett_device", "gett_sgett_device",
    "gett_zgett", "gett_cgett", "gett_zgett_device", "gett_cgett_device",
    "gett_validate", "gett_derive_output_extents",
    "gett_zero_view_d", "gett_zero_view_s", "gett_zero_view_d_device", "gett_zero_view_s_device",
    "gett_set_kernel", "gett_set_split_k", "gett_set_pipeline", "gett_set_stream_k", "gett_set_tma", "gett_set_bulk", "gett_set_wide", "gett_set_pdl", "gett_set_pair", "gett_set_complex_embed", "gett_last_kernel", "gett_last_error",
    "gett_launch_count", "gett_release_caches", "gett_abi_version",
    "gett_dgett_multi", "gett_sgett_multi", "gett_set_devices", "gett_set_multi", "gett_last_multi",
    "gett_multi_schedule", "gett_pack", "gett_pack_device", "gett_set_kr",
    "gett_plan_create", "gett_execute", "gett_execute_device", "gett_plan_destroy",
)

ERR_INFO_WORDS = 6
E_CUDA, E_INVALID_ARG, E_NOMEM, E_UNSUPPORTED = -1, -2, -3, -4


class GettRuntimeError(RuntimeError):
    """A CUDA or internal failure reported by the native library."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    i64p = ctypes.POINTER(ctypes.c_int64)
    i32p = ctypes.POINTER(ctypes.c_int32)
    vp = ctypes.c_void_p
    gett_args = [ctypes.c_int, i64p, i64p, vp, ctypes.c_int64, ctypes.c_int64,
                 ctypes.c_int, i64p, i64p, vp, ctypes.c_int64, ctypes.c_int64,
                 ctypes.c_int, i64p, i64p, ctypes.c_int, i64p,
                 ctypes.c_int, i64p, vp, ctypes.c_int64, ctypes.c_int64]
    for name in ("gett_dgett", "gett_sgett", "gett_zgett", "gett_cgett"):
        f = getattr(lib, name)
        f.restype = ctypes.c_int
        f.argtypes = gett_args + [i32p, i64p, ctypes.c_int]
    for name in ("gett_dgett_device", "gett_sgett_device", "gett_zgett_device", "gett_cgett_device"):
        f = getattr(lib, name)
        f.restype = ctypes.c_int
        f.argtypes = gett_args + [vp, i32p, i64p, ctypes.c_int]
    for name in ("gett_dgett_multi", "gett_sgett_multi"):
        f = getattr(lib, name)
        f.restype = ctypes.c_int
        f.argtypes = gett_args + [ctypes.c_int, i32p, i32p, i64p, ctypes.c_int]
    lib.gett_multi_schedule.restype = ctypes.c_int
    lib.gett_multi_schedule.argtypes = [
        ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64,
        ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64,
        ctypes.c_int, i64p, i64p, ctypes.c_int, i64p, ctypes.c_int, i64p,
        ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, i64p, i32p, i64p, ctypes.c_int]
    lib.gett_plan_create.restype = ctypes.c_int
    lib.gett_plan_create.argtypes = [
        ctypes.c_char, ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64,
        ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64,
        ctypes.c_int, i64p, i64p, ctypes.c_int, i64p, ctypes.c_int, i64p,
        ctypes.c_int64, ctypes.c_int64, ctypes.c_int, i32p, ctypes.POINTER(ctypes.c_void_p), i32p, i64p,
        ctypes.c_int]
    lib.gett_execute.restype = ctypes.c_int
    lib.gett_execute.argtypes = [vp, vp, vp, vp]
    lib.gett_execute_device.restype = ctypes.c_int
    lib.gett_execute_device.argtypes = [vp, vp, vp, vp, vp]
    lib.gett_plan_destroy.restype = None
    lib.gett_plan_destroy.argtypes = [vp]
    lib.gett_pack.restype = ctypes.c_int
    lib.gett_pack.argtypes = [ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                              vp, vp]
    lib.gett_pack_device.restype = ctypes.c_int
    lib.gett_pack_device.argtypes = lib.gett_pack.argtypes + [vp]
    lib.gett_set_devices.restype = ctypes.c_int
    lib.gett_set_devices.argtypes = [ctypes.c_int, i32p]
    lib.gett_set_multi.restype = ctypes.c_int
    lib.gett_set_multi.argtypes = [ctypes.c_int]
    lib.gett_last_multi.restype = ctypes.c_char_p
    lib.gett_last_multi.argtypes = []
    lib.gett_validate.restype = ctypes.c_int
    lib.gett_validate.argtypes = [
        ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64,
        ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64,
        ctypes.c_int, i64p, i64p, ctypes.c_int, i64p, ctypes.c_int, i64p,
        ctypes.c_int, ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64,
        i32p, i64p, ctypes.c_int]
    lib.gett_derive_output_extents.restype = ctypes.c_int
    lib.gett_derive_output_extents.argtypes = [ctypes.c_int, i64p, ctypes.c_int, i64p,
                                               ctypes.c_int, i64p, i64p, i64p, i64p]
    for name, dev in (("gett_zero_view_d", False), ("gett_zero_view_s", False),
                      ("gett_zero_view_d_device", True), ("gett_zero_view_s_device", True)):
        f = getattr(lib, name)
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_int, i64p, i64p, ctypes.c_int64, ctypes.c_int64, vp] + ([vp] if dev else [])
    lib.gett_set_kernel.restype = ctypes.c_int
    lib.gett_set_kernel.argtypes = [ctypes.c_char_p]
    lib.gett_set_split_k.restype = ctypes.c_int
    lib.gett_set_split_k.argtypes = [ctypes.c_int]
    lib.gett_set_pipeline.restype = ctypes.c_int
    lib.gett_set_pipeline.argtypes = [ctypes.c_int]
    lib.gett_set_stream_k.restype = ctypes.c_int
    lib.gett_set_stream_k.argtypes = [ctypes.c_int]
    lib.gett_set_tma.restype = ctypes.c_int
    lib.gett_set_tma.argtypes = [ctypes.c_int]
    lib.gett_set_bulk.restype = ctypes.c_int
    lib.gett_set_bulk.argtypes = [ctypes.c_int]
    lib.gett_set_wide.restype = ctypes.c_int
    lib.gett_set_wide.argtypes = [ctypes.c_int]
    lib.gett_set_pdl.restype = ctypes.c_int
    lib.gett_set_pdl.argtypes = [ctypes.c_int]
    lib.gett_set_kr.restype = ctypes.c_int
    lib.gett_set_kr.argtypes = [ctypes.c_int]
    lib.gett_set_pair.restype = ctypes.c_int
    lib.gett_set_pair.argtypes = [ctypes.c_int]
    lib.gett_set_complex_embed.restype = ctypes.c_int
    lib.gett_set_complex_embed.argtypes = [ctypes.c_int]
    lib.gett_last_kernel.restype = ctypes.c_char_p
    lib.gett_last_kernel.argtypes = []
    lib.gett_last_error.restype = ctypes.c_char_p
    lib.gett_last_error.argtypes = []
    lib.gett_launch_count.restype = ctypes.c_int64
    lib.gett_launch_count.argtypes = []
    lib.gett_release_caches.restype = None
    lib.gett_release_caches.argtypes = []
    lib.gett_abi_version.restype = ctypes.c_int
    lib.gett_abi_version.argtypes = []
    return lib


LIB = _load()


def i64(seq):
    """A ctypes int64 array holding seq (length >= 1 so the pointer is valid)."""
    seq = [int(x) for x in seq]
    return (ctypes.c_int64 * max(1, len(seq)))(*seq)


def check(rc: int, what: str) -> int:
    """Raise for negative native status codes; pass error counts through."""
    if rc >= 0:
        return rc
    msg = LIB.gett_last_error().decode(errors="replace")
    kind = {E_CUDA: "CUDA failure", E_INVALID_ARG: "invalid argument", E_NOMEM: "out of device memory",
            E_UNSUPPORTED: "unsupported descriptor"}.get(rc, f"status {rc}")
    raise GettRuntimeError(f"{what}: {kind}: {msg}")


def set_kernel(name: str) -> None:
    """Select the kernel family: auto | ref | tiled | serial (see gett_b200.h)."""
    if LIB.gett_set_kernel(name.encode()) != 0:
        raise ValueError(f"unknown kernel {name!r}")


def set_split_k(split: int) -> None:
    if LIB.gett_set_split_k(int(split)) != 0:
        raise ValueError(f"bad split {split}")


def set_pipeline(slabs: int) -> None:
    """Host-path transfer/compute overlap: -1 auto, 0 off, n >= 2 slabs."""
    if LIB.gett_set_pipeline(int(slabs)) != 0:
        raise ValueError(f"bad slab count {slabs}")


def set_stream_k(on: bool) -> None:
    """DGETT persistent stream-K schedule on (default) / off."""
    if LIB.gett_set_stream_k(1 if on else 0) != 0:
        raise ValueError(f"bad stream-K switch {on}")


def set_tma(on: bool) -> None:
    """SGETT TMA-fed operands for affine views on (default) / off."""
    if LIB.gett_set_tma(1 if on else 0) != 0:
        raise ValueError(f"bad TMA switch {on}")


def set_bulk(on: bool) -> None:
    """DGETT bulk-add epilogue (whole C row runs per request) on (default) / off."""
    if LIB.gett_set_bulk(1 if on else 0) != 0:
        raise ValueError(f"bad bulk switch {on}")


def set_pdl(on: bool) -> None:
    """Programmatic dependent launch of the k-run SGETT kernel and the split-K
    reduce (each scheduled while its predecessor in the stream drains) on
    (default) / off."""
    if LIB.gett_set_pdl(1 if on else 0) != 0:
        raise ValueError(f"bad PDL switch {on}")


_WIDE = {"off": 0, "auto": 1, "force": 2}


def set_wide(mode: str = "auto", mixed: bool = False, tail: bool = True) -> None:
    """SGETT wide CTA-pair kernel (256 x 256 per cluster): "off", "auto"
    (default), "force"; mixed=True issues one tf32 + one bf16 MMA per 8 k (the
    k-run kernel's mixed split) instead of the three tf32 MMAs of the 3xTF32
    truncation split (the default); tail=False never cuts a partial last wave's
    tiles into two K halves."""
    code = _WIDE.get(mode, -1) | (4 if mixed else 0) | (0 if tail else 8)
    if mode not in _WIDE or LIB.gett_set_wide(code) != 0:
        raise ValueError(f"bad wide mode {mode!r}")


def set_pair(on: bool) -> None:
    """SGETT CTA-pair (cta_group::2) kernel on / off (default off)."""
    if LIB.gett_set_pair(1 if on else 0) != 0:
        raise ValueError(f"bad pair switch {on}")


def set_complex_embed(on: bool) -> None:
    """cgett/zgett tiled path: one embedded real GETT (default) or four real GETTs."""
    if LIB.gett_set_complex_embed(1 if on else 0) != 0:
        raise ValueError(f"bad complex-embed switch {on}")


def i32(seq):
    """A ctypes int32 array holding seq (length >= 1 so the pointer is valid)."""
    vals = [int(x) for x in seq] or [0]
    return (ctypes.c_int32 * len(vals))(*vals)


def set_devices(devices) -> None:
    """Default device list of the host entry points (dgett/sgett run across
    these devices with the unchanged reference signature); None or () = the
    current device.  A device may repeat (devices=(0, 0): two lanes on one GPU)."""
    devs = [] if devices is None else [int(d) for d in devices]
    check(LIB.gett_set_devices(len(devs), i32(devs)), "set_devices")


def set_kr(mode: str = "auto", fused: bool = False, pair: bool = True, mixed: bool = True) -> None:
    """SGETT k-run kernel: "off", "auto" (default) or "force" (whenever it
    applies); fused=True reduces split-K partials inside the kernel instead of
    with the separate reduce kernel (the default); pair=False never runs pairs
    of X tiles as cta_group::2 clusters (the default does when the tiling
    allows, with two k runs per k-block when they fit); mixed=False issues the
    three tf32 MMAs of the 3xTF32 truncation split instead of one tf32 + one
    bf16 MMA per 8 k (the default)."""
    code = ({"off": 0, "auto": 1, "force": 2}[mode] | (4 if fused else 0) | (0 if pair else 8)
            | (0 if mixed else 16))
    check(LIB.gett_set_kr(code), "set_kr")


def set_multi(strategy: str, staged: bool = False) -> None:
    """Multi-device schedule: "auto" (default), "slabs" or "splitk" (tests);
    staged=True: the split-K reduce copies the partials with cudaMemcpyPeer
    instead of loading them from the peers."""
    code = {"auto": 0, "slabs": 1, "splitk": 2}[strategy] | (4 if staged else 0)
    check(LIB.gett_set_multi(code), "set_multi")


def last_multi() -> str:
    """The last host call's multi-device schedule ("none": one device)."""
    return LIB.gett_last_multi().decode()


def last_kernel() -> str:
    return LIB.gett_last_kernel().decode()


def launch_count() -> int:
    return int(LIB.gett_launch_count())


def release_caches() -> None:
    LIB.gett_release_caches()
