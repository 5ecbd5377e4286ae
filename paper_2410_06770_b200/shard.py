"""Multi-rank partitioning of one xGETT for one-process-per-GPU launchers
(torchrun), on the NATIVE multi-device schedule.

The partition is the one the in-call multi-device path runs
(gett_dgett_multi, include/gett_b200.h): ``schedule()`` asks the native
planner (gett_multi_schedule — validation, mode choice and ranges, no CUDA)
and the helpers here only rewrite arguments:

* slabs — xGETT is closed under slicing a free mode: restricting dimension
  `dim` of the owning operand to [lo, hi) shifts that operand's offset by
  lo·inc and C's by lo·inc_c[perm[i]]; each rank runs its slab, no collective.
  Calls writing disjoint C footprints may run concurrently.
* split-K — the contraction is linear in each contracted pair: restricting
  pair p to [lo, hi) in BOTH A and B yields the partial sum over that K
  slice.  Every rank writes its partial into a zeroed, packed buffer; one
  sum-reduce (NCCL for device buffers) lands ΣP on the owner, which alone adds
  it into C (C₀ is added exactly once).  The add is itself an xGETT with no
  contracted mode (C ← P·1 + C, K = 1).  Results equal the one-call result
  within the K-normalised tolerance (the K sum is reassociated).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _native

_STRATEGY = {"auto": 0, "slabs": 1, "splitk": 2}


@dataclass(frozen=True)
class Schedule:
    strategy: str          # "one" (one device / rank 0 alone), "slabs", "splitk"
    n: int                 # ranks used (ranks >= n get empty work)
    owner: str | None      # slabs: "A" or "B", the operand whose mode is cut
    dim: int               # slabs: that operand's dimension; split-K: the pair index
    ranges: tuple          # per used rank: (lo, hi) of that dimension / pair

    def range(self, rank: int):
        return self.ranges[rank] if rank < self.n else (0, 0)


def _len(buf):
    return int(buf.shape[0]) if hasattr(buf, "shape") else len(buf)


def schedule(args, kw, world: int, strategy: str = "auto"):
    """The native multi-device schedule of xGETT arguments (reference order,
    kernel.py:158-184) over `world` ranks, or the full call's ValidationError
    list when it is invalid (every rank computes the same answer, so all ranks
    return the errors with C untouched).  Needs no GPU."""
    from .plan import decode_errors, error_capacity
    from .layout import TensorView
    from .plan import ContractionSpec

    (rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c) = args
    av = TensorView(rank_a, ext_a, inc_a, kw.get("offset_a", 0), _len(a))
    bv = TensorView(rank_b, ext_b, inc_b, kw.get("offset_b", 0), _len(b))
    spec = ContractionSpec(conts, cont_a, cont_b, perm)
    inc_c = tuple(int(i) for i in inc_c)
    i64 = _native.i64
    cap = error_capacity(av.rank, bv.rank, spec.conts) + 8
    codes = (ctypes.c_int32 * cap)()
    info = (ctypes.c_int64 * (cap * _native.ERR_INFO_WORDS))()
    out = (ctypes.c_int64 * (4 + 2 * world))()
    n = _native.LIB.gett_multi_schedule(
        av.rank, i64(av.extents), i64(av.increments), av.base_offset, av.buffer_len,
        bv.rank, i64(bv.extents), i64(bv.increments), bv.base_offset, bv.buffer_len,
        spec.conts, i64(spec.cont_a), i64(spec.cont_b), len(spec.perm), i64(spec.perm),
        len(inc_c), i64(inc_c), int(kw.get("offset_c", 0)), _len(c), int(world),
        _STRATEGY[strategy], out, codes, info, cap)
    _native.check(n, "multi_schedule")
    if n:
        return decode_errors(min(n, cap), codes, info, av.rank, av.extents, bv.rank, bv.extents,
                             spec, inc_c)
    kind = {0: "one", 1: "slabs", 2: "splitk"}[int(out[0])]
    used = int(out[1])
    ranges = tuple((int(out[4 + 2 * i]), int(out[5 + 2 * i])) for i in range(used)) if kind != "one" else ()
    owner = {0: "A", 1: "B"}.get(int(out[2])) if kind == "slabs" else None
    return Schedule(kind, used, owner, int(out[3]), ranges)


def _free(rank, cont):
    return [d for d in range(rank) if d not in set(cont)]


def shard_call(args, kw, sched: Schedule, rank: int):
    """xGETT arguments restricted to `rank`'s slab of a "slabs" schedule.
    Returns (args, kw, lo, hi); an empty slab has a zero extent (the call
    then writes nothing, kernel.py:93-94)."""
    assert sched.strategy == "slabs"
    (rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c) = args
    kw = dict(kw)
    lo, hi = sched.range(rank)
    dim = sched.dim
    if sched.owner == "A":
        fi = _free(rank_a, cont_a).index(dim)
        ext = list(ext_a)
        ext[dim] = hi - lo
        kw["offset_a"] = kw.get("offset_a", 0) + (lo * inc_a[dim] if hi > lo else 0)
        ext_a = tuple(ext)
    else:
        fi = len(_free(rank_a, cont_a)) + _free(rank_b, cont_b).index(dim)
        ext = list(ext_b)
        ext[dim] = hi - lo
        kw["offset_b"] = kw.get("offset_b", 0) + (lo * inc_b[dim] if hi > lo else 0)
        ext_b = tuple(ext)
    q = perm[fi]
    kw["offset_c"] = kw.get("offset_c", 0) + (lo * inc_c[q] if hi > lo else 0)
    return ((rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c),
            kw, lo, hi)


def output_extents(rank_a, ext_a, cont_a, rank_b, ext_b, cont_b, perm):
    """C's extents: free index i (A's free dims ascending, then B's) lands at
    output position perm[i] (plan.py:119-127 restated)."""
    free = [int(ext_a[d]) for d in _free(rank_a, cont_a)] + [int(ext_b[d]) for d in _free(rank_b, cont_b)]
    out = [0] * len(free)
    for i, e in enumerate(free):
        out[int(perm[i])] = e
    return tuple(out)


def packed_increments(ext):
    inc, s = [0] * len(ext), 1
    for d in range(len(ext) - 1, -1, -1):
        inc[d] = s
        s *= int(ext[d])
    return tuple(inc)


def k_shard_call(args, kw, pair: int, lo: int, hi: int, partial):
    """xGETT arguments computing the K slice [lo, hi) of contracted pair
    `pair` into `partial` (zeroed, packed over C's extents, offset 0)."""
    (rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c) = args
    da, db = int(cont_a[pair]), int(cont_b[pair])
    ea, eb = list(ext_a), list(ext_b)
    ea[da] = eb[db] = hi - lo
    kw = dict(kw)
    kw["offset_a"] = kw.get("offset_a", 0) + (lo * inc_a[da] if hi > lo else 0)
    kw["offset_b"] = kw.get("offset_b", 0) + (lo * inc_b[db] if hi > lo else 0)
    ext_c = output_extents(rank_a, ext_a, cont_a, rank_b, ext_b, cont_b, perm)
    kw["offset_c"] = 0
    return ((rank_a, tuple(ea), inc_a, a, rank_b, tuple(eb), inc_b, b, conts, cont_a, cont_b, perm,
             packed_increments(ext_c), partial), kw)


def accumulate_call(ext_c, partial, one, inc_c, c, offset_c=0):
    """xGETT arguments for C[view] += P·1 (rank_c x rank-0, no contraction)."""
    r = len(ext_c)
    return ((r, tuple(ext_c), packed_increments(ext_c), partial, 0, (), (), one, 0, (), (),
             tuple(range(r)), tuple(inc_c), c), {"offset_a": 0, "offset_b": 0, "offset_c": offset_c})


def splitk_contract(entry, args, kw, rank: int, world: int, *, zeros, ones, reduce, root: int = 0,
                    strategy: str = "splitk"):
    """Run one xGETT as K slices, one per rank, reduced onto `root`, on the
    native schedule (strategy "splitk" forces the K split when the call has a
    contracted pair of extent >= 2; "auto" lets the planner choose, and a
    non-split-K answer runs the whole call on root).

    entry        — the xGETT callable for the buffers' kind (kernel.dgett for
                   numpy, device.sgett_device for CUDA tensors, the oracle in
                   the CPU tests).
    zeros(n)     — a zeroed flat buffer of n elements like C.
    ones()       — a 1-element buffer holding 1.
    reduce(buf)  — in-place sum of buf over ranks onto root (e.g.
                   torch.distributed.reduce; NCCL for CUDA tensors); called by
                   every rank, also those with an empty slice.

    Returns the full call's validation errors ([] on success; every rank
    returns the same list).  Only `root` writes C."""
    sched = schedule(args, kw, world, strategy)
    if isinstance(sched, list):
        return sched
    (rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c) = args
    if sched.strategy != "splitk":
        return entry(*args, **kw) if rank == root else []
    ext_c = output_extents(rank_a, ext_a, cont_a, rank_b, ext_b, cont_b, perm)
    n = 1
    for e in ext_c:
        n *= e
    part = zeros(n)
    lo, hi = sched.range(rank)
    if hi > lo:
        sargs, skw = k_shard_call(args, kw, sched.dim, lo, hi, part)
        errs = entry(*sargs, **skw)
        if errs:
            raise RuntimeError(f"K-slice of a valid call failed validation: {errs}")
    reduce(part)
    if rank == root:
        aargs, akw = accumulate_call(ext_c, part, ones(), inc_c, c, kw.get("offset_c", 0))
        errs = entry(*aargs, **akw)
        if errs:
            raise RuntimeError(f"split-K accumulate failed validation: {errs}")
    return []


def splitk_device(prefix: str, args, kw, group=None, root: int = 0, strategy: str = "splitk"):
    """split-K of one xGETT over the ranks of a torch.distributed group whose
    buffers are CUDA tensors: each rank contracts its K slice on its own GPU
    (device.<prefix>gett_device, stream-ordered) and ncclReduce(sum) lands
    the partials on `root`, which adds them into C.  Every rank passes the same
    arguments (its own device copies of A and B; C is only read/written on
    root).  Returns the full call's validation errors ([] on success)."""
    import torch
    import torch.distributed as dist

    from . import device

    entry = getattr(device, f"{prefix}gett_device")
    c = args[13]
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    return splitk_contract(
        entry, args, kw, rank, world,
        zeros=lambda n: torch.zeros(n, dtype=c.dtype, device=c.device),
        ones=lambda: torch.ones(1, dtype=c.dtype, device=c.device),
        reduce=lambda p: dist.reduce(p, dst=root, op=dist.ReduceOp.SUM, group=group),
        root=root, strategy=strategy)
