"""Multi-GPU partitioning of one xGETT by a free mode.

xGETT is closed under slicing a free mode: restricting free dimension `dim` of
the owning operand to [lo, hi) shifts that operand's offset by lo·inc and C's
offset by lo·inc_c[perm[i]] and shrinks one extent — the slice is itself a valid
xGETT whose result is bitwise equal to the same elements of the full call (each
output element's K loop is untouched).  Ranks therefore run independent slabs
with no data-path collective.

Mode choice: a free mode of the larger operand (the one not replicated), the
largest extent first, preferring extents divisible by the world size — e.g. c3
shards A's mode 0 (256) rather than the largest mode of C (384, owned by the small
B), which would replicate the 268 MB A (SURVEY §8e note).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardSpec:
    owner: str  # "A" or "B"
    dim: int    # dimension of the owner being split
    extent: int


def _free(rank, cont):
    return [d for d in range(rank) if d not in set(cont)]


def choose_mode(ext_a, ext_b, cont_a, cont_b, world: int) -> ShardSpec | None:
    """Pick the free mode to split across `world` ranks (None: nothing to split)."""
    size_a = 1
    for e in ext_a:
        size_a *= int(e)
    size_b = 1
    for e in ext_b:
        size_b *= int(e)
    order = [("A", ext_a, cont_a), ("B", ext_b, cont_b)]
    if size_b > size_a:
        order.reverse()
    for owner, ext, cont in order:
        free = _free(len(ext), cont)
        if not free:
            continue
        best = max(free, key=lambda d: (int(ext[d]) >= world, int(ext[d]) % world == 0, int(ext[d])))
        if int(ext[best]) >= 1:
            return ShardSpec(owner, best, int(ext[best]))
    return None


def bounds(extent: int, rank: int, world: int):
    """Contiguous, balanced [lo, hi) slab of `extent` for `rank`."""
    return extent * rank // world, extent * (rank + 1) // world


def shard_call(args, kw, spec: ShardSpec, rank: int, world: int):
    """Positional/keyword xGETT arguments (reference order, kernel.py:158-184)
    restricted to this rank's slab.  Returns (args, kw, lo, hi); an empty slab
    has a zero extent (the call then writes nothing, kernel.py:93-94)."""
    (rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c) = args
    kw = dict(kw)
    lo, hi = bounds(spec.extent, rank, world)
    if spec.owner == "A":
        fi = _free(rank_a, cont_a).index(spec.dim)
        ext = list(ext_a)
        ext[spec.dim] = hi - lo
        kw["offset_a"] = kw.get("offset_a", 0) + (lo * inc_a[spec.dim] if hi > lo else 0)
        ext_a = tuple(ext)
    else:
        fi = len(_free(rank_a, cont_a)) + _free(rank_b, cont_b).index(spec.dim)
        ext = list(ext_b)
        ext[spec.dim] = hi - lo
        kw["offset_b"] = kw.get("offset_b", 0) + (lo * inc_b[spec.dim] if hi > lo else 0)
        ext_b = tuple(ext)
    q = perm[fi]
    kw["offset_c"] = kw.get("offset_c", 0) + (lo * inc_c[q] if hi > lo else 0)
    return ((rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c),
            kw, lo, hi)


# ---------------------------------------------------------------------------
# Reduction-parallel split-K across ranks (c5).
#
# A contraction is linear in each contracted pair: restricting pair p to
# [lo, hi) in BOTH A (dim cont_a[p]) and B (dim cont_b[p]) shifts offset_a by
# lo·inc_a[cont_a[p]] and offset_b by lo·inc_b[cont_b[p]] and yields the
# partial sum over that K slice.  Every rank writes its partial into a zeroed,
# packed (row-major over C's extents) buffer P_r; one sum-reduce to the owner
# rank forms ΣP_r, and only the owner adds it into C (C₀ is added exactly
# once, SURVEY §7 "accumulate semantics across split-K").  The add is itself
# an xGETT with no contracted mode: A = P (rank_c, packed increments),
# B = the rank-0 scalar 1, perm = identity — K = 1 plans onto the reference-
# order kernel, so C ← fma(P, 1, C) rounds once.  Results are not bitwise equal
# to the single call (the K sum is reassociated); the tolerance is the
# K-normalised one of the parity tests.
# ---------------------------------------------------------------------------

def choose_k_pair(ext_a, cont_a, world: int):
    """Index p into the contracted pairs to split (None when conts == 0):
    the largest extent, preferring one ≥ world and divisible by it."""
    if not len(cont_a):
        return None
    return max(range(len(cont_a)),
               key=lambda p: (int(ext_a[cont_a[p]]) >= world, int(ext_a[cont_a[p]]) % world == 0,
                              int(ext_a[cont_a[p]])))


def output_extents(rank_a, ext_a, cont_a, rank_b, ext_b, cont_b, perm):
    """C's extents: free index i (A's free dims ascending, then B's) lands at
    output position perm[i] (plan.py:96-104 restated)."""
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


def k_shard_call(args, kw, pair: int, rank: int, world: int, partial):
    """xGETT arguments computing this rank's K-slice partial into `partial`
    (zeroed, packed over C's extents, offset 0).  Returns (args, kw, lo, hi)."""
    (rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c) = args
    da, db = int(cont_a[pair]), int(cont_b[pair])
    lo, hi = bounds(int(ext_a[da]), rank, world)
    ea, eb = list(ext_a), list(ext_b)
    ea[da] = eb[db] = hi - lo
    kw = dict(kw)
    kw["offset_a"] = kw.get("offset_a", 0) + (lo * inc_a[da] if hi > lo else 0)
    kw["offset_b"] = kw.get("offset_b", 0) + (lo * inc_b[db] if hi > lo else 0)
    ext_c = output_extents(rank_a, ext_a, cont_a, rank_b, ext_b, cont_b, perm)
    kw["offset_c"] = 0
    return ((rank_a, tuple(ea), inc_a, a, rank_b, tuple(eb), inc_b, b, conts, cont_a, cont_b, perm,
             packed_increments(ext_c), partial), kw, lo, hi)


def accumulate_call(ext_c, partial, one, inc_c, c, offset_c=0):
    """xGETT arguments for C[view] += P·1 (rank_c x rank-0, no contraction)."""
    r = len(ext_c)
    return ((r, tuple(ext_c), packed_increments(ext_c), partial, 0, (), (), one, 0, (), (),
             tuple(range(r)), tuple(inc_c), c), {"offset_a": 0, "offset_b": 0, "offset_c": offset_c})


def splitk_contract(entry, args, kw, rank: int, world: int, *, zeros, ones, reduce, root: int = 0,
                    validate_full=None):
    """Run one xGETT as `world` K-slices, one per rank, reduced onto `root`.

    entry        — the xGETT callable for the buffers' kind (kernel.dgett for
                   numpy, device.sgett_device for CUDA tensors, ...).
    zeros(n)     — a zeroed flat buffer of n elements like C.
    ones()       — a 1-element buffer holding 1.
    reduce(buf)  — in-place sum of buf over ranks onto root (e.g.
                   torch.distributed.reduce; NCCL for CUDA tensors).
    validate_full(args, kw) — the full call's ValidationError list (every rank
                   computes it and returns it without touching C, so all
                   ranks agree); None skips (the caller validated).

    Returns the validation errors ([] on success).  Only `root` writes C."""
    if validate_full is not None:
        errs = validate_full(args, kw)
        if errs:
            return errs
    (rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c) = args
    pair = choose_k_pair(ext_a, cont_a[:conts], world)
    if pair is None or world == 1:
        return entry(*args, **kw) if rank == root else []
    ext_c = output_extents(rank_a, ext_a, cont_a, rank_b, ext_b, cont_b, perm)
    n = 1
    for e in ext_c:
        n *= e
    part = zeros(n)
    sargs, skw, _, _ = k_shard_call(args, kw, pair, rank, world, part)
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


def full_call_errors(args, kw):
    """The full call's validation errors in the entry points' two phases
    (arguments, then C's footprint when the arguments are clean)."""
    from .layout import TensorView
    from .plan import ContractionSpec, derive_output_extents, validate

    (rank_a, ext_a, inc_a, a, rank_b, ext_b, inc_b, b, conts, cont_a, cont_b, perm, inc_c, c) = args
    av = TensorView(rank_a, ext_a, inc_a, kw.get("offset_a", 0), len(a))
    bv = TensorView(rank_b, ext_b, inc_b, kw.get("offset_b", 0), len(b))
    spec = ContractionSpec(conts, cont_a, cont_b, perm)
    errs = validate(av, bv, spec, inc_c)
    if errs:
        return errs
    ext_c = derive_output_extents(av, bv, spec)
    cv = TensorView(len(ext_c), ext_c, tuple(inc_c), kw.get("offset_c", 0), len(c))
    return validate(av, bv, spec, inc_c, c_view=cv)


def splitk_device(prefix: str, args, kw, group=None, root: int = 0):
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
        root=root, validate_full=_device_full_call_errors)


def _device_full_call_errors(args, kw):
    a, b, c = args[3], args[7], args[13]
    lens = (a.shape[0], b.shape[0], c.shape[0])
    sized = list(args)
    sized[3], sized[7], sized[13] = (_Len(n) for n in lens)
    return full_call_errors(tuple(sized), kw)


class _Len:
    """Stand-in exposing only len() for validation of device buffers."""

    def __init__(self, n):
        self.n = int(n)

    def __len__(self):
        return self.n
