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
