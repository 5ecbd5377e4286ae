"""Strided view descriptors — the host-side mirror of gett.layout.

Mirrors /root/reference/pkg/src/gett/layout.py: ``TensorView`` (:55-105) with
the same structural checks (ValueError on construction), ``footprint``
(:108-125), ``num_elements`` (:21-26), ``contiguous_increments`` (:29-40).
The per-element iteration devices (view_offsets, CoordCounter) are not part
of the product: the GPU kernels decode coordinates from the planner's folded
mode groups instead.
"""
from __future__ import annotations

from dataclasses import dataclass, field


def num_elements(extents) -> int:
    """Product of extents; rank 0 holds one element."""
    n = 1
    for e in extents:
        n *= int(e)
    return n


def contiguous_increments(extents) -> tuple:
    """Packed first-dimension-fastest increments [1, e0, e0*e1, ...]."""
    inc = []
    step = 1
    for e in extents:
        inc.append(step)
        step *= int(e)
    return tuple(inc)


@dataclass(frozen=True)
class TensorView:
    """A strided window into a flat buffer of ``buffer_len`` elements.

    Construction checks structure only (lengths match the rank, rank and
    buffer_len non-negative, base_offset non-negative); value problems are
    reported by validation as coded errors.
    """

    rank: int
    extents: tuple
    increments: tuple
    base_offset: int = 0
    buffer_len: int = field(default=0)

    def __post_init__(self):
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))
        object.__setattr__(self, "increments", tuple(int(i) for i in self.increments))
        if self.rank < 0:
            raise ValueError(f"rank must be non-negative, got {self.rank}")
        if len(self.extents) != self.rank or len(self.increments) != self.rank:
            raise ValueError(
                f"rank {self.rank} view needs {self.rank} extents and increments, "
                f"got {len(self.extents)} and {len(self.increments)}")
        if self.base_offset < 0:
            raise ValueError(f"base_offset must be non-negative, got {self.base_offset}")
        if self.buffer_len < 0:
            raise ValueError(f"buffer_len must be non-negative, got {self.buffer_len}")

    @classmethod
    def contiguous(cls, extents, base_offset: int = 0) -> "TensorView":
        extents = tuple(int(e) for e in extents)
        return cls(len(extents), extents, contiguous_increments(extents), base_offset,
                   base_offset + num_elements(extents))

    @property
    def is_empty(self) -> bool:
        return any(e == 0 for e in self.extents)

    @property
    def size(self) -> int:
        return num_elements(self.extents)


def footprint(view: TensorView) -> tuple:
    """(lowest, highest) offset touched, relative to base_offset; extent-0
    dimensions contribute nothing."""
    lo = hi = 0
    for ext, inc in zip(view.extents, view.increments):
        if ext <= 0:
            continue
        span = inc * (ext - 1)
        if span < 0:
            lo += span
        else:
            hi += span
    return lo, hi
