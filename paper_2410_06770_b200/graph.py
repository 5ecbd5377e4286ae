"""CUDA-graph replay of a device-resident xGETT call.

A small contraction (c1: 2.5 MFLOP) costs ~11 µs on the device but ~16 µs of
host work per call (argument checks, validation, plan lookup, launches).  For
a loop that repeats the same call on the same buffers, ``GettGraph`` captures
the native launches of one call once and ``replay()`` re-issues them with a
single graph launch: the same kernels, parameters and results, without the
per-call host work.

    g = GettGraph(dgett_device, rank_a, ext_a, inc_a, a, ..., c)   # runs the call once
    g.replay()                                                    # C += contract(A, B) again

Construction performs the call once (that call builds the plan, the
workspaces and the TMA descriptors, so nothing is allocated during capture)
and captures a second, unexecuted copy.  The captured call reads the buffers'
contents at replay time; the buffers must stay alive and in place.  A DGETT
captured this way runs one CTA per tile (the persistent stream-K schedule's
per-launch publish epochs cannot change between replays).  Worth it for
latency-bound calls: c1 15 -> 8 µs per call.
"""
from __future__ import annotations

from .device import cgett_device, dgett_device, sgett_device, zgett_device

_ENTRIES = (dgett_device, sgett_device, cgett_device, zgett_device)


class GettGraph:
    def __init__(self, entry, *args, **kw):
        import torch

        if entry not in _ENTRIES:
            raise TypeError("entry must be one of the *gett_device functions")
        self._keep = (args, kw)  # the captured pointers must stay valid
        self.graph = torch.cuda.CUDAGraph()
        # the library keeps kernel workspaces per stream: the eager call and the
        # capture run on one side stream, so the capture allocates nothing (the
        # graph then owns that stream's workspaces)
        self._side = side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            errs = entry(*args, **kw)
            if errs:
                raise ValueError(f"the call does not validate: {errs}")
            side.synchronize()
            with torch.cuda.graph(self.graph, stream=side):
                errs = entry(*args, **kw)
        torch.cuda.current_stream().wait_stream(side)
        if errs:
            raise RuntimeError(f"capture failed: {errs}")

    def replay(self) -> None:
        """Re-issue the captured call on the current stream (stream-ordered)."""
        self.graph.replay()
