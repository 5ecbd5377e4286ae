"""Multi-rank host logic on CPU: gloo ranks each contract their part of the
NATIVE multi-device schedule (gett_multi_schedule — the partition
gett_dgett_multi runs in one process) with the CPU oracle: free-mode slabs
gathered must be bitwise equal to the single-call result with bytes outside
each slab untouched; split-K partials reduced onto rank 0 must match within
the K-normalised tolerance.  (The GPU side of each rank is the same dgett
call on a sub-view, covered by test_gpu_parity.py / test_gpu_multi.py; only
one GPU exists per run.)"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2410_06770_b200.shard import schedule, shard_call
from paper_2410_06770_b200.workloads import C1, C3, C4, C5


SMALL = {
    "c1": lambda: C1,
    "c3": lambda: C3.slice_free("A", 0, 0, 8).slice_free("A", 2, 0, 8),
    "c4": lambda: C4.slice_free("A", 0, 0, 4).slice_free("A", 1, 0, 8).slice_free("B", 3, 0, 2),
}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_dir):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = SMALL[name]()
    a, b, c = w.buffers()
    args, kw = w.args(a, b, c)
    sched = schedule(args, kw, world, "slabs")
    assert sched.strategy == "slabs"
    sargs, skw, lo, hi = shard_call(args, kw, sched, rank)
    if hi > lo:
        oracle.oracle_dgett(*sargs, **skw)
    t = torch.from_numpy(c)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    if rank == 0:
        np.savez(os.path.join(out_dir, "parts.npz"), *[o.numpy() for o in out])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "c3", "c4"])
def test_two_rank_slabs_equal_full_call(name, tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _port(), name, str(tmp_path)), nprocs=world, join=True)
    z = np.load(tmp_path / "parts.npz")
    parts = [z[k] for k in z.files]
    w = SMALL[name]()
    a, b, c = w.buffers()
    c0 = c.copy()
    args, kw = w.args(a, b, c)
    oracle.oracle_dgett(*args, **kw)
    # merge: each rank changed only its slab; take changed bytes from each
    merged = c0.copy()
    for p in parts:
        changed = p.view(np.uint64) != c0.view(np.uint64)
        merged[changed] = p[changed]
    assert merged.tobytes() == c.tobytes()


class _Len:
    def __init__(self, n):
        self.n = n

    def __len__(self):
        return self.n


def _sched(w, world, strategy="auto"):
    args, kw = w.args(_Len(w.len_a), _Len(w.len_b), _Len(w.len_c))
    return schedule(args, kw, world, strategy)


def test_native_schedule_of_the_baseline_configs():
    """c2/c3/c4 cut C's outermost free mode (A's mode 0) in 128-row granules;
    c5 (6 output tiles) splits its largest contracted pair (40); c1 is too
    small to split; one rank is always one device."""
    from paper_2410_06770_b200.workloads import C2

    s = _sched(C2, 8)
    assert (s.strategy, s.owner, s.dim, s.n) == ("slabs", "A", 0, 8)
    assert s.ranges == tuple((512 * i, 512 * (i + 1)) for i in range(8))
    s = _sched(C3, 4)
    assert (s.strategy, s.owner, s.dim) == ("slabs", "A", 0) and s.ranges[-1] == (192, 256)
    s = _sched(C4, 8)
    assert (s.strategy, s.owner, s.dim, s.n) == ("slabs", "A", 0, 8)
    assert sum(hi - lo for lo, hi in s.ranges) == 72
    s = _sched(C5, 8)
    assert (s.strategy, s.dim, s.n) == ("splitk", 2, 8) and s.ranges[0] == (0, 5)
    assert _sched(C1, 8).strategy == "one"
    assert _sched(C2, 1).strategy == "one"
    # forced strategies, and more ranks than the cut mode has rows
    s = _sched(C1, 3, "splitk")
    assert s.strategy == "splitk" and s.dim == 1 and s.ranges == ((0, 13), (13, 26), (26, 40))
    s = _sched(C1, 64, "slabs")
    assert s.strategy == "slabs" and s.n == 20  # C1's outermost C mode is B's (20)


def test_schedule_returns_validation_errors():
    args = (2, (2, 3), (3, 1), _Len(6), 2, (2, 3), (3, 1), _Len(6), 1, (1,), (0,), (0, 1), (2, 1),
            _Len(4))
    errs = schedule(args, {}, 2)
    assert isinstance(errs, list) and errs[0].code.name == "ExtentMismatch"


def test_empty_slab_writes_nothing():
    args = (2, (3, 4), (4, 1), _Len(12), 2, (4, 2), (2, 1), _Len(8), 1, (1,), (0,), (0, 1), (2, 1),
            _Len(6))
    s = schedule(args, {}, 8, "slabs")
    assert s.n == 3
    sargs, skw, lo, hi = shard_call(args, {}, s, 5)
    assert hi - lo == 0 and 0 in sargs[1] + sargs[5]


# --- split-K across ranks (reduction-parallel, c5) -------------------------

SPLITK = {
    "c1": lambda: C1,
    "c5": lambda: C5.slice_free("A", 0, 0, 4).slice_free("B", 3, 0, 8),
}


def _splitk_worker(rank, world, port, name, out_dir):
    import torch

    from paper_2410_06770_b200.shard import splitk_contract

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = SPLITK[name]()
    a, b, c = w.buffers()
    args, kw = w.args(a, b, c)
    entry = oracle.oracle_sgett if w.dtype == "s" else oracle.oracle_dgett
    errs = splitk_contract(
        lambda *x, **y: entry(*x, **y) or [], args, kw, rank, world,
        zeros=lambda n: np.zeros(n, dtype=c.dtype), ones=lambda: np.ones(1, dtype=c.dtype),
        reduce=lambda p: dist.reduce(torch.from_numpy(p), dst=0, op=dist.ReduceOp.SUM))
    assert errs == []
    np.save(os.path.join(out_dir, f"c{rank}.npy"), c)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("c1", 2), ("c5", 2), ("c5", 3)])
def test_splitk_ranks_reduce_onto_owner(name, world, tmp_path):
    mp.spawn(_splitk_worker, args=(world, _port(), name, str(tmp_path)), nprocs=world, join=True)
    w = SPLITK[name]()
    a, b, c = w.buffers()
    c0 = c.copy()
    args, kw = w.args(a, b, c)
    (oracle.oracle_sgett if w.dtype == "s" else oracle.oracle_dgett)(*args, **kw)
    root = np.load(tmp_path / "c0.npy")
    # C0 added exactly once, only on the owner; non-owners leave C untouched
    for r in range(1, world):
        assert np.load(tmp_path / f"c{r}.npy").tobytes() == c0.tobytes()
    k = w.size_k
    amax = np.abs(a).max() * np.abs(b).max()
    tol = 1e-5 if w.dtype == "s" else 1e-12
    assert np.abs(root.astype(np.float64) - c).max() <= tol * k * amax + 0.0
    assert not np.array_equal(root, c0)


def test_splitk_slices_and_accumulate_call():
    from paper_2410_06770_b200.shard import (accumulate_call, k_shard_call, output_extents,
                                            packed_increments)

    ext_c = output_extents(len(C5.ext_a), C5.ext_a, C5.cont_a, len(C5.ext_b), C5.ext_b, C5.cont_b,
                           C5.perm)
    assert ext_c == (96, 48, 16) and packed_increments(ext_c) == (768, 16, 1)
    a, b, c = object(), object(), object()
    args = (5, C5.ext_a, C5.inc_a, a, 4, C5.ext_b, C5.inc_b, b, 3, C5.cont_a, C5.cont_b, C5.perm,
            C5.inc_c, c)
    sched = _sched(C5, 3)
    assert sched.ranges == ((0, 13), (13, 26), (26, 40))
    for r in range(3):
        lo, hi = sched.range(r)
        sargs, skw = k_shard_call(args, {"offset_c": 7}, sched.dim, lo, hi, "P")
        assert sargs[1][4] == sargs[5][0] == hi - lo
        assert skw["offset_a"] == lo * C5.inc_a[4] and skw["offset_b"] == lo * C5.inc_b[0]
        assert skw["offset_c"] == 0 and sargs[13] == "P" and sargs[12] == (768, 16, 1)
    aargs, akw = accumulate_call(ext_c, "P", "one", C5.inc_c, c, 7)
    assert aargs[:3] == (3, ext_c, (768, 16, 1)) and aargs[4] == 0 and aargs[8] == 0
    assert aargs[11] == (0, 1, 2) and akw["offset_c"] == 7
