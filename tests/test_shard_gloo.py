"""Multi-rank host logic on CPU: two gloo ranks each contract their free-mode
slab (shard.py) with the CPU oracle; the gathered slabs must be bitwise equal
to the single-call result, and bytes outside each slab untouched.  (The GPU
side of each rank is the same dgett call on a sub-view, covered by
test_gpu_parity.py; only one GPU exists per run.)"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2410_06770_b200.shard import bounds, choose_mode, shard_call
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
    spec = choose_mode(w.ext_a, w.ext_b, w.cont_a, w.cont_b, world)
    sargs, skw, lo, hi = shard_call(args, kw, spec, rank, world)
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


def test_choose_mode_prefers_larger_operand():
    # c3: A (33.5 M) is the big operand: shard its mode 0 (256), not B's 384
    s = choose_mode(C3.ext_a, C3.ext_b, C3.cont_a, C3.cont_b, 8)
    assert (s.owner, s.dim) == ("A", 0)
    s = choose_mode(C4.ext_a, C4.ext_b, C4.cont_a, C4.cont_b, 8)
    assert s.extent == 72
    assert bounds(10, 0, 3) == (0, 3) and bounds(10, 2, 3) == (6, 10)


def test_empty_slab_writes_nothing():
    s = choose_mode((3, 4), (4, 2), (1,), (0,), 8)
    args = (2, (3, 4), (4, 1), None, 2, (4, 2), (2, 1), None, 1, (1,), (0,), (0, 1), (2, 1), None)
    sargs, skw, lo, hi = shard_call(args, {}, s, 0, 8)
    assert hi - lo == 0 and 0 in sargs[1] + sargs[5]


# --- split-K across ranks (reduction-parallel, c5) -------------------------

SPLITK = {
    "c1": lambda: C1,
    "c5": lambda: C5.slice_free("A", 0, 0, 4).slice_free("B", 3, 0, 8),
}


def _splitk_worker(rank, world, port, name, out_dir):
    import torch

    from paper_2410_06770_b200.shard import full_call_errors, splitk_contract

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = SPLITK[name]()
    a, b, c = w.buffers()
    args, kw = w.args(a, b, c)
    entry = oracle.oracle_sgett if w.dtype == "s" else oracle.oracle_dgett
    errs = splitk_contract(
        lambda *x, **y: entry(*x, **y) or [], args, kw, rank, world,
        zeros=lambda n: np.zeros(n, dtype=c.dtype), ones=lambda: np.ones(1, dtype=c.dtype),
        reduce=lambda p: dist.reduce(torch.from_numpy(p), dst=0, op=dist.ReduceOp.SUM),
        validate_full=full_call_errors)
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


def test_splitk_pair_choice_and_slices():
    from paper_2410_06770_b200.shard import (accumulate_call, choose_k_pair, k_shard_call,
                                            output_extents, packed_increments)

    # c5 contracted pairs: A dims (1, 2, 4) = (24, 32, 40); 40 % 8 == 0 -> the 40 pair
    assert choose_k_pair(C5.ext_a, C5.cont_a, 8) == 2
    assert choose_k_pair((3, 4), (), 2) is None
    ext_c = output_extents(len(C5.ext_a), C5.ext_a, C5.cont_a, len(C5.ext_b), C5.ext_b, C5.cont_b,
                           C5.perm)
    assert ext_c == (96, 48, 16) and packed_increments(ext_c) == (768, 16, 1)
    a, b, c = object(), object(), object()
    args = (5, C5.ext_a, C5.inc_a, a, 4, C5.ext_b, C5.inc_b, b, 3, C5.cont_a, C5.cont_b, C5.perm,
            C5.inc_c, c)
    lo_hi = []
    for r in range(3):
        sargs, skw, lo, hi = k_shard_call(args, {"offset_c": 7}, 2, r, 3, "P")
        assert sargs[1][4] == sargs[5][0] == hi - lo
        assert skw["offset_a"] == lo * C5.inc_a[4] and skw["offset_b"] == lo * C5.inc_b[0]
        assert skw["offset_c"] == 0 and sargs[13] == "P" and sargs[12] == (768, 16, 1)
        lo_hi.append((lo, hi))
    assert lo_hi == [(0, 13), (13, 26), (26, 40)]
    aargs, akw = accumulate_call(ext_c, "P", "one", C5.inc_c, c, 7)
    assert aargs[:3] == (3, ext_c, (768, 16, 1)) and aargs[4] == 0 and aargs[8] == 0
    assert aargs[11] == (0, 1, 2) and akw["offset_c"] == 7
