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
from paper_2410_06770_b200.workloads import C1, C3, C4


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
