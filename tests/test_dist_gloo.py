"""CPU tier, world_size 2 over gloo: the N>1 path of bench.py.  Each rank
takes its contiguous slice from the partition planner; the union of the
ranks' outputs (computed here by the CPU oracle) is bit-identical to the
single-rank result -- the analogue of the reference's partition bit-identity
test (proj/tests/test_hetero.cpp:289-308) -- and the max-over-ranks timing
reduction is exact."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, q):
    import oracle as O
    from paper_1711_00289_b200 import gridgen, multigpu
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, T, q_ = gridgen.make_config("c5_50", shape=(24, 32), seed=3)
        b = multigpu.rank_bounds(s, 0.5, world, mode)
        lo, hi = int(b[rank]), int(b[rank + 1])
        d = O.convection("deep", s[lo:hi], T[:, lo:hi], q_[:, lo:hi], first_col=lo)
        sh = O.convection("shallow", s[lo:hi], T[:, lo:hi], q_[:, lo:hi], first_col=lo)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, d.tend_T, d.work, sh.tend_q, sh.work))
        tmax = multigpu.max_over_ranks(float(rank + 1) * 1.5, dist)
        if rank == 0:
            q.put((parts, tmax, list(b)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["balanced", "naive"])
def test_two_rank_partition_is_bit_identical(mode):
    import oracle as O
    from paper_1711_00289_b200 import gridgen
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts, tmax, bounds = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert tmax == 3.0
    s, T, q_ = gridgen.make_config("c5_50", shape=(24, 32), seed=3)
    d = O.convection("deep", s, T, q_)
    sh = O.convection("shallow", s, T, q_)
    assert bounds[0] == 0 and bounds[-1] == s.size
    tT = np.concatenate([p[2] for p in parts], axis=1)
    assert np.array_equal(tT.view(np.int64), d.tend_T.view(np.int64))
    assert np.array_equal(np.concatenate([p[3] for p in parts]), d.work)
    assert np.array_equal(np.concatenate([p[4] for p in parts], axis=1).view(np.int64), sh.tend_q.view(np.int64))
    assert np.array_equal(np.concatenate([p[5] for p in parts]), sh.work)
