"""World-size-2 (gloo, CPU) tests of the signal-sharded multi-GPU path:
shard bounds, local solves on each rank's rows, gather to rank 0, and the
max-over-ranks timing reduction used by bench.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_06236_b200.distributed import gather_rows, local_rows, max_over_ranks, shard_bounds


def test_shard_bounds_cover_exactly():
    for batch in (1, 7, 64, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(batch, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import nfft_oracle as O

        P = 32
        t, data = O.make_inputs(P, 0.3, batch, 16040)
        plan = O.Plan.build(t, O.damping(1e-15, P, 2), 2)  # every rank builds the same plan
        mine = local_rows(torch.from_numpy(data), world, rank)
        out = torch.stack([torch.from_numpy(O.refine5(plan, row.numpy(), 1)) for row in mine]) \
            if mine.shape[0] else torch.zeros((0, P), dtype=torch.complex128)
        full = gather_rows(out, batch, world, rank)
        tmax = max_over_ranks(float(rank + 1), world)
        if rank == 0:
            ref = np.stack([O.refine5(plan, row, 1) for row in data])
            q.put((np.array_equal(full.numpy(), ref), tmax))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [1, 5, 8])
def test_two_rank_sharded_solve_matches_single_process(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    same, tmax = q.get(timeout=10)
    assert same and tmax == 2.0
