"""The signal-sharded multi-GPU path with the PRODUCT kernels:
two ranks, each solving its contiguous block of a job's signals through the
public API on cuda:0 (the only GPU this build gets; the ranks' kernels never
wait on one another — host-side gloo collectives only), the outputs gathered
to rank 0 with gather_rows and compared bitwise with one process solving the
whole job.  Also bench.py's multi-rank leg (timing, max over ranks, the timed
gather) in its oversubscribed test mode."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(P, job):
    from oracle import nfft_oracle as O

    return O.make_inputs(P, 0.3, job, 16046)


def _rank_main(rank, world, port, P, job, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1604_06236_b200 as nf
        from paper_1604_06236_b200.distributed import gather_rows, local_rows

        t, data = _inputs(P, job)
        plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
        mine = local_rows(torch.from_numpy(data), world, rank).cuda()
        x5 = nf.refine_type5(plan, mine, passes=1) if mine.shape[0] else mine
        x4 = nf.refine_type4(plan, mine, passes=1) if mine.shape[0] else mine
        f5 = gather_rows(x5.cpu(), job, world, rank)
        f4 = gather_rows(x4.cpu(), job, world, rank)
        if rank == 0:
            q.put((f5.numpy(), f4.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,job", [(4096, 64), (4096, 37), (1 << 16, 40), (1000, 9), (64, 3)])
def test_two_rank_product_path_bitwise_equals_single_process(P, job):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, P, job, q)) for r in range(2)]
    for p in procs:
        p.start()
    f5, f4 = q.get(timeout=600)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0

    import paper_1604_06236_b200 as nf

    t, data = _inputs(P, job)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2), device=0)
    whole = torch.from_numpy(data).cuda()
    ref5 = nf.refine_type5(plan, whole, passes=1).cpu().numpy()
    ref4 = nf.refine_type4(plan, whole, passes=1).cpu().numpy()
    assert f5.shape == (job, P) and f4.shape == (job, P)
    if P <= 256 or (job // 2 >= 16) == (job >= 16):
        # same kernel family on both sides: bitwise
        assert np.array_equal(f5, ref5) and np.array_equal(f4, ref4)
    else:
        # a shard below 16 signals runs the signal-major chains (type-5 bitwise, type-4 to rounding)
        assert np.array_equal(f5, ref5)
        assert np.abs(f4 - ref4).max() <= 1e-13 * np.abs(ref4).max()


def test_bench_two_ranks_oversubscribed():
    """bench.py --gpus 2 re-launches itself under torch.distributed.run and reports
    n_gpus 2, the max-over-ranks step time and the timed gather (gloo test mode)."""
    cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--oversubscribe", "--config", "c2",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=REPO)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 64 and line["config"]["signals_per_gpu"] == 32
    assert line["gather"]["rank0_rows_ok"] is True
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert max(line["parity"].values()) <= 1e-10
