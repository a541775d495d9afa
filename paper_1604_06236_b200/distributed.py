"""Signal sharding across the GPUs of one box (one process per GPU).

The batched solves are embarrassingly parallel over signals that share one
node set: rank r of G takes a contiguous block of rows, builds the
(deterministic) plan locally, and solves with no communication.  The only
collective is an optional final gather of the outputs to rank 0 (NCCL over
NVLink on a B200 box; gloo in the CPU tests).  SURVEY.md section 8(e).
"""

from __future__ import annotations


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) rows of a `batch`-row operand owned by `rank` (contiguous, balanced)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def local_rows(x, world: int, rank: int):
    """This rank's rows of a [batch, n] operand (a view, no copy)."""
    lo, hi = shard_bounds(x.shape[0], world, rank)
    return x[lo:hi]


def gather_rows(local, batch: int, world: int, rank: int, group=None, dst: int = 0):
    """Collect every rank's [rows_r, n] block into the full [batch, n] tensor on
    `dst` (returns None elsewhere).  Uneven shards are padded to the largest
    block for the collective and trimmed afterwards."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    if local.is_complex():  # collectives move the interleaved (re, im) doubles
        full = gather_rows(torch.view_as_real(local).reshape(local.shape[0], 2 * local.shape[1]), batch, world, rank,
                           group, dst)
        return None if full is None else torch.view_as_complex(full.reshape(batch, -1, 2).contiguous())
    n = local.shape[1]
    rows = [shard_bounds(batch, world, r) for r in range(world)]
    cap = max(hi - lo for lo, hi in rows)
    buf = torch.zeros((cap, n), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, rows)], dim=0)


def max_over_ranks(value: float, world: int, device=None, group=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max over ranks)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
