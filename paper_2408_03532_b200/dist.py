"""Multi-GPU plumbing for the paths that shard.

* Batched PFTs (E1): independent fields; each rank transforms its own fields,
  no collective on the data path.
* Forward-model / residual evaluator (E2): scan positions are split into
  contiguous blocks, each rank evaluates its block with libpftg, and ONE
  all-reduce of the per-rank scalars (NCCL over NVLink on GPUs, gloo in the CPU
  tests) produces Phi = total / N. Results depend on the rank count only
  through the order of that final sum.
* The ePIE sweep (E3) does not shard (every position updates the shared probe
  and overlapping patches): replicas only.
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_range(n: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous block [begin, end) of n items owned by `rank` (sizes differ by <= 1)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("shard_range: bad rank/world")
    base, rem = divmod(n, world_size)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def sharded_reduce(n: int, partial: Callable[[int, int], Sequence[float]], device=None,
                   group=None) -> list[float]:
    """Evaluate partial(begin, end) on this rank's shard and sum the scalars over
    all ranks with a single all_reduce (float64). Returns the global sums."""
    rank, ws = world()
    b, e = shard_range(n, rank, ws)
    vals = [float(v) for v in partial(b, e)]
    if ws == 1:
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [float(v) for v in t.cpu()]


def evaluate_sharded(frame, probe, offsets, d, plan=None, d_crop=None, group=None):
    """Phi (solver.cpp:89-102) and the band residual over all positions, sharded
    by position across the ranks of the default group (BASELINE configs[4])."""
    from .solver import evaluate

    n = len(offsets)

    def part(b, e):
        fs, bs = evaluate(frame, probe, offsets, d, (b, e), plan, d_crop)
        return (fs, bs if bs is not None else 0.0)

    fs, bs = sharded_reduce(n, part, device=frame.device, group=group)
    return fs / n, (bs / n if plan is not None else None)
