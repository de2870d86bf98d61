"""Multi-GPU plumbing for the paths that shard.

* Batched PFTs (E1): independent fields. A global batch of B fields is split
  into contiguous blocks (``shard_range``); every field is generated from
  (seed, global field index) (``make_fields``), so a rank's block is
  bit-identical to the same slice of the single-rank batch; each rank
  transforms its block (``pft_fwd_adj_sharded``) with no collective on the
  data path -- the only collective is the scalar max of the step time /
  a scalar checksum.
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


def field_seed(seed: int, index: int) -> int:
    """Generator seed of global field ``index`` (E1: independent of the rank count)."""
    return (int(seed) * 1_000_003 + int(index)) & ((1 << 63) - 1)


def make_fields(seed: int, begin: int, end: int, n1: int, n2: int | None = None,
                dtype=torch.complex64, device="cuda") -> torch.Tensor:
    """Fields [begin, end) of a seeded batch of i.i.d. standard-normal real and
    imaginary parts (BASELINE configs[1]); field f depends only on (seed, f)."""
    n2 = n1 if n2 is None else n2
    real = torch.float32 if dtype == torch.complex64 else torch.float64
    out = torch.empty((end - begin, n1, n2), dtype=dtype, device=device)
    g = torch.Generator(device=device)
    for i, f in enumerate(range(begin, end)):
        g.manual_seed(field_seed(seed, f))
        re = torch.randn((n1, n2), generator=g, device=device, dtype=real)
        im = torch.randn((n1, n2), generator=g, device=device, dtype=real)
        out[i] = torch.complex(re, im)
    return out


def pft_fwd_adj_sharded(plan, fields: torch.Tensor):
    """E1 step on this rank's block: band = pft_apply_2d(fields), back =
    pft_adjoint_2d(band) (BASELINE configs[1]: the adjoint of the forward output)."""
    from .pft import pft_adjoint_2d, pft_apply_2d
    band = pft_apply_2d(plan, fields)
    return band, pft_adjoint_2d(plan, band)


def checksum(t: torch.Tensor, group=None) -> float:
    """Global scalar checksum sum |x|^2 over every rank's block (one float64
    all-reduce): equal to the single-rank value up to summation order."""
    v = torch.tensor([float(torch.sum(torch.view_as_real(t).double() ** 2))], dtype=torch.float64,
                     device=t.device if dist.get_backend(group) == "nccl" else "cpu") \
        if dist.is_available() and dist.is_initialized() else None
    if v is None:
        return float(torch.sum(torch.view_as_real(t).double() ** 2))
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    return float(v.item())
