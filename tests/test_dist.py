"""Multi-process (world_size 2, gloo on 127.0.0.1) tests of the sharded paths'
host logic: position sharding + the single scalar all-reduce of the evaluator
(SURVEY §8(e) E2), with the oracle standing in for the per-rank GPU partial."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_03532_b200.dist import shard_range, sharded_reduce


@pytest.mark.parametrize("n", [0, 1, 7, 400, 1600])
@pytest.mark.parametrize("ws", [1, 2, 3, 4, 8])
def test_shard_range_partitions(n, ws):
    seen = []
    for r in range(ws):
        b, e = shard_range(n, r, ws)
        assert 0 <= b <= e <= n
        seen.extend(range(b, e))
    assert seen == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(7)
    n, w = 96, 32
    frame = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    probe = (rng.standard_normal((w, w)) + 1j * rng.standard_normal((w, w)))
    offs = np.array([[r, c] for r in (0, 20, 40, 64) for c in (0, 30, 64)], np.int64)
    d = np.abs(rng.standard_normal((len(offs), w, w))) * 5
    return frame, probe, offs, d


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import pft_oracle as O
    frame, probe, offs, d = _problem()
    tot = sharded_reduce(len(offs), lambda b, e: (O.evaluate_shard(frame, probe, offs, d, b, e), e - b))
    out[rank] = (tot[0] / len(offs), tot[1])
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_objective_gloo_world2():
    from oracle import pft_oracle as O
    frame, probe, offs, d = _problem()
    want = O.objective_value(frame, probe, offs, d)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(2):
        phi, count = out[r]
        assert count == len(offs)  # every position evaluated exactly once
        assert abs(phi - want) <= 1e-12 * want


def _e1_worker(rank, ws, port, total, out):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2408_03532_b200.dist import checksum, make_fields, shard_range
    b, e = shard_range(total, rank, ws)
    mine = make_fields(5, b, e, 16, 24, torch.complex64, "cpu")
    blocks = [None] * ws
    dist.all_gather_object(blocks, (b, e, mine.numpy()))
    cs = checksum(mine)
    if rank == 0:
        out["blocks"] = blocks
        out["checksum"] = cs
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,total", [(2, 64), (2, 7), (3, 64)])
def test_e1_field_sharding_gloo(ws, total):
    """E1 (BASELINE configs[1], batch sharded over ranks): the rank blocks
    partition the global batch and their union is bit-identical to the
    single-rank batch (fields depend only on (seed, global index)); the scalar
    checksum all-reduce equals the single-rank value."""
    import torch
    from paper_2408_03532_b200.dist import make_fields
    want = make_fields(5, 0, total, 16, 24, torch.complex64, "cpu").numpy()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_e1_worker, args=(r, ws, port, total, out)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    blocks = out["blocks"]
    got = np.concatenate([blk for (_, _, blk) in blocks])
    assert [(b, e) for (b, e, _) in blocks] == [shard_range(total, r, ws) for r in range(ws)]
    assert got.shape == want.shape and np.array_equal(got, want)
    ref = float(np.sum(np.abs(want.astype(np.complex128)) ** 2))
    assert abs(out["checksum"] - ref) <= 1e-9 * ref
