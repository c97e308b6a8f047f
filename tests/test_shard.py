"""Multi-rank host logic on CPU (gloo, world_size 2): stripe partitioning, the
max-over-ranks timing reduction, and that sharded outputs equal a single run
(each rank encodes its stripes with the oracle-free generator + C++ compiler's
bitmatrix semantics; no GPU needed)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_02692_b200.shard import aggregate_throughput, max_over_ranks, stripe_range


def test_stripe_range_cover():
    for world in (1, 2, 3, 8):
        for total in (0, 1, 7, 1024, 8192):
            spans = [stripe_range(r, world, total=total) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    assert stripe_range(3, 8, per_rank=1024) == (3072, 4096)
    with pytest.raises(ValueError):
        stripe_range(2, 2, total=4)


def test_aggregate():
    assert aggregate_throughput([10, 10], [1.0, 2.0]) == 10.0


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    lo, hi = stripe_range(rank, world, per_rank=3)
    # each rank: its stripes' data, XOR-reduced (a stand-in per-rank result), and a fake time
    acc = np.zeros(64, dtype=np.uint8)
    for s in range(lo, hi):
        acc ^= synth.stripe_data(9, s, 2, 64).reshape(2, 64)[0]
    t = max_over_ranks(0.5 + rank, dist)
    buf = torch.from_numpy(acc.astype(np.int64))
    gathered = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    if rank == 0:
        q.put((t, [g.numpy().astype(np.uint8) for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 1.5                                  # max over ranks
    import synth
    whole = np.zeros(64, dtype=np.uint8)
    for s in range(6):
        whole ^= synth.stripe_data(9, s, 2, 64).reshape(2, 64)[0]
    assert (parts[0] ^ parts[1] == whole).all()      # shards partition the stripes exactly
