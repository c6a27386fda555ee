"""World-size-2 gloo tests of the N>1 host logic of bench.py (CPU only):
sentence sharding across ranks (disjoint, covering batches, no collective on
the data path) and the max-over-ranks / sum-over-ranks reductions of the
timing statistics."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    sents = bench.corpus()
    shard = bench.shard_batches(sents, rank, world)
    ids = sorted(i for b in shard for i in b)   # corpus indices this rank decodes
    # per-rank "timing" and token counts reduced exactly as bench.py does
    secs = torch.tensor([1.0 + rank, 100.0 * (rank + 1)], dtype=torch.float64)
    mx = secs.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = secs.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    gathered = [None] * world
    dist.all_gather_object(gathered, ids)
    if rank == 0:
        q.put((gathered, mx.tolist(), sm.tolist()))
    dist.destroy_process_group()


def test_sharding_and_reductions_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, mx, sm = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the ranks' shards are disjoint and together cover the corpus (no collective on the data path)
    assert not set(gathered[0]) & set(gathered[1])
    assert len(gathered[0]) + len(gathered[1]) == 8192
    # value = all ranks' tokens / max-over-ranks time
    assert mx[0] == 2.0 and sm[1] == 300.0


def test_batches_partition_corpus():
    import bench
    sents = bench.corpus()
    assert len(sents) == bench.CORPUS
    lens = np.array([len(s) for s in sents])
    assert lens.min() >= 5 and lens.max() <= 100
    batches = bench.sorted_batches(sents)
    assert all(len(b) == bench.PER_GPU for b in batches)
    flat = [i for b in batches for i in b]
    assert sorted(flat) == list(range(bench.CORPUS))
    blens = [lens[b] for b in batches]
    assert all(blens[k].max() <= blens[k + 1].min() for k in range(len(blens) - 1))   # length-sorted
    for world in (1, 2, 4, 8):
        shards = [bench.shard_batches(sents, r, world) for r in range(world)]
        got = sorted(i for sh in shards for b in sh for i in b)
        assert got == list(range(bench.CORPUS))
        work = [sum(int(np.ceil(1.5 * lens[i])) + 1 for b in sh for i in b) for sh in shards]
        assert max(work) / min(work) < 1.05   # snake-order dealing balances the ranks
    idx = bench.cpu_sample(sents, 8)
    assert len(set(idx)) == 8 and lens[idx].min() < 20 and lens[idx].max() > 85


def test_product_splitter_matches_bench_and_covers():
    """translate_batch(..., devices=[...]) shards with decoder.shard_batches: the same
    snake-order deal of length-sorted batches as bench.py, disjoint and covering for
    any device count, ragged last batch included."""
    import bench
    from paper_1804_05038_b200.decoder import shard_batches
    sents = bench.corpus()
    lens = [len(s) for s in sents]
    for world in (1, 2, 3, 4, 8):
        prod = shard_batches(lens, bench.PER_GPU, world)
        assert prod == [bench.shard_batches(sents, r, world) for r in range(world)]
    for n, mb, world in ((1, 256, 4), (7, 3, 2), (1000, 256, 3), (513, 256, 8)):
        ls = list(np.random.default_rng(n).integers(1, 120, n))
        sh = shard_batches(ls, mb, world)
        flat = sorted(i for r in sh for b in r for i in b)
        assert flat == list(range(n))
        assert all(len(b) <= mb for r in sh for b in r)


def _product_worker(rank, world, port, q):
    """Each rank derives its own shard from the product splitter (no data exchange);
    the gathered shards are disjoint and cover the corpus."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_05038_b200.decoder import shard_batches
    ls = list(np.random.default_rng(3).integers(5, 101, 999))
    mine = sorted(i for b in shard_batches(ls, 64, world)[rank] for i in b)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


def test_product_splitter_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_product_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert not set(gathered[0]) & set(gathered[1])
    assert sorted(gathered[0] + gathered[1]) == list(range(999))
