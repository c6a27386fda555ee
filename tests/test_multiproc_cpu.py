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
    ids = []
    for step in range(4):
        b = bench.batch_for(step, rank, world, sents)
        ids.append(int(b[0][0]) * 1000 + len(b[0]))
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
    # each rank decodes a different batch at every step (no overlap between ranks)
    for step in range(4):
        assert gathered[0][step] != gathered[1][step]
    # value = all ranks' tokens / max-over-ranks time
    assert mx[0] == 2.0 and sm[1] == 300.0


def test_batches_partition_corpus():
    import bench
    sents = bench.corpus()
    assert len(sents) == bench.CORPUS
    lens = np.array([len(s) for s in sents])
    assert lens.min() >= 5 and lens.max() <= 100
    for world in (1, 2, 4, 8):
        seen = set()
        steps = bench.CORPUS // bench.PER_GPU // world
        for step in range(steps):
            for rank in range(world):
                b = bench.batch_for(step, rank, world, sents)
                assert len(b) == bench.PER_GPU
                key = id(b[0])
                assert key not in seen
                seen.add(key)
        assert len(seen) == bench.CORPUS // bench.PER_GPU
