#!/usr/bin/env python
"""K7 (vocabulary-sharded output projection) against the replicated fused vocab
path at the cfg5 decode step shape: N = 1280 hypotheses, V = 50000, K = 512,
k = 5.  One JSON line.

  python benchmarks/k7.py                       # 1 GPU: shards emulated one after another
  torchrun --nproc-per-node G benchmarks/k7.py  # G GPUs: one shard per rank, NCCL all-gather

Per step and rank the sharded path costs: the shard's fused stats + shard merge
(V / G rows), the all-gather of G x N x 80 bytes, and the combine.  On one GPU
the all-gather is not measured (no peers); the line reports the per-shard
kernels and the combine, and the replicated path's time for the same step."""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1804_05038_b200 import vocab_shard as VS  # noqa: E402


def timed(fn, reps=20):
    """Device time per call (us) of fn's kernels captured in one CUDA graph (no host
    round trips: the raw C-ABI calls, not the Python wrappers that check flags)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e30
    for _ in range(3):
        ev[0].record()
        g.replay()
        ev[1].record()
        ev[1].synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]) / reps * 1e3)
    return best


def timed_eager(fn, reps=20):
    """Per-call time (us) of an eager loop bracketed by CUDA events (collectives)."""
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    ev[1].synchronize()
    return ev[0].elapsed_time(ev[1]) / reps * 1e3


def main():
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    N, V, K, k = 1280, 50000, 512, 5
    rng = np.random.default_rng(0)
    W = torch.from_numpy(rng.integers(-127, 128, (V, K)).astype(np.int8)).cuda()
    X = torch.from_numpy(rng.integers(-127, 128, (N, K)).astype(np.int8)).cuda()
    ws = torch.full((1,), 9000.0, device="cuda")
    xs = torch.full((1,), 500.0, device="cuda")
    bias = torch.from_numpy(rng.normal(0, 0.5, V).astype(np.float32)).cuda()
    live = torch.from_numpy(rng.normal(-10, 3, N)).cuda()
    from paper_1804_05038_b200 import _lib
    f = torch.zeros(4, dtype=torch.int32, device="cuda")
    cs = torch.empty((N, k), dtype=torch.float64, device="cuda")
    ct = torch.empty((N, k), dtype=torch.int32, device="cuda")
    scr = torch.empty(int(_lib.load().qnmt_vocab_candidates_scratch(N, V)), dtype=torch.uint8, device="cuda")

    def rep_call():
        _lib.call("qnmt_vocab_candidates", X.data_ptr(), N, K, xs.data_ptr(), None, W.data_ptr(), V, K, K,
                  ws.data_ptr(), V, bias.data_ptr(), live.data_ptr(), k, scr.data_ptr(), cs.data_ptr(),
                  ct.data_ptr(), f.data_ptr(), torch.cuda.current_stream().cuda_stream)
    rep = timed(rep_call)
    G = world if world > 1 else 8
    lo, hi = VS.shard_bounds(V, G)[rank if world > 1 else 0]
    parts = torch.empty((G * N, VS.part_bytes()), dtype=torch.uint8, device="cuda")
    mine = parts[(rank if world > 1 else 0) * N:((rank if world > 1 else 0) + 1) * N]

    def part_call():
        _lib.call("qnmt_vocab_shard_partials", X.data_ptr(), N, K, xs.data_ptr(), None, W.data_ptr() + lo * K,
                  hi - lo, K, K, ws.data_ptr(), 1 << 30, bias.data_ptr() + 4 * lo, lo, scr.data_ptr(),
                  mine.data_ptr(), f.data_ptr(), torch.cuda.current_stream().cuda_stream)
    part = timed(part_call)
    for g, (a, b) in enumerate(VS.shard_bounds(V, G)):
        VS.shard_partials(X, xs, None, W, ws, bias, a, b, out=parts[g * N:(g + 1) * N])

    def comb_call():
        _lib.call("qnmt_vocab_shard_combine", parts.data_ptr(), G, N, live.data_ptr(), k, cs.data_ptr(),
                  ct.data_ptr(), f.data_ptr(), torch.cuda.current_stream().cuda_stream)
    comb = timed(comb_call)
    line = {"what": "K7 vocab-sharded candidates vs replicated fused path", "N": N, "V": V, "K": K, "k": k,
            "shards": G, "replicated_us": rep, "shard_partials_us": part, "combine_us": comb,
            "exchange_bytes_per_rank": N * VS.part_bytes() * G}
    a = VS.unsharded(X, xs, None, W, ws, bias, live, k)
    b = VS.candidates(X, xs, None, W, ws, bias, live, k, shards=G, group=group)
    line["identical"] = bool(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]))
    if world > 1:
        src = mine.clone()
        ag = timed_eager(lambda: dist.all_gather_into_tensor(parts, src))
        full = timed_eager(lambda: VS.candidates(X, xs, None, W, ws, bias, live, k, group=group))
        line.update({"allgather_us": ag, "sharded_step_us": full})
    else:
        line["sharded_step_us_excl_allgather"] = part + comb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
