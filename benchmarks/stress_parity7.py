#!/usr/bin/env python
"""Seventh randomized parity sweep: ENGINE REUSE -- a few long-lived models, hundreds of
translate_batch / translate calls each with changing batch sizes, beams, ratios, stream counts
and sentence lengths (step graphs cached per (sentences, beam), history blocks regrown, engines
swapped for longer sentences), from several host threads at once -- against cached oracle results.

  python benchmarks/stress_parity7.py [seconds=240] [seed=0]
"""
import concurrent.futures as cf
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_05038_b200 as pb  # noqa: E402
from oracle import qnmt_oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0 = time.time()
models = []
for k in range(3):
    dims = dict(src_vocab=60 + 20 * k, tgt_vocab=[90, 400, 2500][k], embed=[16, 32, 32][k], hidden=[32, 64, 128][k],
                attn=[16, 48, 64][k], readout=[16, 32, 32][k])
    params = pb.synthetic_model(pb.Dims(**dims), 500 + k, 0.3, 0.1, [0.5, 1.5, 1.0][k])
    om = O.QModel(O.Dims(**dims), params.tensors, tier="B")
    pool = [rng.integers(3, dims["src_vocab"], int(rng.integers(1, 40))).tolist() for _ in range(60)]
    models.append((pb.quantize_model(params), om, pool, {}))


def want(mi, si, beam, ratio):
    _, om, pool, cache = models[mi]
    key = (si, beam, ratio)
    if key not in cache:
        cache[key] = om.translate(pool[si], beam, ratio)
    return cache[key]


def one_call(args):
    mi, idx, beam, ratio, mb, streams = args
    qm, _, pool, _ = models[mi]
    got = pb.translate_batch(qm, [pool[i] for i in idx], pb.DecodeConfig(beam=beam, max_ratio=ratio, precision="int8"),
                             max_batch=mb, return_ids=True, streams=streams)
    return args, got


calls = 0
while time.time() - t0 < budget:
    jobs = []
    for _ in range(int(rng.choice([1, 2, 3]))):   # concurrent callers (the engine pool is thread-safe)
        mi = int(rng.integers(0, 3))
        idx = rng.integers(0, 60, int(rng.choice([1, 2, 7, 30]))).tolist()
        jobs.append((mi, idx, int(rng.choice([1, 2, 5, 9])), float(rng.choice([0.5, 1.5, 3.0])),
                     int(rng.choice([1, 4, 16, 64])), int(rng.choice([1, 2, 3]))))
    with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        for args, got in ex.map(one_call, jobs):
            mi, idx, beam, ratio, mb, streams = args
            for i, (toks, lp) in zip(idx, got):
                et, elp = want(mi, i, beam, ratio)
                if toks != et or lp != elp:
                    print("MISMATCH", args, i, toks, et, lp, elp)
                    sys.exit(1)
            calls += 1
print(f"stress parity 7 ok: {calls} translate_batch calls on 3 long-lived models, {time.time() - t0:.0f} s")
