#!/usr/bin/env python
"""Randomized guard-band sweep: checked engines (QNMT_CANARY=1: a 0xA5 band after every device
buffer of the engine) on random models / engine sizes / batches / beams, incl. the batch-1
persistent kernels and one-sentence encodes; every decode must leave all bands intact and equal
an unchecked engine's output.  (The write-side memcheck this GPU pool allows.)

  python benchmarks/stress_canary.py [seconds=240] [seed=0]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
lib = _lib.load()


def canaries(e):
    return int(lib.qnmt_engine_check_canaries(e._h, torch.cuda.current_stream().cuda_stream))


t0 = time.time()
n_eng = n_dec = 0
while time.time() - t0 < budget:
    dims = dict(src_vocab=int(rng.integers(20, 200)), tgt_vocab=int(rng.choice([21, 88, 297, 1333, 5000])),
                embed=int(rng.choice([8, 16, 32, 64])), hidden=int(rng.choice([12, 16, 48, 64, 128, 256])),
                attn=int(rng.choice([10, 16, 48, 64, 256])), readout=int(rng.choice([6, 16, 32, 64])))
    params = pb.synthetic_model(pb.Dims(**dims), int(rng.integers(1, 1 << 30)), 0.3, 0.1, float(rng.choice([0.0, 1.5])),
                                str(rng.choice(["transform", "zero"])), str(rng.choice(["current", "previous"])))
    qm = pb.quantize_model(params)
    S, L, B = int(rng.choice([1, 3, 8, 24])), int(rng.choice([4, 20, 40])), int(rng.choice([1, 3, 5, 16]))
    os.environ["QNMT_CANARY"] = "1"
    e = pb.Engine(qm, S, L, B)
    del os.environ["QNMT_CANARY"]
    ref = pb.Engine(qm, S, L, B)
    assert canaries(e) == 0 and canaries(ref) == -1
    for _ in range(4):
        n = int(rng.integers(1, S + 1))
        beam = int(rng.integers(1, B + 1))
        ratio = float(rng.choice([0.5, 1.5, 3.0]))
        sents = [rng.integers(3, dims["src_vocab"], int(rng.integers(1, L + 1))).tolist() for _ in range(n)]
        got = e.translate_ids(sents, beam, ratio)
        bad = canaries(e)
        if bad != 0 or got != ref.translate_ids(sents, beam, ratio):
            print("FAIL", dims, S, L, B, n, beam, ratio, "guard bytes changed:", bad)
            sys.exit(1)
        e.encode_batch(sents[:1])
        if canaries(e) != 0:
            print("FAIL encode", dims, S, L, B, len(sents[0]))
            sys.exit(1)
        n_dec += 1
    n_eng += 1
print(f"stress canary ok: {n_eng} checked engines, {n_dec} decodes, all guard bands intact, {time.time() - t0:.0f} s")
