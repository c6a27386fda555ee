#!/usr/bin/env python
"""Fifth randomized parity sweep: the batch-1 latency path -- one sentence, beam 1 (persistent
greedy decoder, persistent / cluster-resident encoder) over a wide range of model sizes, sentence
lengths and length ratios, against the oracle, exact; each also with the step-graph engine
(qnmt_set_greedy1(0)).

  python benchmarks/stress_parity5.py [seconds=240] [seed=0]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_05038_b200 as pb  # noqa: E402
from oracle import qnmt_oracle as O  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
lib = _lib.load()
t0 = time.time()
n = 0
while time.time() - t0 < budget:
    dims = dict(src_vocab=int(rng.integers(20, 300)), tgt_vocab=int(rng.choice([21, 100, 297, 1000, 3001, 7000])),
                embed=int(rng.choice([16, 32, 64, 128])), hidden=int(rng.choice([16, 48, 64, 128, 192, 256, 512])),
                attn=int(rng.choice([16, 48, 64, 256, 512])), readout=int(rng.choice([16, 32, 64, 128])))
    s0 = str(rng.choice(["transform", "zero"]))
    seed = int(rng.integers(1, 1 << 30))
    eos = float(rng.choice([0.0, 1.0, 3.0]))
    params = pb.synthetic_model(pb.Dims(**dims), seed, float(rng.choice([0.05, 0.2])), 0.1, eos, s0, "current")
    om = O.QModel(O.Dims(**dims), params.tensors, s0_mode=s0, tier="B")
    qm = pb.quantize_model(params)
    for _ in range(3):
        s = rng.integers(3, dims["src_vocab"], int(rng.integers(1, 60))).tolist()
        ratio = float(rng.choice([0.5, 1.0, 1.5, 3.0]))
        cfg = pb.DecodeConfig(beam=1, max_ratio=ratio, precision="int8")
        want = om.translate(s, 1, ratio)
        got = pb.translate_batch(qm, [s], cfg, return_ids=True)[0]
        old = lib.qnmt_set_greedy1(0)
        got2 = pb.translate_batch(qm, [s], cfg, return_ids=True)[0]
        lib.qnmt_set_greedy1(old)
        if got[0] != want[0] or got[1] != want[1] or got2 != got:
            print("MISMATCH", dims, s0, seed, eos, ratio, s, got, got2, want)
            sys.exit(1)
        n += 1
print(f"stress parity 5 ok: {n} one-sentence greedy decodes, {time.time() - t0:.0f} s")
