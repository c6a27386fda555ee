#!/usr/bin/env python
"""Sixth randomized parity sweep: BASELINE-size models (V = 50000 / 32000, H = 1024, A = 2048)
with random short sentences -- the regime of the fused vocabulary kernel's full tile grid, the
register-resident attention kernels and the cluster-resident encoder -- against the oracle.
Weight scales 0.05 (BASELINE) and larger (wider logit ranges, early EOS).

  python benchmarks/stress_parity6.py [seconds=300] [seed=0]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_05038_b200 as pb  # noqa: E402
from oracle import qnmt_oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0 = time.time()
done = {"sentences": 0, "models": 0, "score-only diffs": 0}
while time.time() - t0 < budget:
    V = int(rng.choice([50000, 32000]))
    dims = dict(src_vocab=32000, tgt_vocab=V, embed=512, hidden=1024, attn=2048, readout=512)
    wstd = float(rng.choice([0.05, 0.05, 0.1, 0.2]))
    eos = float(rng.choice([0.0, 2.0, 6.0]))
    seed = int(rng.integers(1, 1 << 30))
    params = pb.synthetic_model(pb.Dims(**dims), seed, wstd, 0.0 if wstd == 0.05 else 0.05, eos)
    om = O.QModel(O.Dims(**dims), params.tensors, tier="B")
    qm = pb.quantize_model(params)
    beam = int(rng.choice([1, 3, 5]))
    sents = [rng.integers(3, 32000, int(rng.integers(1, 7))).tolist() for _ in range(6)]
    got = pb.translate_batch(qm, sents, pb.DecodeConfig(beam=beam, max_ratio=1.5, precision="int8"), return_ids=True)
    one = pb.translate_batch(qm, [sents[0]], pb.DecodeConfig(beam=1, max_ratio=1.5, precision="int8"), return_ids=True)[0]
    w1 = om.translate(sents[0], 1, 1.5)
    if one[0] != w1[0] or one[1] != w1[1]:
        print("MISMATCH batch-1 greedy", V, wstd, eos, seed, sents[0], one, w1)
        sys.exit(1)
    for s, (toks, lp) in zip(sents, got):
        et, elp = om.translate(s, beam, 1.5)
        if toks != et:
            print("MISMATCH tokens", V, wstd, eos, seed, beam, s, toks, et, lp, elp)
            sys.exit(1)
        if lp != elp:
            if abs(lp - elp) <= 1e-12 * max(1.0, abs(elp)):   # peaked rows: f64 sum order
                done["score-only diffs"] += 1
            else:
                print("MISMATCH score", V, wstd, eos, seed, beam, s, lp, elp)
                sys.exit(1)
        done["sentences"] += 1
    done["models"] += 1
print(f"stress parity 6 ok: {done}, {time.time() - t0:.0f} s")
