#!/usr/bin/env python
"""Peaked log-softmax rows at BASELINE size: a large EOS bias makes one logit lead by 20..60, so
lse - max = log(1 + eps) with eps down to < 2^-52.  Decodes against the oracle:
tokens, and the f64 log-prob difference in ulps of the oracle's value."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_05038_b200 as pb  # noqa: E402
from oracle import qnmt_oracle as O  # noqa: E402

rng = np.random.default_rng(1)
dims = dict(src_vocab=32000, tgt_vocab=50000, embed=512, hidden=1024, attn=2048, readout=512)
for eos in (10.0, 20.0, 30.0, 37.0, 40.0, 60.0):
    params = pb.synthetic_model(pb.Dims(**dims), 1804, 0.05, 0.0, eos)
    om = O.QModel(O.Dims(**dims), params.tensors, tier="B")
    qm = pb.quantize_model(params)
    worst, worst_abs, tok_bad, n = 0.0, 0.0, 0, 0
    for beam in (1, 5):
        sents = [rng.integers(3, 32000, int(rng.integers(1, 6))).tolist() for _ in range(4)]
        got = pb.translate_batch(qm, sents, pb.DecodeConfig(beam=beam, max_ratio=1.5, precision="int8"), return_ids=True)
        for s, (toks, lp) in zip(sents, got):
            et, elp = om.translate(s, beam, 1.5)
            tok_bad += toks != et
            if lp != elp:
                u = abs(lp - elp) / np.spacing(abs(elp)) if elp != 0 else float("inf")
                worst = max(worst, u)
                worst_abs = max(worst_abs, abs(lp - elp))
            n += 1
    print(f"eos_bias {eos:5.1f}: {n} decodes, token mismatches {tok_bad}, worst log-prob difference {worst_abs:.2e} absolute "
          f"({worst_abs / 2.220446049250313e-16:.1f} ulps of 1.0; {worst:.3g} ulps of the value), "
          f"example log-prob {elp!r}")
