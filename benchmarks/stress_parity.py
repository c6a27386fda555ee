#!/usr/bin/env python
"""Randomized parity sweep (not part of the test suite: minutes of oracle time): random small
models (dims, flags, EOS bias), random batches, beams and ratios through translate_batch and
translate vs the numpy oracle (Tier B), exact tokens and f64 log-probs.

  python benchmarks/stress_parity.py [seconds=240] [seed=0]
"""
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
cases = sents_done = 0
while time.time() - t0 < budget:
    hidden = int(rng.choice([16, 32, 48, 64, 96, 128, 160, 192]))
    embed = int(rng.choice([16, 32, 48, 64]))
    attn = int(rng.choice([16, 32, 40, 64, 96]))
    readout = int(rng.choice([16, 24, 32, 48]))
    vs, vt = int(rng.integers(20, 300)), int(rng.integers(20, 400))
    s0 = str(rng.choice(["transform", "zero"]))
    aq = str(rng.choice(["current", "previous"]))
    eos = float(rng.choice([0.0, 0.5, 1.5, 3.0]))
    wstd = float(rng.choice([0.05, 0.2, 0.5]))
    dims = dict(src_vocab=vs, tgt_vocab=vt, embed=embed, hidden=hidden, attn=attn, readout=readout)
    seed = int(rng.integers(1, 1 << 30))
    params = pb.synthetic_model(pb.Dims(**dims), seed, wstd, 0.1, eos, s0, aq)
    om = O.QModel(O.Dims(**dims), params.tensors, s0_mode=s0, attention_query=aq, tier="B")
    qm = pb.quantize_model(params)
    beam = int(rng.choice([1, 1, 2, 3, 5, 5, 8]))
    ratio = float(rng.choice([0.5, 1.0, 1.5, 2.5]))
    n = int(rng.choice([1, 2, 9, 17, 33]))
    mb = int(rng.choice([4, 16, 64]))
    sents = [rng.integers(3, vs, int(rng.integers(1, 24))).tolist() for _ in range(n)]
    cfg = pb.DecodeConfig(beam=beam, max_ratio=ratio, precision="int8")
    nstreams = int(rng.choice([1, 3]))
    try:
        got = pb.translate_batch(qm, sents, cfg, max_batch=mb, return_ids=True, streams=nstreams)
    except Exception as exc:   # noqa: BLE001
        print("GPU ERROR", type(exc).__name__, exc)
        print("config", dims, s0, aq, eos, wstd, seed, beam, ratio, n, mb, nstreams)
        for i, s in enumerate(sents):
            try:
                om.translate(s, beam, ratio)
                o = "oracle ok"
            except Exception as oe:   # noqa: BLE001
                o = f"oracle raises {type(oe).__name__}: {oe}"
            try:
                pb.translate_batch(qm, [s], cfg, return_ids=True)
                g1 = "gpu alone ok"
            except Exception as ge:   # noqa: BLE001
                g1 = f"gpu alone raises {type(ge).__name__}"
            print(i, len(s), o, "|", g1)
        sys.exit(2)
    for s, (toks, lp) in zip(sents, got):
        et, elp = om.translate(s, beam, ratio)
        if toks != et or lp != elp:
            print("MISMATCH", dims, s0, aq, eos, wstd, seed, beam, ratio, n, mb, s, toks, et, lp, elp)
            sys.exit(1)
    # one-sentence path (persistent kernels when beam == 1)
    k = int(rng.integers(0, n))
    one = pb.translate_batch(qm, [sents[k]], cfg, return_ids=True)[0]
    if one != got[k]:
        print("MISMATCH one-sentence vs batch", dims, s0, aq, seed, beam, ratio, sents[k], one, got[k])
        sys.exit(1)
    cases += 1
    sents_done += n
print(f"stress parity ok: {cases} random models, {sents_done} sentences, {time.time() - t0:.0f} s")
