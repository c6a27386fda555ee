#!/usr/bin/env python
"""Fourth randomized parity sweep: (a) the fp32 precision path (translate_batch on ModelParams,
precision="fp32") against the oracle's fp32 model; (b) wide beams (13..16), long ratios (3.0: the
history block is regrown) and tie-heavy vocabularies (repeated W_vocab rows) on the int8 path;
(c) device lists [0, 0] / [0, 0, 0] (sentence sharding in one process) -- exact.

  python benchmarks/stress_parity4.py [seconds=240] [seed=0]
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
F32 = np.float32
counts = {"fp32": 0, "wide/long/ties": 0, "device lists": 0}


def fail(*a):
    print("MISMATCH", *a)
    sys.exit(1)


while time.time() - t0 < budget:
    mode = int(rng.integers(0, 3))
    dims = dict(src_vocab=int(rng.integers(20, 150)), tgt_vocab=int(rng.integers(20, 500)),
                embed=int(rng.choice([8, 16, 32])), hidden=int(rng.choice([12, 32, 48, 64, 128])),
                attn=int(rng.choice([10, 16, 40, 64])), readout=int(rng.choice([6, 16, 32])))
    s0, aq = str(rng.choice(["transform", "zero"])), str(rng.choice(["current", "previous"]))
    seed = int(rng.integers(1, 1 << 30))
    eos = float(rng.choice([0.0, 0.5, 2.0]))
    params = pb.synthetic_model(pb.Dims(**dims), seed, float(rng.choice([0.1, 0.3])), 0.1, eos, s0, aq)
    tag = (dims, s0, aq, seed, eos)
    if mode == 0:
        om = O.QModel(O.Dims(**dims), params.tensors, s0_mode=s0, attention_query=aq, tier="B", precision="fp32")
        beam = int(rng.choice([1, 2, 4, 6]))
        sents = [rng.integers(3, dims["src_vocab"], int(rng.integers(1, 16))).tolist() for _ in range(int(rng.choice([1, 4, 11])))]
        cfg = pb.DecodeConfig(beam=beam, max_ratio=1.5, precision="fp32")
        got = pb.translate_batch(params, sents, cfg, max_batch=8, return_ids=True)
        for s, (toks, lp) in zip(sents, got):
            et, elp = om.translate(s, beam, 1.5)
            if toks != et or lp != elp:
                fail("fp32", tag, beam, s, toks, et, lp, elp)
        counts["fp32"] += 1
    elif mode == 1:
        dup = int(rng.choice([0, 0, 3, 17]))
        if dup:
            w = params.tensors["out.w_vocab"]
            params.tensors["out.w_vocab"] = np.ascontiguousarray(w[np.arange(dims["tgt_vocab"]) % dup]).astype(F32)
        om = O.QModel(O.Dims(**dims), params.tensors, s0_mode=s0, attention_query=aq, tier="B")
        qm = pb.quantize_model(params)
        beam = int(rng.choice([5, 13, 14, 16]))
        ratio = float(rng.choice([1.5, 3.0]))
        sents = [rng.integers(3, dims["src_vocab"], int(rng.integers(1, 20))).tolist() for _ in range(int(rng.choice([1, 3, 9])))]
        got = pb.translate_batch(qm, sents, pb.DecodeConfig(beam=beam, max_ratio=ratio, precision="int8"), max_batch=8,
                                 return_ids=True)
        for s, (toks, lp) in zip(sents, got):
            et, elp = om.translate(s, beam, ratio)
            if toks != et or lp != elp:
                fail("wide/long/ties", tag, dup, beam, ratio, s, toks, et, lp, elp)
        counts["wide/long/ties"] += 1
    else:
        om = O.QModel(O.Dims(**dims), params.tensors, s0_mode=s0, attention_query=aq, tier="B")
        qm = pb.quantize_model(params)
        beam = int(rng.choice([1, 3, 5]))
        sents = [rng.integers(3, dims["src_vocab"], int(rng.integers(1, 16))).tolist() for _ in range(int(rng.choice([2, 7, 20])))]
        devs = [0] * int(rng.choice([2, 3]))
        got = pb.translate_batch(qm, sents, pb.DecodeConfig(beam=beam, max_ratio=1.5, precision="int8"), max_batch=4,
                                 return_ids=True, devices=devs)
        for s, (toks, lp) in zip(sents, got):
            et, elp = om.translate(s, beam, 1.5)
            if toks != et or lp != elp:
                fail("devices", tag, devs, beam, s, toks, et, lp, elp)
        counts["device lists"] += 1
print(f"stress parity 4 ok: {counts}, {time.time() - t0:.0f} s")
