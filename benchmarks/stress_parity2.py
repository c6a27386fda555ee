#!/usr/bin/env python
"""Second randomized parity sweep (companion of stress_parity.py): (a) larger hidden sizes
(cluster-resident encoder sizes), longer sentences, beams up to 12; (b) ensembles of 2-3 members;
(c) qmath-level products with random shapes (LinearOp paths: fused batch <= 8, cluster
quantization + tcgen05 for wider batches) -- all against the numpy oracle, exact.

  python benchmarks/stress_parity2.py [seconds=240] [seed=0]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_05038_b200 as pb  # noqa: E402
from oracle import qnmt_oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0 = time.time()
F32 = np.float32
counts = {"models": 0, "ensembles": 0, "products": 0}


def fail(*a):
    print("MISMATCH", *a)
    sys.exit(1)


while time.time() - t0 < budget:
    mode = int(rng.integers(0, 3))
    if mode == 0:   # larger models, longer sentences, wider beams
        hidden = int(rng.choice([64, 128, 192, 256, 320]))
        dims = dict(src_vocab=int(rng.integers(30, 200)), tgt_vocab=int(rng.integers(30, 600)),
                    embed=int(rng.choice([16, 32, 64])), hidden=hidden, attn=int(rng.choice([32, 64, 128])),
                    readout=int(rng.choice([16, 32, 64])))
        s0, aq = str(rng.choice(["transform", "zero"])), str(rng.choice(["current", "previous"]))
        seed = int(rng.integers(1, 1 << 30))
        params = pb.synthetic_model(pb.Dims(**dims), seed, float(rng.choice([0.1, 0.3])), 0.1,
                                    float(rng.choice([0.0, 1.0, 2.0])), s0, aq)
        om = O.QModel(O.Dims(**dims), params.tensors, s0_mode=s0, attention_query=aq, tier="B")
        qm = pb.quantize_model(params)
        beam = int(rng.choice([1, 3, 5, 9, 12]))
        n = int(rng.choice([1, 3, 10]))
        sents = [rng.integers(3, dims["src_vocab"], int(rng.integers(1, 50))).tolist() for _ in range(n)]
        cfg = pb.DecodeConfig(beam=beam, max_ratio=float(rng.choice([0.7, 1.5])), precision="int8")
        got = pb.translate_batch(qm, sents, cfg, max_batch=16, return_ids=True)
        for s, (toks, lp) in zip(sents, got):
            et, elp = om.translate(s, beam, cfg.max_ratio)
            if toks != et or lp != elp:
                fail("model", dims, s0, aq, seed, beam, cfg.max_ratio, s, toks, et, lp, elp)
        # the encoder alone (one sentence: persistent / cluster kernels) against the oracle
        eng = pb.Engine(qm, 4, 64, 4)
        st1, att1, s01, _, _ = eng.encode_batch([sents[0]])
        ost, oatt, os0 = om.encode(sents[0])
        if not (np.array_equal(st1.t().cpu().numpy(), ost) and np.array_equal(att1.t().cpu().numpy(), oatt)
                and np.array_equal(s01.t().cpu().numpy(), os0)):
            fail("encoder", dims, s0, aq, seed, sents[0])
        eng.close() if hasattr(eng, "close") else None
        counts["models"] += 1
    elif mode == 1:   # ensembles
        d = dict(src_vocab=int(rng.integers(30, 200)), tgt_vocab=int(rng.integers(30, 300)),
                 embed=int(rng.choice([16, 32])), hidden=int(rng.choice([32, 48, 64])),
                 attn=int(rng.choice([16, 40, 64])), readout=int(rng.choice([16, 32])))
        nm = int(rng.choice([2, 3]))
        seeds = [int(rng.integers(1, 1 << 30)) for _ in range(nm)]
        ps = [pb.synthetic_model(pb.Dims(**d), sd, 0.3, 0.1, 0.6) for sd in seeds]
        qms = [pb.quantize_model(p) for p in ps]
        oms = [O.QModel(O.Dims(**d), p.tensors) for p in ps]
        beam = int(rng.choice([1, 2, 4, 6]))
        srcs = [rng.integers(3, d["src_vocab"], int(rng.integers(1, 16))).tolist() for _ in range(int(rng.choice([1, 5, 18])))]
        got = pb.translate_batch(qms, srcs, pb.DecodeConfig(beam=beam, max_ratio=1.5, precision="int8"),
                                 max_batch=16, return_ids=True)
        for s, g in zip(srcs, got):
            want = O.translate_ensemble(oms, [s] * nm, beam, 1.5)
            if g[0] != want[0] or g[1] != want[1]:
                fail("ensemble", d, seeds, beam, s, g, want)
        counts["ensembles"] += 1
    else:   # quantize + product + dequant with random shapes
        M = int(rng.integers(1, 700))
        K = int(rng.choice([4, 12, 16, 48, 64, 100, 128, 512, 1024, 1040, 2048]))
        N = int(rng.choice([1, 2, 5, 8, 9, 16, 33, 64, 65, 130]))
        w = (rng.normal(0, 1, (M, K)) * 10.0 ** rng.uniform(-2, 1)).astype(F32)
        x = (rng.normal(0, 1, (K, N)) * 10.0 ** rng.uniform(-2, 2)).astype(F32)
        wq = pb.quantize(torch.from_numpy(w).cuda())
        xq = pb.quantize_activations(torch.from_numpy(x).cuda())
        y = pb.qgemm_panel(wq, xq)
        y = y.cpu().numpy() if isinstance(y, torch.Tensor) else np.asarray(y)
        wc, ws = O.quantize(w)
        xc, xs = O.quantize_activations(x)
        want = O.qgemm(wc, ws, xc, xs)
        if not np.array_equal(y, want):
            fail("product", M, K, N, float(np.abs(y - want).max()))
        counts["products"] += 1
print(f"stress parity 2 ok: {counts}, {time.time() - t0:.0f} s")
