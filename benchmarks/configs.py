#!/usr/bin/env python
"""Secondary measurements for the other BASELINE.json configs (one JSON line each).

  cfg1  qgemm_panel W[3072x1024] x X[1024xB], B in {1, 64}: device time of the
        product kernel (CUDA events), cold L2 (64 rotating weight copies,
        ~200 MB > 126 MB L2), GB/s over the algorithmic bytes and int-op/s.
  cfg2  Network.encode, l = 50 (latency).
  cfg3  translate, greedy, 50 steps, V = 32000 (latency, tokens/s).
  cfg4  64 sentences, l ~ U[10, 80], beam 5 (sentences/s, tokens/s).
  host  per-step floor: one sentence, l = 100, beam 5 (151 steps).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402


def peaks():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except OSError:
        return {"hbm_gbs": 6650.0}


def cfg1(reps=64):
    out = []
    w = np.random.default_rng(1804).normal(0, 0.05, (3072, 1024)).astype(np.float32)
    wq = pb.quantize(torch.from_numpy(w).cuda())
    copies = [wq.device_data().clone() for _ in range(reps)]
    for bsz in (1, 64):
        x = np.random.default_rng(5038 + bsz).normal(0, 1, (1024, bsz)).astype(np.float32)
        xq = pb.quantize_activations(torch.from_numpy(x).cuda())
        X = xq.device_data().t().contiguous()
        Y = torch.empty((bsz, 3072), dtype=torch.float32, device="cuda")
        for c in copies[:4]:
            pb.qmath.gemm_kmajor(c, wq.device_scale(), 3072, X, xq.device_scale(), Y=Y)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        times = []
        for it in range(3):
            ev[0].record()
            for c in copies:
                pb.qmath.gemm_kmajor(c, wq.device_scale(), 3072, X, xq.device_scale(), Y=Y)
            ev[1].record()
            ev[1].synchronize()
            times.append(ev[0].elapsed_time(ev[1]) / len(copies) / 1e3)
        t = min(times)
        nbytes = 3072 * 1024 + 4 * 1024 * bsz + 4 * 3072 * bsz
        out.append({"config": f"cfg1 B={bsz}", "us_per_product": t * 1e6, "GBps": nbytes / t / 1e9,
                    "hbm_frac_of_measured": nbytes / t / 1e9 / peaks()["hbm_gbs"],
                    "int_ops_per_s": 2 * 3072 * 1024 * bsz / t, "algorithmic_bytes": nbytes,
                    "note": "64 rotating weight copies (cold L2); product kernel incl. fused dequant epilogue"})
    return out


def model(V):
    d = pb.Dims(32000, V, 512, 1024, 2048, 512)
    return pb.synthetic_model(d, 1804)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main():
    res = cfg1()
    params = model(32000)
    qm = pb.quantize_model(params)
    net = pb.build_network(qm)
    src50 = np.random.default_rng(5038).integers(3, 32000, 50)
    t = timed(lambda: net.encode(src50))
    res.append({"config": "cfg2 encode l=50", "ms": t * 1e3})
    toks = [params.src_tokens[i] for i in src50]
    cfg = pb.DecodeConfig(beam=1, max_ratio=0.98, precision="int8")
    t = timed(lambda: pb.translate(qm, toks, cfg))
    res.append({"config": "cfg3 greedy 50 steps (encoder + decoder)", "ms": t * 1e3,
                "tokens_per_s": 50 / t, "ms_per_step": t * 1e3 / 51})
    # cfg4: 64 sentences, l ~ U[10, 80], beam 5, max_ratio 1.5 (batched, tcgen05 path)
    rng4 = np.random.default_rng(4)
    c4 = [rng4.integers(3, 32000, int(rng4.integers(10, 81))).tolist() for _ in range(64)]
    cfg4 = pb.DecodeConfig(beam=5, max_ratio=1.5, precision="int8")
    for mb, ns in ((64, 1), (32, 2), (16, 3)):
        toks = []

        def run4():
            toks[:] = pb.translate_batch(qm, c4, cfg4, max_batch=mb, return_ids=True, streams=ns)
        t = timed(run4, 3)
        ntok = sum(len(r[0]) for r in toks)
        res.append({"config": f"cfg4 64 sentences beam 5 (batches of {mb}, {ns} streams)", "ms": t * 1e3,
                    "sentences_per_s": 64 / t, "tokens_per_s": ntok / t})
    src100 = np.random.default_rng(7).integers(3, 32000, 100)
    t = timed(lambda: pb.translate(qm, [params.src_tokens[i] for i in src100], pb.DecodeConfig(5, 1.5, "int8")), 3)
    res.append({"config": "1 sentence l=100 beam 5 (151 steps)", "ms": t * 1e3, "ms_per_step": t * 1e3 / 151})
    for r in res:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
