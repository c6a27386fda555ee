#!/usr/bin/env python
"""cfg4 (64 sentences, beam 5, V = 32000): batch size x engine streams of translate_batch."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench_cfgs  # noqa: E402
import paper_1804_05038_b200 as pb  # noqa: E402

c = json.load(open(os.path.join(ROOT, "tests", "golden", "baseline_corpora.json")))["cfg4"]
params = pb.synthetic_model(pb.Dims(**bench_cfgs.DIMS32), 1804)
qm = pb.quantize_model(params)
srcs = [case["src"] for case in c["cases"]]
cfg = pb.DecodeConfig(beam=c["beam"], max_ratio=c["max_ratio"], precision="int8")
ref = None
for mb, st in [(64, 1), (64, 3), (32, 2), (32, 3), (22, 3), (16, 2), (16, 3), (16, 4), (11, 3), (8, 3), (8, 4)]:
    pb.translate_batch(qm, srcs, cfg, max_batch=mb, return_ids=True, streams=st)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pb.translate_batch(qm, srcs, cfg, max_batch=mb, return_ids=True, streams=st)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    if ref is None:
        ref = res
    print(json.dumps({"max_batch": mb, "streams": st, "ms": round(1e3 * float(np.median(ts)), 2),
                      "identical": res == ref}))
