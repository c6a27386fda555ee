#!/usr/bin/env python
"""One cfg4 decode (64 sentences, beam 5, V = 32000) for ncu launch lists."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench_cfgs  # noqa: E402
import paper_1804_05038_b200 as pb  # noqa: E402

c = json.load(open(os.path.join(ROOT, "tests", "golden", "baseline_corpora.json")))["cfg4"]
params = pb.synthetic_model(pb.Dims(**bench_cfgs.DIMS32), 1804)
qm = pb.quantize_model(params)
srcs = [case["src"] for case in c["cases"]]
cfg = pb.DecodeConfig(beam=c["beam"], max_ratio=c["max_ratio"], precision="int8")
for _ in range(2):
    res = pb.translate_batch(qm, srcs, cfg, max_batch=64, return_ids=True)
print(sum(len(r[0]) for r in res))
