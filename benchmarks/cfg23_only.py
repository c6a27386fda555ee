#!/usr/bin/env python
"""cfg2 / cfg3 (batch-1 encoder and greedy latency path) alone: the bench's own measurement
(no CPU reference beside it)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench_cfgs  # noqa: E402
import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402

params = pb.synthetic_model(pb.Dims(**bench_cfgs.DIMS32), 1804)
model = (params, pb.quantize_model(params), None, None)
for r in bench_cfgs.cfg2_cfg3(pb, _lib.load(), 6458.7, None, model):
    keep = {k: r[k] for k in r if k in ("config", "value", "unit", "ms", "us_per_step", "parity", "e2e", "fp32_path")}
    print(json.dumps(keep))
