#!/usr/bin/env python
"""cfg1 (one LinearOp product, B = 1 and 64) alone: the bench's own measurement without the rest."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench_cfgs  # noqa: E402
import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402

for r in bench_cfgs.cfg1(pb, _lib.load(), 6458.7, None):
    print(json.dumps({k: r[k] for k in ("config", "us_per_product", "value", "unit", "kernels_per_product", "parity")}))
