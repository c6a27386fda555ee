#!/usr/bin/env python
"""Device time of each length-sorted cfg5 batch decoded alone (one engine, one stream),
for the cost model bench.shard_batches balances ranks with.  One JSON line per batch."""

import importlib.util
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402

spec = importlib.util.spec_from_file_location("qbench", os.path.join(ROOT, "bench.py"))
B = importlib.util.module_from_spec(spec)
spec.loader.exec_module(B)


def main():
    qm = pb.quantize_model(pb.synthetic_model(pb.Dims(**B.DIMS), B.MODEL_SEED))
    sents = B.corpus()
    batches = B.sorted_batches(sents)
    e = pb.Engine(qm, B.PER_GPU, 100, B.BEAM)
    st = torch.cuda.current_stream()
    for k, b in enumerate(batches):
        ids = torch.from_numpy(np.concatenate([sents[i] for i in b])).cuda()
        lens = np.array([len(sents[i]) for i in b], dtype=np.int32)
        ts = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.call("qnmt_decode_batch_device", e._h, ids.data_ptr(), lens.ctypes.data, len(b), B.BEAM,
                      B.MAX_RATIO, st.cuda_stream)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(json.dumps({"batch": k, "min_len": int(lens.min()), "max_len": int(lens.max()),
                          "sum_len": int(lens.sum()), "sum_len2": int((lens.astype(np.int64) ** 2).sum()),
                          "ms": min(ts)}), flush=True)


if __name__ == "__main__":
    main()
