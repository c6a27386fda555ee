#!/usr/bin/env python
"""Encoder vs decoder time of one length-sorted cfg5 batch (256 sentences around the
median length): CUDA events around encode_batch and around the whole decode."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402
import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402


def main():
    params = pb.synthetic_model(pb.Dims(**B.DIMS), B.MODEL_SEED)
    qm = pb.quantize_model(params)
    sents = B.corpus()
    batches = B.sorted_batches(sents)
    eng = pb.Engine(qm, 256, 100, B.BEAM)
    out = []
    for bi in (4, 16, 28):
        batch = [sents[i] for i in batches[bi]]
        lens = np.array([len(s) for s in batch], dtype=np.int32)
        ids = torch.from_numpy(np.concatenate(batch)).cuda()
        for _ in range(2):
            eng.encode_batch(batch)
            _lib.call("qnmt_decode_batch_device", eng._h, ids.data_ptr(), lens.ctypes.data, len(batch), B.BEAM,
                      B.MAX_RATIO, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        eng.encode_batch(batch)
        ev[1].record()
        ev[2].record()
        _lib.call("qnmt_decode_batch_device", eng._h, ids.data_ptr(), lens.ctypes.data, len(batch), B.BEAM,
                  B.MAX_RATIO, torch.cuda.current_stream().cuda_stream)
        ev[3].record()
        torch.cuda.synchronize()
        out.append({"batch": bi, "len": [int(lens.min()), int(lens.max())], "encode_ms": ev[0].elapsed_time(ev[1]),
                    "encode_plus_decode_ms": ev[2].elapsed_time(ev[3])})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
