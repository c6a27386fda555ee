#!/usr/bin/env python
"""Decode ONE length-sorted batch of the cfg5 bench corpus (256 sentences, beam 5,
V 50000) through the engine, on one stream -- the unit ncu profiles: a warm-up
decode, then the decode to capture (use -k / --launch-skip to pick kernels of
a mid-decode step).  Env: QNMT_ATT_EXP / QNMT_ATT_CTX select attention variants.

  python benchmarks/one_batch.py [batch_index=16] [repeats=1]
"""

import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402


def main():
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    lib = _lib.load()
    if os.environ.get("QNMT_ATT_EXP") is not None:
        lib.qnmt_set_att_exp(int(os.environ["QNMT_ATT_EXP"]))
    if os.environ.get("QNMT_ATT_FS") is not None:   # A/B switch: scale fused into the scorer
        lib.qnmt_set_att_fused_scale(int(os.environ["QNMT_ATT_FS"]))
    if os.environ.get("QNMT_ATT_S8") is not None:   # A/B switch: bulk-staged two-MUFU scorer
        lib.qnmt_set_att_score8(int(os.environ["QNMT_ATT_S8"]))
    if os.environ.get("QNMT_ATT_CTX") is not None:
        lib.qnmt_set_att_ctx(int(os.environ["QNMT_ATT_CTX"]))
    params = pb.synthetic_model(pb.Dims(**bench.DIMS), bench.MODEL_SEED)
    qm = pb.quantize_model(params)
    sents = bench.corpus()
    batch = bench.sorted_batches(sents)[b]
    ids = [sents[i] for i in batch]
    eng = pb.Engine(qm, bench.PER_GPU, 100, bench.BEAM)
    eng.translate_ids(ids, bench.BEAM, bench.MAX_RATIO)   # warm-up (graph capture)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        toks, _ = eng.translate_ids(ids, bench.BEAM, bench.MAX_RATIO)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"batch {b}: lengths {min(map(len, ids))}..{max(map(len, ids))}, {sum(map(len, toks))} tokens, "
          f"{dt * 1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
