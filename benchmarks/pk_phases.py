#!/usr/bin/env python
"""Phase timings of the persistent batch-1 greedy kernel (cfg3: l = 50, V = 32000):
%globaltimer after each grid barrier of each step (CTA 0), median over steps."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200.engine import engine_pool  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402

NAMES = ["P0 emb/s + GEMV Wx2,Uzr2", "P1 gates + GEMV Uc2", "P2 combine + GEMV Uatt,Uzr3", "P3 scale + scores",
         "P4 softmax + context", "P5 q(ctx) + GEMV Wx3", "P6 gates + GEMV Uc3", "P7 combine + GEMV Ws",
         "P8 readout + vocab GEMV", "P9 partials", "P10 lse + tie scan", "P11 search"]


def main():
    params = pb.synthetic_model(pb.Dims(32000, 32000, 512, 1024, 2048, 512), 1804)
    qm = pb.quantize_model(params)
    src = [params.src_tokens[i] for i in np.random.default_rng(5038).integers(3, 32000, 50)]
    cfg = pb.DecodeConfig(beam=1, max_ratio=0.98, precision="int8")
    pb.translate(qm, src, cfg)
    e = engine_pool(qm).all[0]
    lib = _lib.load()
    lib.qnmt_engine_stamps(e._h, 1)
    pb.translate(qm, src, cfg)
    torch.cuda.synchronize()
    buf = np.zeros((256, 11), dtype=np.int64)
    n = lib.qnmt_engine_stamps_read(e._h, buf.ctypes.data, 256, torch.cuda.current_stream().cuda_stream)
    st = buf[:n].astype(np.float64)
    d = np.diff(st, axis=1) / 1e3                      # phases 1..10 (us)
    step = np.diff(st[:, 0]) / 1e3                     # stamp 0 to next step's stamp 0
    out = {"steps": int(n), "step_us_median": float(np.median(step)),
           "phases_us_median": {NAMES[k + 1]: float(np.median(d[:, k])) for k in range(10)}}
    out["phases_us_median"]["P11 + next P0 (remainder)"] = out["step_us_median"] - float(np.median(d.sum(axis=1)))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
