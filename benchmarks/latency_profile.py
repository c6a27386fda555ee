#!/usr/bin/env python
"""cfg3 latency path (batch 1, greedy, l = 50, V = 32000): one warm-up
translation, then one translation bracketed by cudaProfilerStart/Stop so that
``ncu --profile-from-start off`` sees exactly one encoder + 50 decoder steps.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/cfg3_launches.csv python benchmarks/latency_profile.py
Without ncu it prints the device time of the translation (CUDA events)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_05038_b200 as pb  # noqa: E402


def main():
    beam = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    params = pb.synthetic_model(pb.Dims(32000, 32000, 512, 1024, 2048, 512), 1804)
    qm = pb.quantize_model(params)
    src = [params.src_tokens[i] for i in np.random.default_rng(5038).integers(3, 32000, 50)]
    cfg = pb.DecodeConfig(beam=beam, max_ratio=0.98, precision="int8")
    for _ in range(3):
        pb.translate(qm, src, cfg)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.profiler.start()
    ev[0].record()
    out = pb.translate(qm, src, cfg)
    ev[1].record()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ms = ev[0].elapsed_time(ev[1])
    print(json.dumps({"config": f"cfg3 l=50 beam {beam}, 50 steps", "ms": ms, "ms_per_step": ms / 51,
                      "tokens": len(out[0])}))


if __name__ == "__main__":
    main()
