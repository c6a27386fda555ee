#!/usr/bin/env python
"""A small decode exercising every kernel family of the library (encoder,
batched beam decode with CUDA-graph steps, fused vocab path, attention scorer
variants and context kernels, tcgen05 GEMMs, persistent greedy, K7 shards),
sized to finish under compute-sanitizer.  benchmarks/sanitize.sh runs it under
memcheck, racecheck and synccheck (kernels filtered to the qnmt namespace)."""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402
from paper_1804_05038_b200 import vocab_shard as VS  # noqa: E402


def main():
    lib = _lib.load()
    # 16-aligned dims: stacked tcgen05 GEMMs, fused vocab kernel, one-MUFU scorer
    d = pb.Dims(500, 1000, 64, 64, 128, 64)
    params = pb.synthetic_model(d, 3, weight_std=0.3, bias_std=0.1, eos_bias=0.5)
    qm = pb.quantize_model(params)
    rng = np.random.default_rng(0)
    sents = [rng.integers(3, 500, int(rng.integers(2, 30))).tolist() for _ in range(24)]
    outs = []
    for mode, ctx in ((0, 1), (2, 2)):
        lib.qnmt_set_att_exp(mode)
        lib.qnmt_set_att_ctx(ctx)
        outs.append(pb.translate_batch(qm, sents, pb.DecodeConfig(beam=5, max_ratio=1.5, precision="int8"),
                                       max_batch=12, return_ids=True, streams=2))
    assert outs[0] == outs[1]
    pb.translate(qm, [params.src_tokens[i] for i in sents[0]], pb.DecodeConfig(beam=1, precision="int8"))
    net = pb.build_network(qm)
    enc = net.encode(sents[1])
    net.decoder_step(np.array([2, 5, 7]), net.initial_state(enc, 3), enc)
    # K7 shards
    X = torch.from_numpy(rng.integers(-127, 128, (40, 64)).astype(np.int8)).cuda()
    W = torch.from_numpy(rng.integers(-127, 128, (3000, 64)).astype(np.int8)).cuda()
    xs = torch.full((1,), 500.0, device="cuda")
    ws = torch.full((1,), 900.0, device="cuda")
    bias = torch.zeros(3000, device="cuda")
    live = torch.zeros(40, dtype=torch.float64, device="cuda")
    a = VS.unsharded(X, xs, None, W, ws, bias, live, 5)
    b = VS.candidates(X, xs, None, W, ws, bias, live, 5, shards=3)
    assert torch.equal(a[1], b[1])
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
