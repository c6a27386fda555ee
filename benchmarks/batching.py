#!/usr/bin/env python
"""Corpus-level batching experiments on the cfg5 model (8192 sentences, beam 5):
(a) batches of 256 in corpus order, (b) length-sorted batches of 256,
(c) length-sorted batches decoded by E engines on E streams (one host thread
each).  Prints total tokens/s for each (device work of the whole corpus,
wall clock with a device sync at the end)."""

from __future__ import annotations

import json
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench as B  # noqa: E402
import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _lib  # noqa: E402


def run(engines, batches, streams):
    lock = threading.Lock()
    queue = list(range(len(batches)))
    toks = [0]

    def worker(i):
        e, s = engines[i], streams[i]
        with torch.cuda.stream(s):
            while True:
                with lock:
                    if not queue:
                        return
                    b = queue.pop(0)
                toks_b, _ = e.translate_ids(batches[b], B.BEAM, B.MAX_RATIO)
                with lock:
                    toks[0] += sum(len(t) for t in toks_b)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(i,)) for i in range(len(engines))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    return toks[0], time.perf_counter() - t0


def main():
    params = pb.synthetic_model(pb.Dims(**B.DIMS), B.MODEL_SEED)
    qm = pb.quantize_model(params)
    sents = B.corpus()
    order = sorted(range(len(sents)), key=lambda i: (len(sents[i]), i))
    unsorted = [sents[i:i + 256] for i in range(0, len(sents), 256)]
    srt = [[sents[j] for j in order[i:i + 256]] for i in range(0, len(sents), 256)]
    out = []
    for ne in (1, 2, 3):
        engines = [pb.Engine(qm, 256, 100, B.BEAM) for _ in range(ne)]
        streams = [torch.cuda.Stream() for _ in range(ne)]
        for name, batches in (("corpus order", unsorted), ("length-sorted", srt)):
            if ne > 1 and name == "corpus order":
                continue
            run(engines, batches[:ne * 2], streams)   # warm-up: graphs for the sizes in use
            run(engines, batches, streams)
            toks, dt = run(engines, batches, streams)
            out.append({"batches": name, "engines": ne, "tokens": toks, "s": dt, "tokens_per_s": toks / dt})
            print(json.dumps(out[-1]), flush=True)
        for e in engines:
            e.close()


if __name__ == "__main__":
    main()
