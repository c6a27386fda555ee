#!/usr/bin/env python
"""Per-row phase clocks of k_vocab_merge (library built with -DQNMT_VM_PROF via
benchmarks/build_variant.sh vmprof vocab_topk.cu -DQNMT_VM_PROF; run with QNMT_LIB_PATH)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1804_05038_b200 import _lib, vocab_shard as VS  # noqa: E402
from test_gpu_vocab_shard import _case  # noqa: E402

lib = _lib.load()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1280
X, xs, seg, W, ws, bias, live = _case(50000, 512, N, 5, 0, 7)
for _ in range(3):
    VS.unsharded(X, xs, seg, W, ws, bias, live, 5)
torch.cuda.synchronize()
buf = np.zeros((N, 8), np.int64)
lib.qnmt_debug_vm_prof.argtypes = [C.c_void_p, C.c_int]
rc = lib.qnmt_debug_vm_prof(buf.ctypes.data, N)
assert rc == 0
t = buf[:, :5].astype(np.float64)
ok = t[:, 4] > 0
d = np.diff(t, axis=1) / 1.965e3   # us at 1.965 GHz
names = ["pass1 (max, sum)", "tau + pass2 list", "flag scan + rescans", "scores + ranks"]
print("rows", N, "fast-path rows", int(ok.sum()))
for i, nm in enumerate(names):
    print(f"{nm:24s} median {np.median(d[ok, i]):7.2f} us  p95 {np.percentile(d[ok, i], 95):7.2f}  max {d[ok, i].max():7.2f}")
tot = (t[ok, 4] - t[ok, 0]) / 1.965e3
print(f"{'row total':24s} median {np.median(tot):7.2f} us  p95 {np.percentile(tot, 95):7.2f}  max {tot.max():7.2f}")
span = (t[ok, 4].max() - t[ok, 0].min()) / 1.965e3
print("first start -> last end (different SM clocks: indicative)", round(span, 2), "us")
slow = np.sort(d[ok, 2][d[ok, 2] > 1.0])
print("rows with rescans:", len(slow), "phase-3 us:", np.round(slow, 1).tolist())
