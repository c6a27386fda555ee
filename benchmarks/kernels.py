#!/usr/bin/env python
"""Per-kernel device times at the cfg5 decode-step shapes (N = 1280 live columns
= 256 sentences x beam 5), each captured 20x in a CUDA graph and timed with
CUDA events (no host launch overhead), plus cfg1's batch-1 GEMV with 64
rotating weight copies (cold L2).  One JSON line per kernel."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_05038_b200 as pb  # noqa: E402
from paper_1804_05038_b200 import _dev, _lib  # noqa: E402

PEAK = {"hbm_gbs": 6461.2, "int8_tops_spec": 4500.0}
try:
    PEAK.update(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json"))))
except OSError:
    pass


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e9
    for _ in range(5):
        ev[0].record()
        g.replay()
        ev[1].record()
        ev[1].synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]) / reps)
    return best * 1e-3


def gemm_case(name, M, K, N, seg_count=256):
    rng = np.random.default_rng(M + K + N)
    W = torch.from_numpy(rng.integers(-127, 128, (M, K)).astype(np.int8)).cuda()
    X = torch.from_numpy(rng.integers(-127, 128, (N, K)).astype(np.int8)).cuda()
    ws = torch.rand(1, device="cuda") + 1
    xs = torch.rand(seg_count, device="cuda") + 1
    seg = torch.arange(N, device="cuda", dtype=torch.int32) // max(1, N // seg_count)
    Y = torch.empty((N, M), dtype=torch.float32, device="cuda")
    t = graph_time(lambda: pb.qmath.gemm_kmajor(W, ws, M, X, xs, col_seg=seg, Y=Y))
    ops = 2.0 * M * N * K
    nbytes = M * K + N * K + 4 * M * N
    return {"kernel": "gemm_i8 (tcgen05)" if N > 8 else "gemm_i8 (dp4a gemv)", "shape": name, "M": M, "N": N,
            "K": K, "us": t * 1e6, "TOPS": ops / t / 1e12, "tensor_frac_of_spec": ops / t / 1e12 / PEAK["int8_tops_spec"],
            "GBps": nbytes / t / 1e9}


def int_mm_case(M, K, N):
    """cuBLASLt int8 GEMM (torch._int_mm, int32 out) on the same shape: the library ceiling."""
    a = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda").t()
    c = torch.empty((N, M), dtype=torch.int32, device="cuda")
    try:
        t = graph_time(lambda: torch._int_mm(a, b, out=c), reps=5)
    except Exception as ex:   # noqa: BLE001
        return {"kernel": "cublasLt int8 (torch._int_mm)", "M": M, "N": N, "K": K, "error": str(ex)[:200]}
    ops = 2.0 * M * N * K
    return {"kernel": "cublasLt int8 (torch._int_mm)", "M": M, "N": N, "K": K, "us": t * 1e6, "TOPS": ops / t / 1e12,
            "tensor_frac_of_spec": ops / t / 1e12 / PEAK["int8_tops_spec"]}


def topk_case(N=1280, V=50000, k=5):
    x = torch.randn((N, V), device="cuda") * 0.2
    live = torch.randn(N, dtype=torch.float64, device="cuda")
    cs = torch.empty((N, k), dtype=torch.float64, device="cuda")
    ct = torch.empty((N, k), dtype=torch.int32, device="cuda")
    f = _dev.flag()
    st = lambda: torch.cuda.current_stream().cuda_stream
    t = graph_time(lambda: _lib.call("qnmt_topk_candidates", x.data_ptr(), N, V, V, live.data_ptr(), k,
                                     cs.data_ptr(), ct.data_ptr(), f.data_ptr(), st()))
    return {"kernel": "topk_candidates", "N": N, "V": V, "us": t * 1e6, "GBps": 4.0 * N * V / t / 1e9,
            "hbm_frac_of_measured": 4.0 * N * V / t / 1e9 / PEAK["hbm_gbs"]}


def attention_case(S=256, beam=5, A=2048, H2=2048, seed=0, sorted_batch=None):
    """One decoder step of attention for 256 sentences x 5 hypotheses, l ~ U[5, 100]
    (sorted_batch=k: the lengths of the k-th length-sorted batch of the cfg5 corpus,
    what the bench's engines see)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(5, 101, S).astype(np.int32)
    if sorted_batch is not None:
        crng = np.random.default_rng(5038)
        cl = np.sort(crng.integers(5, 101, 8192))
        lens = cl[sorted_batch * S:(sorted_batch + 1) * S].astype(np.int32)
    rows = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    P = int(lens.sum())
    N = S * beam
    att = torch.randn((P, A), device="cuda") * 0.5
    states = torch.randn((P, H2), device="cuda") * 0.5
    u = torch.randn((N, A), device="cuda") * 0.5
    v = torch.randint(-127, 128, (A,), dtype=torch.int8, device="cuda")
    vs = torch.full((1,), 90.0, device="cuda")
    off = torch.arange(0, N, beam, dtype=torch.int32, device="cuda")
    cnt = torch.full((S,), beam, dtype=torch.int32, device="cuda")
    rows_d = torch.from_numpy(rows).cuda()
    lens_d = torch.from_numpy(lens).cuda()
    ctx = torch.empty((N, H2), device="cuda")
    scratch = torch.empty(N * (104 + A) + 256, dtype=torch.int32, device="cuda")
    mm = torch.empty((S, 2, A), device="cuda")
    ex = torch.empty_like(att)
    f = _dev.flag()
    _lib.call("qnmt_attention_stats", att.data_ptr(), rows_d.data_ptr(), lens_d.data_ptr(), S, A, mm.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    _lib.call("qnmt_attention_exp", att.data_ptr(), att.numel(), ex.data_ptr(), torch.cuda.current_stream().cuda_stream)
    t = graph_time(lambda: _lib.call("qnmt_attention", u.data_ptr(), A, N, off.data_ptr(), cnt.data_ptr(), S,
                                     att.data_ptr(), mm.data_ptr(), ex.data_ptr(), states.data_ptr(), rows_d.data_ptr(),
                                     lens_d.data_ptr(), 100,
                                     A, H2, v.data_ptr(), vs.data_ptr(), ctx.data_ptr(), H2, None, 0,
                                     scratch.data_ptr(), f.data_ptr(), torch.cuda.current_stream().cuda_stream))
    tanh_count = beam * A * int(lens.sum())
    nbytes = 4.0 * (2 * P * A + P * H2 + N * A + N * H2)   # att_proj x2 passes, states, u, ctx
    return {"kernel": "attention step", "N": N, "sum_l": P, "us": t * 1e6, "tanh_per_s": tanh_count / t,
            "GBps": nbytes / t / 1e9}


def vocab_case(N=1280, V=50000, K=512, k=5, fused=True):
    """Vocab projection + candidates of one cfg5 decode step: fused (vocab_topk.cu)
    vs tcgen05 GEMM (bias) + single-pass candidate kernel."""
    rng = np.random.default_rng(7)
    W = torch.from_numpy(rng.integers(-127, 128, (V, K)).astype(np.int8)).cuda()
    X = torch.from_numpy(rng.integers(-127, 128, (N, K)).astype(np.int8)).cuda()
    ws = torch.full((1,), 3000.0, device="cuda")
    xs = torch.full((N // 5,), 2000.0, device="cuda") + torch.rand(N // 5, device="cuda")
    seg = torch.arange(N, device="cuda", dtype=torch.int32) // 5
    bias = torch.randn(V, device="cuda") * 0.1
    live = torch.randn(N, dtype=torch.float64, device="cuda")
    cs = torch.empty((N, k), dtype=torch.float64, device="cuda")
    ct = torch.empty((N, k), dtype=torch.int32, device="cuda")
    f = _dev.flag()
    st = lambda: torch.cuda.current_stream().cuda_stream
    if fused:
        scratch = torch.empty(int(_lib.load().qnmt_vocab_candidates_scratch(N, V)), dtype=torch.uint8,
                              device="cuda")
        fn = lambda: _lib.call("qnmt_vocab_candidates", X.data_ptr(), N, K, xs.data_ptr(), seg.data_ptr(),
                               W.data_ptr(), V, K, K, ws.data_ptr(), V, bias.data_ptr(), live.data_ptr(), k,
                               scratch.data_ptr(), cs.data_ptr(), ct.data_ptr(), f.data_ptr(), st())
    else:
        Y = torch.empty((N, V), dtype=torch.float32, device="cuda")

        def fn():
            pb.qmath.gemm_kmajor(W, ws, V, X, xs, col_seg=seg, bias=bias, Y=Y)
            _lib.call("qnmt_topk_candidates", Y.data_ptr(), N, V, V, live.data_ptr(), k, cs.data_ptr(),
                      ct.data_ptr(), f.data_ptr(), st())
    t = graph_time(fn, reps=5)
    out = {"kernel": "vocab+candidates " + ("fused" if fused else "gemm+topk"), "N": N, "V": V, "K": K,
           "us": t * 1e6, "logits_per_s": N * V / t, "TOPS": 2.0 * N * V * K / t / 1e12}
    if fused:   # merge path per row (pad of the row's first 24-byte partial)
        np_ = scratch.numel() // (24 * N)
        pad = scratch.view(torch.int32).view(N, np_ * 6)[:, 5].cpu().numpy()
        vals, cnts = np.unique(pad, return_counts=True)
        out["merge_paths"] = {int(v): int(c) for v, c in zip(vals, cnts)}
    return out


def gemv_cold(bsz):
    w = torch.randint(-127, 128, (3072, 1024), dtype=torch.int8, device="cuda")
    copies = [w.clone() for _ in range(64)]
    X = torch.randint(-127, 128, (bsz, 1024), dtype=torch.int8, device="cuda")
    ws = torch.ones(1, device="cuda")
    xs = torch.ones(1, device="cuda")
    Y = torch.empty((bsz, 3072), dtype=torch.float32, device="cuda")
    it = iter(range(10 ** 9))

    def run(static):
        for c in copies:
            pb.qmath.gemm_kmajor(c, ws, 3072, X, xs, Y=Y, w_static=static)
    t_iso = graph_time(lambda: run(False), reps=1) / len(copies)
    t = graph_time(lambda: run(True), reps=1) / len(copies)
    nbytes = 3072 * 1024 + 4 * 1024 * bsz + 4 * 3072 * bsz
    return {"kernel": "cfg1 qgemm_panel", "B": bsz, "us": t * 1e6, "GBps": nbytes / t / 1e9,
            "hbm_frac_of_measured": nbytes / t / 1e9 / PEAK["hbm_gbs"], "TOPS": 2 * 3072 * 1024 * bsz / t / 1e12,
            "us_no_prefetch": t_iso * 1e6, "GBps_no_prefetch": nbytes / t_iso / 1e9,
            "note": "64 rotating weight copies (201 MB > 126 MB L2) in one CUDA graph; 'us' with the PDL weight "
                    "prefetch (W streams while the previous product drains), 'us_no_prefetch' without"}


def gemv_large(M, K):
    """Batch-1 GEMV over one large weight matrix (the vocab projection, or 64 MB) with
    rotating copies (> L2): the HBM-streaming rate of the GEMV kernel once the matrix
    is big enough to hide the launch and DRAM latency that bound cfg1's 3 MB product."""
    reps = max(2, int(256e6 // (M * K)))
    w = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
    copies = [w.clone() for _ in range(reps)]
    X = torch.randint(-127, 128, (1, K), dtype=torch.int8, device="cuda")
    ws = torch.ones(1, device="cuda")
    xs = torch.ones(1, device="cuda")
    Y = torch.empty((1, M), dtype=torch.float32, device="cuda")

    def run():
        for c in copies:
            pb.qmath.gemm_kmajor(c, ws, M, X, xs, Y=Y, w_static=True)
    t = graph_time(run, reps=1) / len(copies)
    nbytes = M * K + K + 4 * M
    return {"kernel": "gemv batch 1 (large)", "M": M, "K": K, "us": t * 1e6, "GBps": nbytes / t / 1e9,
            "hbm_frac_of_measured": nbytes / t / 1e9 / PEAK["hbm_gbs"],
            "note": f"{len(copies)} rotating weight copies ({len(copies) * M * K / 1e6:.0f} MB > L2)"}


def main():
    which = sys.argv[1:] or ["gemm", "topk", "gemv"]
    out = []
    if "gemm" in which:
        N = 1280
        for name, M, K in [("dec_r Wx", 3072, 512), ("dec Uzr", 2048, 1024), ("dec Uc", 1024, 1024),
                           ("att U", 2048, 1024), ("dec_q Wx", 3072, 2048), ("readout Ws", 512, 1024),
                           ("readout Wc", 512, 2048), ("vocab", 50000, 512)]:
            out.append(gemm_case(name, M, K, N))
        out.append(gemm_case("enc x-side", 3072, 512, 13000, 13000))
        out.append(gemm_case("enc Uzr", 2048, 1024, 256))
    if "big" in which:   # tensor-bound shapes: tcgen05 K3 vs cuBLASLt int8 (torch._int_mm) as the measured ceiling
        for M, N, K in [(8192, 8192, 8192), (16384, 8192, 4096), (50000, 1280, 512)]:
            out.append(gemm_case(f"big {M}x{N}x{K}", M, K, N))
            out.append(int_mm_case(M, K, N))
    if "topk" in which:
        out.append(topk_case())
    if "vocab" in which:
        out += [vocab_case(fused=True), vocab_case(fused=False)]
    if "att" in which:
        for sb in (None, 16):
            for mode in (2, 1, 0):   # scorer: score7, score6 (one-MUFU), score5 (two-MUFU)
                old = _lib.load().qnmt_set_att_exp(mode)
                r = attention_case(sorted_batch=sb)
                r["att_exp"] = mode
                r["batch"] = "random lengths" if sb is None else f"sorted cfg5 batch {sb}"
                out.append(r)
                _lib.load().qnmt_set_att_exp(old)
    if "gemv" in which:
        out += [gemv_cold(1), gemv_cold(64), gemv_large(50000, 512), gemv_large(16384, 4096)]
    for r in out:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
