#!/usr/bin/env python
"""Third randomized parity sweep: the op-level API -- LinearOp.apply, gru_step, attend and the
teacher-forced decoder_step on random models with random column counts (1..40) and input
magnitudes (1e-3..30: every code range of the attention scorer), plus the K7 vocabulary shards
against the unsharded candidates -- all against the numpy oracle (Tier B), exact.

  python benchmarks/stress_parity3.py [seconds=240] [seed=0]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1804_05038_b200 as pb  # noqa: E402
from oracle import qnmt_oracle as O  # noqa: E402
from paper_1804_05038_b200 import vocab_shard as VS  # noqa: E402
from test_gpu_vocab_shard import _case  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0 = time.time()
F32 = np.float32
counts = {"op models": 0, "shard cases": 0}


def fail(*a):
    print("MISMATCH", *a)
    sys.exit(1)


def eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def near_midpoint(fn, v, tol=1e-6):
    """True if fn(v) (extended precision) lies within tol f32-ulps of an f32 rounding midpoint for
    some element: fp64 evaluations of the activation (numpy's and CUDA's) may then round apart."""
    ld = np.longdouble
    e = fn(v.astype(ld))
    f = e.astype(F32)
    lo, hi = np.nextafter(f, F32(-np.inf)), np.nextafter(f, F32(np.inf))
    d = np.minimum(np.abs(e - (f.astype(ld) + lo.astype(ld)) / 2) / (f.astype(ld) - lo.astype(ld)),
                   np.abs((f.astype(ld) + hi.astype(ld)) / 2 - e) / (hi.astype(ld) - f.astype(ld)))
    return bool((d < tol).any())


def gru_midpoint_case(om, x, h):
    lin = om.linear
    sig = lambda v: 1 / (1 + np.exp(-v))   # noqa: E731
    pz = lin("dec_r.wz", x, "dec_r.bz") + lin("dec_r.uz", h)
    pr = lin("dec_r.wr", x, "dec_r.br") + lin("dec_r.ur", h)
    r = O.sigmoid(pr, "B")
    pc = lin("dec_r.wc", x, "dec_r.bc") + lin("dec_r.uc", r * h)
    return near_midpoint(sig, pz) or near_midpoint(sig, pr) or near_midpoint(np.tanh, pc)


while time.time() - t0 < budget:
    if rng.random() < 0.85:
        dims = dict(src_vocab=int(rng.integers(20, 120)), tgt_vocab=int(rng.integers(20, 700)),
                    embed=int(rng.choice([8, 16, 32, 48])), hidden=int(rng.choice([12, 16, 32, 48, 64, 128])),
                    attn=int(rng.choice([10, 16, 40, 64, 128, 256])), readout=int(rng.choice([6, 16, 32, 48])))
        s0, aq = str(rng.choice(["transform", "zero"])), str(rng.choice(["current", "previous"]))
        seed = int(rng.integers(1, 1 << 30))
        wstd = float(rng.choice([0.05, 0.3, 1.0]))
        params = pb.synthetic_model(pb.Dims(**dims), seed, wstd, 0.1, 0.5, s0, aq)
        om = O.QModel(O.Dims(**dims), params.tensors, s0_mode=s0, attention_query=aq, tier="B")
        net = pb.build_network(pb.quantize_model(params))
        H, E = dims["hidden"], dims["embed"]
        tag = (dims, s0, aq, seed, wstd)
        for _ in range(3):
            P = int(rng.choice([1, 2, 5, 8, 9, 16, 40]))
            mag = float(10.0 ** rng.uniform(-3, 1.5))
            x = (rng.normal(0, 1, (E, P)) * mag).astype(F32)
            h = (rng.normal(0, 1, (H, P)) * float(10.0 ** rng.uniform(-2, 0.5))).astype(F32)
            if not eq(net.dec_r.update_in.apply(x), om.linear("dec_r.wz", x, "dec_r.bz")):
                fail("linear", tag, P, mag)
            g_out = np.asarray(pb.gru_step(net.dec_r, x, h))
            o_out = om.gru_step("dec_r", x, h)
            if not eq(g_out, o_out):
                os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
                np.savez(os.path.join(ROOT, "gpurun_out", "stress3_gru_fail.npz"), x=x, h=h, gpu=g_out, oracle=o_out,
                         dims=np.array(list(dims.values())), seed=seed, wstd=wstd)
                idx = np.argwhere(g_out != o_out)
                if gru_midpoint_case(om, x, h):   # fp64 libm vs CUDA at an f32 midpoint
                    counts["midpoint cases"] = counts.get("midpoint cases", 0) + 1
                    continue
                print("gru_step diff at", idx.tolist()[:5], g_out[tuple(idx[0])], o_out[tuple(idx[0])],
                      "again:", eq(np.asarray(pb.gru_step(net.dec_r, x, h)), o_out))
                fail("gru_step", tag, P, mag)
        src = rng.integers(3, dims["src_vocab"], int(rng.integers(1, 30))).tolist()
        enc = net.encode(np.asarray(src))
        ost, oatt, os0 = om.encode(src)
        if not (eq(enc.states, ost) and eq(enc.att_proj, oatt) and eq(enc.s0, os0)):
            fail("encode", tag, src)
        for _ in range(3):
            P = int(rng.choice([1, 2, 5, 12, 16]))
            q = (rng.normal(0, 1, (H, P)) * float(10.0 ** rng.uniform(-3, 1.5))).astype(F32)
            ctx, alpha = pb.attend(net.attention, q, enc)
            octx, oalpha = om.attend(q, ost, oatt)
            if not (eq(alpha, oalpha) and eq(ctx, octx)):
                fail("attend", tag, P, len(src))
            y = rng.integers(0, dims["tgt_vocab"], P)
            s = (rng.normal(0, 1, (H, P)) * 0.5).astype(F32)
            sp = (rng.normal(0, 1, (H, P)) * 0.5).astype(F32)
            lp, st2, al = net.decoder_step(y, pb.DecoderState(s, sp), enc)
            olp, osn, osi, oal = om.decoder_step(y, s, sp, (ost, oatt, os0))
            if not (eq(st2.s_prime, osi) and eq(st2.s, osn) and eq(al, oal) and eq(lp, olp)):
                fail("decoder_step", tag, P, len(src))
        counts["op models"] += 1
    else:
        V = int(rng.choice([20, 300, 3001, 12345, 50000]))
        K = int(rng.choice([16, 64, 512]))
        N = int(rng.choice([5, 37, 300]))
        k = int(rng.integers(1, 9))
        dup = int(rng.choice([0, 0, 7, 97]))
        G = int(rng.choice([1, 2, 3, 5, 8]))
        if k > V:
            continue
        X, xs, seg, W, ws, bias, live = _case(V, K, N, k, dup, int(rng.integers(1, 1 << 30)))
        cs0, ct0 = VS.unsharded(X, xs, seg, W, ws, bias, live, k)
        cs1, ct1 = VS.candidates(X, xs, seg, W, ws, bias, live, k, shards=G)
        if not (torch.equal(ct0, ct1) and torch.equal(cs0, cs1)):
            fail("shards", V, K, N, k, dup, G)
        counts["shard cases"] += 1
print(f"stress parity 3 ok: {counts}, {time.time() - t0:.0f} s")
