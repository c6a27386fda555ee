"""Generate golden fixtures by running the REFERENCE implementation (qnmt).

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Two modes of the reference are recorded:

* Tier A -- the unmodified reference.
* Tier B -- the reference with exactly five elementwise functions of
  ``qnmt.layers`` replaced by "evaluate in float64, round once to float32"
  versions: ``sigmoid`` (layers.py:35), ``tanh_f32`` (:42), ``softmax`` (:47),
  ``_log_softmax_cols`` (:60) and the ``gemm_f32`` name used for the
  attention context (:237).  Quantization, integer GEMMs, scales, gate
  arithmetic and search remain the reference's own code.  Tier B is the
  end-to-end bit-exact contract of the B200 kernels.

Outputs (committed, small): ``qmath_kat.npz``, ``small_model.npz``,
``translate_small.json``, ``baseline_dims.npz``.
"""

from __future__ import annotations

import contextlib
import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import qnmt  # noqa: E402  (the reference)
from qnmt import layers as ref_layers  # noqa: E402
from qnmt import model as ref_model  # noqa: E402
from qnmt import qmath as ref_qmath  # noqa: E402
from qnmt.decoder import DecodeConfig, translate  # noqa: E402

F32, F64 = np.float32, np.float64


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# Tier-B patch
# ---------------------------------------------------------------------------

def _sigmoid_b(v):
    ref_layers._require_finite(v, "sigmoid")
    v64 = v.astype(F64)
    with np.errstate(over="ignore"):
        pos = 1.0 / (1.0 + np.exp(-v64))
        e = np.exp(v64)
        neg = e / (1.0 + e)
    return np.where(v64 >= 0, pos, neg).astype(F32)


def _tanh_b(v):
    ref_layers._require_finite(v, "tanh")
    return np.tanh(v.astype(F64)).astype(F32)


def _softmax_b(v, axis=0):
    ref_layers._require_finite(v, "softmax")
    v64 = v.astype(F64)
    e = np.exp(v64 - np.max(v64, axis=axis, keepdims=True))
    return (e / np.sum(e, axis=axis, keepdims=True)).astype(F32)


def _log_softmax_cols_b(v):
    v64 = v.astype(F64)
    t = v64 - np.max(v64, axis=0, keepdims=True)
    lse = np.log(np.sum(np.exp(t), axis=0, keepdims=True))
    if not np.isfinite(lse).all():
        raise ref_layers.NumericError("log_softmax received non-finite logits")
    return (t - lse).astype(F32)


def _gemm_f32_b(a, b):
    return (np.asarray(a, F64) @ np.asarray(b, F64)).astype(F32)


@contextlib.contextmanager
def tier_b():
    saved = {k: getattr(ref_layers, k) for k in
             ("sigmoid", "tanh_f32", "softmax", "_log_softmax_cols", "gemm_f32")}
    ref_layers.sigmoid = _sigmoid_b
    ref_layers.tanh_f32 = _tanh_b
    ref_layers.softmax = _softmax_b
    ref_layers._log_softmax_cols = _log_softmax_cols_b
    ref_layers.gemm_f32 = _gemm_f32_b
    try:
        yield
    finally:
        for k, v in saved.items():
            setattr(ref_layers, k, v)


# ---------------------------------------------------------------------------
# models: same recipe as oracle.synthetic_tensors / package synthetic model
# ---------------------------------------------------------------------------

def make_params(dims: ref_model.Dims, seed: int, bias_std=0.0, s0_mode="transform",
                attention_query="current", weight_std=0.05, eos_bias=0.0):
    from oracle.qnmt_oracle import Dims as ODims, synthetic_tensors
    od = ODims(**dims.as_dict())
    tensors = synthetic_tensors(od, seed, weight_std, bias_std, eos_bias)
    vs = ref_model._synthetic_vocab(dims.src_vocab)
    vt = ref_model._synthetic_vocab(dims.tgt_vocab)
    return ref_model._build_params(dims, tensors, vs, vt, s0_mode, attention_query), tensors


# ---------------------------------------------------------------------------
# 1. qmath known answers
# ---------------------------------------------------------------------------

def gen_qmath():
    out = {}
    cases = {
        "zeros": np.zeros((3, 3), F32),
        "ten": np.array([[10.0]], F32),
        "ties": np.array([[2.0, 1.0, -1.0]], F32),
        "halfulp": np.array([[127.0, 0.49999997]], F32),
        "u8x8": np.random.default_rng(7).uniform(-1, 1, (8, 8)).astype(F32),
        "n5x7": np.random.default_rng(3).normal(0, 10, (5, 7)).astype(F32),
        "u6x5": np.random.default_rng(11).uniform(-50, 50, (6, 5)).astype(F32),
        "n64x200": np.random.default_rng(12).normal(0, 1, (64, 200)).astype(F32),
        "tiny": (np.random.default_rng(13).normal(0, 1, (4, 9)) * 1e-30).astype(F32),
        "huge": (np.random.default_rng(14).normal(0, 1, (4, 9)) * 1e30).astype(F32),
        "halfgrid": (np.arange(-300, 301, dtype=F32) / F32(2.0)).reshape(1, -1),
    }
    for name, m in cases.items():
        q = ref_qmath.quantize(m)
        out[f"q_{name}_in"] = m
        out[f"q_{name}_codes"] = q.data
        out[f"q_{name}_scale"] = np.array(q.scale, F64)
        qa = ref_qmath.quantize_activations(m)
        assert np.array_equal(qa.data, q.data) and qa.scale == q.scale
    # random int8 GEMMs (test_qmath.py:41-44 operand style), incl. ragged shapes
    rng = np.random.default_rng(2024)
    shapes = [(1, 1, 1), (4, 8, 1), (6, 10, 5), (13, 33, 8), (64, 64, 3), (3, 5, 2),
              (7, 70, 2), (33, 129, 7), (100, 96, 16), (5, 1000, 8), (1000, 1000, 1)]
    for i, (m, k, p) in enumerate(shapes):
        a = ref_qmath.QuantizedMatrix(rng.integers(-127, 128, (m, k)).astype(np.int8),
                                      float(F32(rng.uniform(0.5, 200.0))))
        b = ref_qmath.QuantizedMatrix(rng.integers(-127, 128, (k, p)).astype(np.int8),
                                      float(F32(rng.uniform(0.5, 200.0))))
        y = ref_qmath.qgemm_panel(a, b)
        assert np.array_equal(y, ref_qmath.qgemm(a, b))
        out[f"g{i}_a"], out[f"g{i}_b"] = a.data, b.data
        out[f"g{i}_sa"], out[f"g{i}_sb"] = np.array(a.scale, F64), np.array(b.scale, F64)
        out[f"g{i}_y"] = y
    out["g_count"] = np.array(len(shapes))
    # cfg1: W ~ N(0,0.05) [3072x1024], X ~ N(0,1) [1024xB], B in {1, 64}
    w = np.random.default_rng(1804).normal(0, 0.05, (3072, 1024)).astype(F32)
    wq = ref_qmath.quantize(w)
    out["cfg1_w_scale"] = np.array(wq.scale, F64)
    out["cfg1_w_codes_sha"] = np.array(sha(wq.data))
    for bsz in (1, 64):
        x = np.random.default_rng(5038 + bsz).normal(0, 1, (1024, bsz)).astype(F32)
        xq = ref_qmath.quantize_activations(x)
        y = ref_qmath.qgemm_panel(wq, xq)
        acc = wq.data.astype(np.int64) @ xq.data.astype(np.int64)
        out[f"cfg1_b{bsz}_x_scale"] = np.array(xq.scale, F64)
        out[f"cfg1_b{bsz}_x_codes_sha"] = np.array(sha(xq.data))
        out[f"cfg1_b{bsz}_acc_sha"] = np.array(sha(acc.astype(np.int32)))
        out[f"cfg1_b{bsz}_y_sha"] = np.array(sha(y))
        out[f"cfg1_b{bsz}_y_head"] = y[:64].copy()
    np.savez_compressed(os.path.join(HERE, "qmath_kat.npz"), **out)
    print("qmath_kat.npz:", len(out), "arrays")


# ---------------------------------------------------------------------------
# 2. small model: op-level (both tiers) + translations (Tier B and A)
# ---------------------------------------------------------------------------

SMALL_DIMS = dict(src_vocab=40, tgt_vocab=37, embed=8, hidden=12, attn=10, readout=6)
MED_DIMS = dict(src_vocab=300, tgt_vocab=251, embed=32, hidden=48, attn=40, readout=24)
# (tag, dims, seed, weight_std, bias_std, eos_bias, s0_mode, attention_query)
MODELS = [
    ("small", SMALL_DIMS, 11, 0.05, 0.05, 0.0, "transform", "current"),
    ("med", MED_DIMS, 12, 0.05, 0.05, 0.0, "transform", "current"),
    ("eos", SMALL_DIMS, 13, 0.6, 0.1, 0.75, "transform", "current"),   # terminates early
    ("eosmed", MED_DIMS, 14, 0.3, 0.1, 0.6, "transform", "current"),
    ("flags", SMALL_DIMS, 15, 0.6, 0.1, 0.5, "zero", "previous"),      # model-header flags
]


def op_level(prefix, params, out, rng, p=3, length=7):
    qm = ref_model.quantize_model(params)
    net = ref_layers.build_network(qm)
    d = params.dims
    ids = rng.integers(3, d.src_vocab, length)
    enc = net.encode(ids)
    out[f"{prefix}_src"] = ids
    out[f"{prefix}_states"] = enc.states
    out[f"{prefix}_att_proj"] = enc.att_proj
    out[f"{prefix}_s0"] = enc.s0
    # teacher-forced decoder step at width p from a random state
    s = rng.normal(0, 0.5, (d.hidden, p)).astype(F32)
    sp = rng.normal(0, 0.5, (d.hidden, p)).astype(F32)
    y = rng.integers(0, d.tgt_vocab, p)
    st = ref_layers.DecoderState(s=s, s_prime=sp)
    lp, st2, alpha = net.decoder_step(y, st, enc)
    out[f"{prefix}_step_s"], out[f"{prefix}_step_sp"], out[f"{prefix}_step_y"] = s, sp, y
    out[f"{prefix}_step_lp"] = lp
    out[f"{prefix}_step_snew"] = st2.s
    out[f"{prefix}_step_sint"] = st2.s_prime
    out[f"{prefix}_step_alpha"] = alpha
    # single ops
    x = rng.normal(0, 1, (d.embed, p)).astype(F32)
    h = rng.normal(0, 0.5, (d.hidden, p)).astype(F32)
    out[f"{prefix}_gru_x"], out[f"{prefix}_gru_h"] = x, h
    out[f"{prefix}_gru_out"] = ref_layers.gru_step(net.dec_r, x, h)
    ctx, al = ref_layers.attend(net.attention, h, enc)
    out[f"{prefix}_att_ctx"], out[f"{prefix}_att_alpha"] = ctx, al
    out[f"{prefix}_lin_out"] = net.dec_r.update_in.apply(x)


def gen_small():
    out = {}
    tr = {"cases": []}
    for tag, dims_kw, seed, ws, bs, eb, s0m, aq in MODELS:
        dims = ref_model.Dims(**dims_kw)
        params, _ = make_params(dims, seed, bias_std=bs, weight_std=ws, eos_bias=eb,
                                s0_mode=s0m, attention_query=aq)
        for tier in ("A", "B"):
            rng = np.random.default_rng(100 + seed)
            ctx = tier_b() if tier == "B" else contextlib.nullcontext()
            with ctx:
                op_level(f"{tag}{tier}", params, out, rng)
        qm = ref_model.quantize_model(params)
        rng = np.random.default_rng(200 + seed)
        for n in range(24):
            length = int(rng.integers(1, 12))
            ids = rng.integers(3, dims.src_vocab, length).tolist()
            if n % 7 == 3:
                ids[0] = 1  # UNK id in the source
            beam = [1, 2, 3, 5, 8][n % 5]
            ratio = [1.5, 3.0, 0.5, 2.0][n % 4]
            toks = [params.src_tokens[i] for i in ids]
            cfg = DecodeConfig(beam=beam, max_ratio=ratio, precision="int8")
            case = {"model": tag, "src": ids, "beam": beam, "max_ratio": ratio}
            for tier in ("A", "B"):
                ctx = tier_b() if tier == "B" else contextlib.nullcontext()
                with ctx:
                    words, logp = translate(qm, toks, cfg)
                tgt_index = {t: i for i, t in enumerate(params.tgt_tokens)}
                case[f"out_{tier}"] = [tgt_index[w] for w in words]
                case[f"logp_{tier}"] = logp
            tr["cases"].append(case)
    tr["models"] = {m[0]: dict(dims=m[1], seed=m[2], weight_std=m[3], bias_std=m[4],
                               eos_bias=m[5], s0_mode=m[6], attention_query=m[7])
                    for m in MODELS}
    np.savez_compressed(os.path.join(HERE, "small_model.npz"), **out)
    with open(os.path.join(HERE, "translate_small.json"), "w") as fh:
        json.dump(tr, fh, indent=1)
    print("small_model.npz:", len(out), "arrays; translate_small.json:", len(tr["cases"]), "cases")


# ---------------------------------------------------------------------------
# 3. BASELINE dims (cfg2/cfg3 and one beam-5 sentence)
# ---------------------------------------------------------------------------

BASE_DIMS = dict(src_vocab=32000, tgt_vocab=32000, embed=512, hidden=1024, attn=2048, readout=512)


def gen_baseline():
    out = {}
    dims = ref_model.Dims(**BASE_DIMS)
    params, _ = make_params(dims, 1804)
    qm = ref_model.quantize_model(params)
    out["w_scales"] = np.array([qm.stats[k].scale for k in sorted(qm.stats)], F64)
    out["w_scale_names"] = np.array(sorted(qm.stats))
    net = ref_layers.build_network(qm)
    rng = np.random.default_rng(5038)
    src50 = rng.integers(3, 32000, 50)
    out["src50"] = src50
    with tier_b():
        enc = net.encode(src50)
        out["B_states_sha"] = np.array(sha(enc.states))
        out["B_att_proj_sha"] = np.array(sha(enc.att_proj))
        out["B_states_col0"] = enc.states[:, 0].copy()
        out["B_states_col49"] = enc.states[:, 49].copy()
        out["B_s0"] = enc.s0
        toks = [params.src_tokens[i] for i in src50]
        words, logp = translate(qm, toks, DecodeConfig(beam=1, max_ratio=0.98, precision="int8"))
        idx = {t: i for i, t in enumerate(params.tgt_tokens)}
        out["B_greedy50"] = np.array([idx[w] for w in words])
        out["B_greedy50_logp"] = np.array(logp, F64)
        # first decoder step log-probs (teacher forced from s0)
        st = net.initial_state(enc, 1)
        lp, st2, alpha = net.decoder_step(np.array([2]), st, enc)
        out["B_step1_lp_sha"] = np.array(sha(lp))
        out["B_step1_lp_top"] = np.sort(lp[:, 0])[-16:]
        out["B_step1_alpha"] = alpha
        out["B_step1_snew"] = st2.s
        src10 = src50[:10]
        toks10 = [params.src_tokens[i] for i in src10]
        words, logp = translate(qm, toks10, DecodeConfig(beam=5, max_ratio=1.5, precision="int8"))
        out["B_beam5_src"] = src10
        out["B_beam5"] = np.array([idx[w] for w in words])
        out["B_beam5_logp"] = np.array(logp, F64)
    # Tier A (unpatched) op-level at full dims: one decoder step at P=5
    enc_a = net.encode(src50[:20])
    out["A_enc20_states_col0"] = enc_a.states[:, 0].copy()
    s = np.repeat(enc_a.s0, 5, axis=1)
    y = np.array([2, 5, 77, 1000, 31999])
    lp, st2, alpha = net.decoder_step(y, ref_layers.DecoderState(s=s, s_prime=s.copy()), enc_a)
    out["A_step_y"] = y
    out["A_step_lp_top"] = np.sort(lp, axis=0)[-8:]
    out["A_step_argmax"] = np.argmax(lp, axis=0)
    out["A_step_snew"] = st2.s
    np.savez_compressed(os.path.join(HERE, "baseline_dims.npz"), **out)
    print("baseline_dims.npz:", len(out), "arrays")


# ensembles (decoder.py:115-120): members share the target vocabulary; member 2 has a
# smaller source vocabulary (its UNK mapping differs) and the "previous" query flags
ENSEMBLES = [
    ("ens2", [("e_a", dict(SMALL_DIMS), 21, 0.6, 0.1, 0.75, "transform", "current"),
              ("e_b", dict(SMALL_DIMS), 22, 0.6, 0.1, 0.75, "transform", "current")]),
    ("ens3", [("e_c", dict(SMALL_DIMS), 23, 0.5, 0.1, 0.6, "transform", "current"),
              ("e_d", dict(SMALL_DIMS, src_vocab=SMALL_DIMS["src_vocab"] - 9), 24, 0.5, 0.1, 0.6, "zero", "previous"),
              ("e_e", dict(SMALL_DIMS), 25, 0.05, 0.05, 0.0, "transform", "current")]),
    ("ensdup", [("e_a", dict(SMALL_DIMS), 21, 0.6, 0.1, 0.75, "transform", "current"),
                ("e_a", dict(SMALL_DIMS), 21, 0.6, 0.1, 0.75, "transform", "current")]),
]


def gen_ensemble():
    """Tier-B (and Tier-A) ensemble translations by the reference's translate()."""
    out = {"ensembles": {}, "cases": []}
    for tag, members in ENSEMBLES:
        qms, src_tokens = [], None
        for mtag, dims_kw, seed, ws, bs, eb, s0m, aq in members:
            params, _ = make_params(ref_model.Dims(**dims_kw), seed, bias_std=bs, weight_std=ws, eos_bias=eb,
                                    s0_mode=s0m, attention_query=aq)
            qms.append(ref_model.quantize_model(params))
            src_tokens = src_tokens or params.src_tokens
        out["ensembles"][tag] = [dict(tag=m[0], dims=m[1], seed=m[2], weight_std=m[3], bias_std=m[4], eos_bias=m[5],
                                      s0_mode=m[6], attention_query=m[7]) for m in members]
        rng = np.random.default_rng(300 + len(tag))
        for n in range(10):
            length = int(rng.integers(1, 10))
            ids = rng.integers(3, len(src_tokens), length).tolist()
            toks = [src_tokens[i] for i in ids]
            beam = [1, 3, 5, 2, 8][n % 5]
            ratio = [1.5, 3.0, 2.0][n % 3]
            cfg = DecodeConfig(beam=beam, max_ratio=ratio, precision="int8")
            case = {"ensemble": tag, "src_tokens": toks, "beam": beam, "max_ratio": ratio}
            for tier in ("A", "B"):
                ctx = tier_b() if tier == "B" else contextlib.nullcontext()
                with ctx:
                    words, logp = translate(qms, toks, cfg)
                tgt_index = {t: i for i, t in enumerate(qms[0].tgt_tokens)}
                case[f"out_{tier}"] = [tgt_index[w] for w in words]
                case[f"logp_{tier}"] = logp
            out["cases"].append(case)
    with open(os.path.join(HERE, "ensemble_small.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("ensemble_small.json:", len(out["cases"]), "cases")


def gen_fp32():
    """The reference's fp32 path (precision="fp32": LinearOp's float branch,
    layers.py:138-145): Tier-B / Tier-A translations, op-level outputs, a
    compare_precisions report, and BLEU / edit-distance known answers."""
    import importlib
    ref_bleu = importlib.import_module("qnmt.bleu")
    from qnmt import decoder as ref_decoder
    out = {"cases": [], "ops": {}, "parity": {}, "bleu": [], "edit": []}
    arrays = {}
    for tag, dims_kw, seed, ws, bs, eb, s0m, aq in MODELS:
        dims = ref_model.Dims(**dims_kw)
        params, _ = make_params(dims, seed, bias_std=bs, weight_std=ws, eos_bias=eb, s0_mode=s0m,
                                attention_query=aq)
        rng = np.random.default_rng(400 + seed)
        for n in range(8):
            length = int(rng.integers(1, 10))
            ids = rng.integers(3, dims.src_vocab, length).tolist()
            beam = [1, 3, 5, 2][n % 4]
            ratio = [1.5, 3.0, 2.0][n % 3]
            toks = [params.src_tokens[i] for i in ids]
            cfg = DecodeConfig(beam=beam, max_ratio=ratio, precision="fp32")
            case = {"model": tag, "src": ids, "beam": beam, "max_ratio": ratio}
            for tier in ("A", "B"):
                ctx = tier_b() if tier == "B" else contextlib.nullcontext()
                with ctx:
                    words, logp = translate(params, toks, cfg)
                tgt_index = {t: i for i, t in enumerate(params.tgt_tokens)}
                case[f"out_{tier}"] = [tgt_index[w] for w in words]
                case[f"logp_{tier}"] = logp
            out["cases"].append(case)
        # op level, Tier B: encoder outputs and one decoder step at P = 3
        with tier_b():
            net = ref_layers.build_network(params)
            src = rng.integers(3, dims.src_vocab, 6)
            enc = net.encode(src)
            st = net.initial_state(enc, 3)
            y = rng.integers(0, dims.tgt_vocab, 3)
            lp, st2, alpha = net.decoder_step(y, st, enc)
            x = rng.normal(0, 1, (dims.embed, 4)).astype(F32)
            lin = net.dec_r.update_in.apply(x)
        for k, v in (("src", src), ("states", enc.states), ("att_proj", enc.att_proj), ("s0", enc.s0), ("y", y),
                     ("lp", lp), ("s_new", st2.s), ("s_int", st2.s_prime), ("alpha", alpha), ("x", x),
                     ("lin_wz", lin)):
            arrays[f"{tag}_{k}"] = np.asarray(v)
        if tag in ("eos", "med"):   # compare_precisions (Tier B) over a small corpus
            corpus = [[params.src_tokens[i] for i in rng.integers(3, dims.src_vocab, int(rng.integers(1, 9)))]
                      for _ in range(12)]
            with tier_b():
                rep = ref_decoder.compare_precisions(params, corpus, DecodeConfig(beam=3, max_ratio=1.5))
            out["parity"][tag] = {"corpus": corpus, "report": rep.to_dict(), "fp32": rep.fp32_outputs,
                                  "int8": rep.int8_outputs}
    rng = np.random.default_rng(77)
    for _ in range(40):   # BLEU / edit distance known answers
        nl = int(rng.integers(1, 5))
        hyps = [[f"t{v}" for v in rng.integers(0, 6, int(rng.integers(0, 12)))] for _ in range(nl)]
        refs = [[f"t{v}" for v in rng.integers(0, 6, int(rng.integers(0, 12)))] for _ in range(nl)]
        if _ % 2:   # near-copies: non-zero scores
            refs = [[f"t{v}" for v in rng.integers(0, 9, int(rng.integers(4, 14)))] for _ in range(nl)]
            hyps = [r[:int(rng.integers(1, len(r) + 1))] + [f"t{int(rng.integers(0, 9))}"] for r in refs]
        try:
            b = ref_bleu.bleu([" ".join(h) for h in hyps], [" ".join(r) for r in refs])
        except Exception as exc:   # noqa: BLE001
            b = type(exc).__name__
        out["bleu"].append({"hyps": hyps, "refs": refs, "bleu": b})
        out["edit"].append({"a": hyps[0], "b": refs[0], "d": ref_decoder.edit_distance(hyps[0], refs[0])})
    out["models"] = {m[0]: dict(dims=m[1], seed=m[2], weight_std=m[3], bias_std=m[4], eos_bias=m[5],
                                s0_mode=m[6], attention_query=m[7]) for m in MODELS}
    with open(os.path.join(HERE, "fp32_small.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "fp32_ops.npz"), **arrays)
    print("fp32_small.json:", len(out["cases"]), "translations,", len(out["parity"]), "parity reports;",
          "fp32_ops.npz:", len(arrays), "arrays")


MODELFILE_ARGS = dict(src_vocab=14, tgt_vocab=13, embed=4, hidden=6, seed=11, attn=5, readout=3)


def gen_modelfile():
    """A QNMT file written by the reference's save_model, and the reference
    loader's verdict (exception type, byte offset) on each corruption of it."""
    import tempfile

    import modelfile_cases
    from qnmt import errors as ref_errors

    params = ref_model.generate_model(**MODELFILE_ARGS)
    path = os.path.join(HERE, "model_tiny.qnmt")
    ref_model.save_model(params, path)
    blob = open(path, "rb").read()
    verdicts = {"generate_model_args": MODELFILE_ARGS, "file_sha256": hashlib.sha256(blob).hexdigest(),
                "cases": {}}
    with tempfile.TemporaryDirectory() as d:
        for name, data in modelfile_cases.cases(blob).items():
            p = os.path.join(d, name)
            with open(p, "wb") as fh:
                fh.write(data)
            try:
                ref_model.load_model(p)
                verdicts["cases"][name] = {"error": None}
            except ref_errors.QnmtError as exc:
                verdicts["cases"][name] = {"error": type(exc).__name__, "offset": getattr(exc, "offset", None)}
    with open(os.path.join(HERE, "model_tiny_errors.json"), "w") as fh:
        json.dump(verdicts, fh, indent=1, sort_keys=True)
    print("model_tiny.qnmt:", len(blob), "bytes;", len(verdicts["cases"]), "corruption verdicts")



# ---------------------------------------------------------------------------
# 4. BASELINE configs: Tier-A teacher-forced ops at full dims, the cfg4 corpus,
#    a cfg5 sample, and the Tier-A vs Tier-B agreement report
# ---------------------------------------------------------------------------

CFG5_DIMS = dict(BASE_DIMS, tgt_vocab=50000)


def _decode_many(qm, corpora, cfg, threads=8):
    """The reference's translate() over many sentences (one per thread, as the
    reference's own bench.py:129-132 does): [(ids, logp)]."""
    from concurrent.futures import ThreadPoolExecutor
    idx = {t: i for i, t in enumerate(qm.tgt_tokens)}

    def one(toks):
        words, lp = translate(qm, toks, cfg)
        return [idx[w] for w in words], lp

    with ThreadPoolExecutor(threads) as pool:
        return list(pool.map(one, corpora))


def _trace_search(net, toks, beam, ratio):
    """decoder.py:88-160 for one model, recording each step's chosen candidates
    {token path: score} and every candidate's score by path (for the first step
    at which two tiers' selections differ).  Returns (steps, final ids, logp)."""
    from qnmt.decoder import _select_candidates
    ids = net.src_ids(toks)
    enc = net.encode(ids)
    V = net.dims.tgt_vocab
    max_steps = int(np.ceil(ratio * len(toks))) + 1
    live = [()]
    scores = np.zeros(1, F64)
    st = net.initial_state(enc, 1)
    y = np.array([2], np.int64)
    fin = []
    steps = []
    for _ in range(max_steps):
        lp, st2, _ = net.decoder_step(y, st, enc)
        flat = (scores[:, None] + lp.T.astype(F64)).ravel()
        chosen = _select_candidates(flat, beam, V)
        top = np.argsort(-flat, kind="stable")[:4 * beam]
        steps.append({"chosen": {live[f // V] + (f % V,): float(flat[f]) for f in chosen},
                      "cand": {live[f // V] + (f % V,): float(flat[f]) for f in top}})
        nl, ns, npar, ny = [], [], [], []
        for f in chosen:
            par, tok = divmod(f, V)
            if tok == 2:
                fin.append((live[par] + (tok,), float(flat[f])))
            else:
                nl.append(live[par] + (tok,)); ns.append(float(flat[f])); npar.append(par); ny.append(tok)
        if not nl:
            break
        live, scores = nl, np.array(ns, F64)
        st = st2.select(np.array(npar, np.int64))
        y = np.array(ny, np.int64)
        if fin and max(h[1] for h in fin) >= scores.max():
            break
    else:
        fin += [(p, float(s)) for p, s in zip(live, scores)]
    best = min(fin, key=lambda h: (-h[1], list(h[0])))
    out = list(best[0][:-1]) if best[0] and best[0][-1] == 2 else list(best[0])
    return steps, out, best[1]


def _divergence(net, toks, beam, ratio):
    """First step where Tier A and Tier B select different candidates, with the
    score gap (under each tier) between the candidates that swapped places."""
    ta, outa, lpa = _trace_search(net, toks, beam, ratio)
    with tier_b():
        tb, outb, lpb = _trace_search(net, toks, beam, ratio)
    for t, (sa, sb) in enumerate(zip(ta, tb)):
        ka, kb = set(sa["chosen"]), set(sb["chosen"])
        if ka == kb:
            continue
        only_a, only_b = sorted(ka - kb), sorted(kb - ka)
        # under tier B: best B-only pick vs the A-only pick B ranked highest (and vice versa)
        gap_b = min(sb["chosen"][p] for p in only_b) - max(sb["cand"].get(p, -np.inf) for p in only_a)
        gap_a = min(sa["chosen"][p] for p in only_a) - max(sa["cand"].get(p, -np.inf) for p in only_b)
        shared = [p for p in sa["cand"] if p in sb["cand"]]
        disc = max(abs(sa["cand"][p] - sb["cand"][p]) for p in shared) if shared else float("nan")
        return {"step": t, "gap_B": float(gap_b), "gap_A": float(gap_a), "tier_discrepancy": float(disc),
                "score_at_step": float(max(sb["chosen"].values())), "out_A": outa, "out_B": outb,
                "logp_A": lpa, "logp_B": lpb}
    return {"step": None, "out_A": outa, "out_B": outb, "logp_A": lpa, "logp_B": lpb}


def _first_diff(a, b):
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return i
    return None if len(a) == len(b) else min(len(a), len(b))


def gen_baseline_parity():
    """cfg3/cfg4/cfg5 outputs of the reference in both tiers, Tier-A op outputs at
    BASELINE dims on fixed inputs, and the agreement report (tier_agreement.json)."""
    out = {}
    report = {"note": "Tier A = unmodified reference, Tier B = reference with its five elementwise functions in "
                      "fp64 rounded once (the GPU contract). For each sentence whose outputs differ: the first "
                      "decode step at which the two tiers select different candidates, and the score gap between "
                      "the swapped candidates under each tier.",
              "configs": {}}
    dims = ref_model.Dims(**BASE_DIMS)
    params, _ = make_params(dims, 1804)
    qm = ref_model.quantize_model(params)
    net = ref_layers.build_network(qm)
    rng = np.random.default_rng(5038)
    src50 = rng.integers(3, 32000, 50)
    # -- Tier A (and B) teacher-forced ops at full dims, l = 20, P = 3 ------------
    src20 = src50[:20]
    enc_a = net.encode(src20)
    out["tf_src"] = src20
    out["tf_states"], out["tf_att_proj"], out["tf_s0"] = enc_a.states, enc_a.att_proj, enc_a.s0
    r = np.random.default_rng(77)
    s = (np.repeat(enc_a.s0, 3, axis=1) + r.normal(0, 0.05, (1024, 3))).astype(F32)
    sp = (s + r.normal(0, 0.05, (1024, 3))).astype(F32)
    y = np.array([2, 77, 31999])
    out["tf_s"], out["tf_sp"], out["tf_y"] = s, sp, y
    x = r.normal(0, 1, (512, 3)).astype(F32)
    xq = r.normal(0, 0.3, (2048, 3)).astype(F32)
    h = r.normal(0, 0.5, (1024, 3)).astype(F32)
    out["tf_x"], out["tf_xq"], out["tf_h"] = x, xq, h
    encs = ref_layers.EncoderStates(states=enc_a.states, att_proj=enc_a.att_proj, s0=enc_a.s0)
    for tier in ("A", "B"):
        ctx = tier_b() if tier == "B" else contextlib.nullcontext()
        with ctx:
            lp, st2, alpha = net.decoder_step(y, ref_layers.DecoderState(s=s, s_prime=sp), encs)
            out[f"tf{tier}_lp"] = lp
            out[f"tf{tier}_snew"], out[f"tf{tier}_sint"], out[f"tf{tier}_alpha"] = st2.s, st2.s_prime, alpha
            out[f"tf{tier}_gru_r"] = ref_layers.gru_step(net.dec_r, x, h)
            out[f"tf{tier}_gru_q"] = ref_layers.gru_step(net.dec_q, xq, h)
            c, a = ref_layers.attend(net.attention, h, encs)
            out[f"tf{tier}_att_ctx"], out[f"tf{tier}_att_alpha"] = c, a
    # -- cfg3 greedy 50 steps, Tier A ------------------------------------------------
    toks50 = [params.src_tokens[i] for i in src50]
    cfg3 = DecodeConfig(beam=1, max_ratio=0.98, precision="int8")
    words, lpa = translate(qm, toks50, cfg3)
    idx = {t: i for i, t in enumerate(params.tgt_tokens)}
    out["A_greedy50"], out["A_greedy50_logp"] = np.array([idx[w] for w in words]), np.array(lpa, F64)
    gold = np.load(os.path.join(HERE, "baseline_dims.npz"))
    rep3 = {"sentences": 1, "beam": 1, "rows": []}
    fd = _first_diff(list(out["A_greedy50"]), list(gold["B_greedy50"]))
    rep3["rows"].append({"i": 0, "len": 50, "identical": fd is None, "first_token_diff": fd,
                         "logp_A": float(lpa), "logp_B": float(gold["B_greedy50_logp"])})
    report["configs"]["cfg3"] = rep3
    # -- cfg4: 64 sentences, l ~ U[10, 80], beam 5, max_ratio 1.5, V = 32000 -----------
    rng4 = np.random.default_rng(5042)
    corpus4 = [rng4.integers(3, 32000, int(rng4.integers(10, 81))) for _ in range(64)]
    toks4 = [[params.src_tokens[i] for i in c] for c in corpus4]
    cfg4 = DecodeConfig(beam=5, max_ratio=1.5, precision="int8")
    with tier_b():
        res_b = _decode_many(qm, toks4, cfg4)
    res_a = _decode_many(qm, toks4, cfg4)
    cases4 = []
    for i, (c, rb, ra) in enumerate(zip(corpus4, res_b, res_a)):
        cases4.append({"src": c.tolist(), "out_B": rb[0], "logp_B": rb[1], "out_A": ra[0], "logp_A": ra[1]})
    report["configs"]["cfg4"] = _agreement(net, params, corpus4, res_a, res_b, 5, 1.5)
    # -- cfg5 sample: 16 sentences of the bench corpus (l ~ U[5, 100]), V = 50000 ------
    dims5 = ref_model.Dims(**CFG5_DIMS)
    params5, _ = make_params(dims5, 1804)
    qm5 = ref_model.quantize_model(params5)
    net5 = ref_layers.build_network(qm5)
    r5 = np.random.default_rng(5038)
    lens5 = r5.integers(5, 101, 8192)
    corpus5_all = [r5.integers(3, 32000, int(n)) for n in lens5]
    order = sorted(range(8192), key=lambda i: (len(corpus5_all[i]), i))
    pick = [order[(2 * k + 1) * 8192 // 32] for k in range(16)]
    corpus5 = [corpus5_all[i] for i in pick]
    toks5 = [[params5.src_tokens[i] for i in c] for c in corpus5]
    with tier_b():
        res5_b = _decode_many(qm5, toks5, cfg4)
    res5_a = _decode_many(qm5, toks5, cfg4)
    cases5 = [{"corpus_index": int(i), "src": c.tolist(), "out_B": rb[0], "logp_B": rb[1], "out_A": ra[0],
               "logp_A": ra[1]} for i, c, rb, ra in zip(pick, corpus5, res5_b, res5_a)]
    report["configs"]["cfg5"] = _agreement(net5, params5, corpus5, res5_a, res5_b, 5, 1.5)
    np.savez_compressed(os.path.join(HERE, "baseline_parity.npz"), **out)
    with open(os.path.join(HERE, "baseline_corpora.json"), "w") as fh:
        json.dump({"cfg4": {"seed": 5042, "beam": 5, "max_ratio": 1.5, "model_seed": 1804, "dims": BASE_DIMS,
                            "cases": cases4},
                   "cfg5": {"corpus_seed": 5038, "beam": 5, "max_ratio": 1.5, "model_seed": 1804, "dims": CFG5_DIMS,
                            "cases": cases5}}, fh)
    with open(os.path.join(HERE, "tier_agreement.json"), "w") as fh:
        json.dump(report, fh, indent=1)
    print("baseline_parity.npz:", len(out), "arrays; cfg4", len(cases4), "cfg5", len(cases5), "sentences")


def _agreement(net, params, corpus, res_a, res_b, beam, ratio):
    rows = []
    for i, (c, ra, rb) in enumerate(zip(corpus, res_a, res_b)):
        row = {"i": i, "len": len(c), "identical": ra[0] == rb[0], "first_token_diff": _first_diff(ra[0], rb[0]),
               "logp_A": ra[1], "logp_B": rb[1]}
        if not row["identical"]:
            d = _divergence(net, [params.src_tokens[j] for j in c], beam, ratio)
            assert d["out_A"] == ra[0] and d["out_B"] == rb[0], "traced search != translate()"
            row.update({k: d[k] for k in ("step", "gap_B", "gap_A", "tier_discrepancy", "score_at_step")})
        rows.append(row)
    same = sum(r["identical"] for r in rows)
    return {"sentences": len(rows), "identical": same, "beam": beam, "max_ratio": ratio, "rows": rows}

if __name__ == "__main__":
    which = sys.argv[1:] or ["qmath", "small", "baseline", "modelfile", "ensemble", "fp32", "parity"]
    if "fp32" in which:
        gen_fp32()
    if "ensemble" in which:
        gen_ensemble()
    if "modelfile" in which:
        gen_modelfile()
    if "qmath" in which:
        gen_qmath()
    if "small" in which:
        gen_small()
    if "baseline" in which:
        gen_baseline()
    if "parity" in which:
        gen_baseline_parity()
