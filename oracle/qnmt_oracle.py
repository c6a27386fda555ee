"""CPU oracle for the int8 attentional-GRU decode path.  TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The B200 package
(``paper_1804_05038_b200``) never imports it and fails loudly when its CUDA
library is missing.

It restates, in plain numpy, the algorithm of the reference package ``qnmt``
(``/root/reference/pkg/src/qnmt``) for the hot path named by BASELINE.json's
``north_star``: quantize -> exact int8 GEMM -> dequantize feeding the GRU
encoder, conditional-GRU decoder, attention, output net and greedy/beam search.
Every function cites the reference file:line it follows.

Numerics ("tiers")
---------------------------------------------
* Quantization, integer products, dequantization, f32 gate arithmetic,
  bias adds and the search are the reference's own rules, bit for bit.
* ``tier="B"`` (default): the five elementwise functions that the reference
  evaluates with numpy's f32 SIMD ufuncs / OpenBLAS
  (``layers.py:35-67`` sigmoid, tanh_f32, softmax, _log_softmax_cols and the
  context ``gemm_f32`` at ``layers.py:237``) are evaluated in float64 and
  rounded once to float32.  This is the end-to-end bit-exact contract the
  B200 kernels implement (they compute the same functions in fp64).
  It is pinned by ``tests/golden/make_golden.py``, which runs the *reference
  itself* with exactly those five functions monkey-patched and records its
  outputs (``tests/golden/*.npz``).
* ``tier="A"``: the unmodified reference f32 formulas (numpy f32 ufuncs).
  Used to compare against goldens of the unpatched reference within the
  op-level tolerance.

Parity pin status: PINNED -- qmath known-answer vectors restated from
``pkg/tests/test_qmath.py`` and goldens produced by running the reference in
this container (``tests/golden/make_golden.py``); see
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

F32 = np.float32
F64 = np.float64

INT8_MAX = 127                 # qmath.py:38
INT32_SAFE_K = 131_000         # qmath.py:41
PAD_ID, UNK_ID, EOS_ID = 0, 1, 2   # model.py:33


class OracleError(Exception):
    """Raised with ``kind`` in {"invalid-input", "numeric", "shape", "vocab",
    "empty", "config"} mirroring ``errors.py:4-47``."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------------------
# quantization (qmath.py:119-187)
# ---------------------------------------------------------------------------

def encode_codes(m: np.ndarray, max_abs) -> tuple[np.ndarray, float]:
    """qmath.py:136-142 (_encode) + :119-133 (_encode_i8).

    scale = fl32(127 / max|m|) (1.0 when max is 0);
    q = sign(v) * floor(fl32(|v| + 0.5)), v = fl32(m * scale), clamp +-127.
    """
    m = np.ascontiguousarray(m, dtype=F32)
    if float(max_abs) == 0.0:
        return np.zeros(m.shape, dtype=np.int8), 1.0
    scale32 = F32(127.0) / F32(max_abs)
    v = m * scale32
    q = np.floor(np.abs(v) + F32(0.5)).astype(F32)
    q = np.where(v < 0, -q, q)
    q = np.clip(q, F32(-127.0), F32(127.0))
    return q.astype(np.int8), float(scale32)


def quantize(m: np.ndarray) -> tuple[np.ndarray, float]:
    """qmath.py:145-154: weights; non-finite -> invalid-input."""
    m = np.ascontiguousarray(m, dtype=F32)
    if m.ndim != 2 or m.shape[0] < 1 or m.shape[1] < 1:
        raise OracleError("shape", f"need non-empty 2-D matrix, got {m.shape}")
    if not np.isfinite(m).all():
        raise OracleError("invalid-input", "cannot quantize non-finite values")
    return encode_codes(m, np.max(np.abs(m)))


def quantize_activations(x: np.ndarray) -> tuple[np.ndarray, float]:
    """qmath.py:157-182: activations; non-finite -> numeric."""
    x = np.ascontiguousarray(x, dtype=F32)
    if not np.isfinite(x).all():
        raise OracleError("numeric", "activations contain non-finite values")
    return encode_codes(x, np.max(np.abs(x)) if x.size else F32(0))


def dequantize(codes: np.ndarray, scale: float) -> np.ndarray:
    """qmath.py:185-187."""
    return codes.astype(F32) / F32(scale)


def int_product(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Exact sum_k a_ik b_kj (qmath.py:205-228).  Computed as a float64 BLAS
    product, which is exact while K * 127^2 < 2^53; returned as int64."""
    if a.shape[1] != b.shape[0]:
        raise OracleError("shape", f"inner dimensions disagree: {a.shape} @ {b.shape}")
    k = a.shape[1]
    if k * 127 * 127 < 2 ** 53:
        return (a.astype(F64) @ b.astype(F64)).astype(np.int64)
    return a.astype(np.int64) @ b.astype(np.int64)


def scale_output(acc: np.ndarray, sa: float, sb: float) -> np.ndarray:
    """qmath.py:379-381: fl32(f64(acc) / (f64(sa) * f64(sb)))."""
    denom = F64(sa) * F64(sb)
    return (acc.astype(F64) / denom).astype(F32)


def qgemm(a_codes, sa, b_codes, sb) -> np.ndarray:
    """qmath.py:384-427 (qgemm and qgemm_panel are bit-identical)."""
    if b_codes.shape[1] < 1:
        raise OracleError("shape", "right-hand operand must have at least one column")
    return scale_output(int_product(a_codes, b_codes), sa, sb)


# ---------------------------------------------------------------------------
# elementwise functions (layers.py:30-67), both tiers
# ---------------------------------------------------------------------------

def _require_finite(v, op):
    if not np.isfinite(v).all():
        raise OracleError("numeric", f"{op} received non-finite input")


def sigmoid(v, tier="B"):
    """layers.py:35-39."""
    _require_finite(v, "sigmoid")
    if tier == "A":
        z = np.exp(-np.abs(v))
        return np.where(v >= 0, 1.0 / (1.0 + z), z / (1.0 + z)).astype(F32, copy=False)
    v64 = v.astype(F64)
    with np.errstate(over="ignore"):
        pos = 1.0 / (1.0 + np.exp(-v64))
        e = np.exp(v64)
        neg = e / (1.0 + e)
    return np.where(v64 >= 0, pos, neg).astype(F32)


def tanh(v, tier="B"):
    """layers.py:42-44."""
    _require_finite(v, "tanh")
    if tier == "A":
        return np.tanh(v)
    return np.tanh(v.astype(F64)).astype(F32)


def softmax0(v, tier="B"):
    """layers.py:47-51 along axis 0."""
    _require_finite(v, "softmax")
    if tier == "A":
        e = np.exp(v - np.max(v, axis=0, keepdims=True))
        return e / np.sum(e, axis=0, keepdims=True)
    v64 = v.astype(F64)
    e = np.exp(v64 - np.max(v64, axis=0, keepdims=True))
    return (e / np.sum(e, axis=0, keepdims=True)).astype(F32)


def log_softmax_cols(v, tier="B"):
    """layers.py:60-67."""
    if tier == "A":
        t = v - np.max(v, axis=0, keepdims=True)
        lse = np.log(np.sum(np.exp(t), axis=0, keepdims=True))
        if not np.isfinite(lse).all():
            raise OracleError("numeric", "log_softmax received non-finite logits")
        return t - lse
    v64 = v.astype(F64)
    t = v64 - np.max(v64, axis=0, keepdims=True)
    lse = np.log(np.sum(np.exp(t), axis=0, keepdims=True))
    if not np.isfinite(lse).all():
        raise OracleError("numeric", "log_softmax received non-finite logits")
    return (t - lse).astype(F32)


def gemm_f32(a, b, tier="B"):
    """qmath.py:434-440 (numpy/OpenBLAS a @ b).  Tier B: fp64 product rounded once."""
    if tier == "A":
        return a @ b
    return (a.astype(F64) @ b.astype(F64)).astype(F32)


def context(states, alpha, tier="B"):
    """layers.py:237 (gemm_f32(enc.states, alpha))."""
    if tier == "A":
        return states @ alpha
    return (states.astype(F64) @ alpha.astype(F64)).astype(F32)


# ---------------------------------------------------------------------------
# model: tensor directory and quantized weights (model.py:42-223, :394-437)
# ---------------------------------------------------------------------------

@dataclass
class Dims:
    src_vocab: int
    tgt_vocab: int
    embed: int
    hidden: int
    attn: int
    readout: int


GRU_FIELDS = ("wz", "uz", "bz", "wr", "ur", "br", "wc", "uc", "bc")   # model.py:36


def tensor_specs(d: Dims):
    """model.py:151-177 (serialization order)."""
    specs = [("src_embed", (d.src_vocab, d.embed)), ("tgt_embed", (d.tgt_vocab, d.embed))]
    for cell, in_dim in (("enc_fwd", d.embed), ("enc_bwd", d.embed),
                         ("dec_r", d.embed), ("dec_q", 2 * d.hidden)):
        h = d.hidden
        shp = {"wz": (h, in_dim), "uz": (h, h), "bz": (h,), "wr": (h, in_dim), "ur": (h, h),
               "br": (h,), "wc": (h, in_dim), "uc": (h, h), "bc": (h,)}
        specs.extend((f"{cell}.{f}", shp[f]) for f in GRU_FIELDS)
    specs.extend([
        ("attn.w_enc", (d.attn, 2 * d.hidden)), ("attn.b_enc", (d.attn,)),
        ("attn.u_state", (d.attn, d.hidden)), ("attn.v", (1, d.attn)),
        ("out.w_state", (d.readout, d.hidden)), ("out.w_embed", (d.readout, d.embed)),
        ("out.w_ctx", (d.readout, 2 * d.hidden)), ("out.b_readout", (d.readout,)),
        ("out.w_vocab", (d.tgt_vocab, d.readout)), ("out.b_vocab", (d.tgt_vocab,)),
        ("s0.w", (d.hidden, d.hidden)), ("s0.b", (d.hidden,)),
    ])
    return specs


class QModel:
    """Quantized model (model.py:394-437): every 2-D tensor except the two
    embeddings becomes (int8 codes, f32 scale); embeddings and biases stay f32."""

    def __init__(self, dims: Dims, tensors: dict, s0_mode="transform",
                 attention_query="current", tier="B", precision="int8"):
        self.dims = dims
        self.tier = tier
        self.precision = precision
        self.s0_mode = s0_mode
        self.attention_query = attention_query
        self.f = {}
        self.q = {}
        for name, shape in tensor_specs(dims):
            arr = np.ascontiguousarray(tensors[name], dtype=F32)
            assert tuple(arr.shape) == tuple(shape), (name, arr.shape, shape)
            if len(shape) == 2 and name not in ("src_embed", "tgt_embed") and precision == "int8":
                self.q[name] = quantize(arr)
            else:
                self.f[name] = arr

    # layers.py:118-146 (LinearOp.apply, int8 branch; float branch :138-143 -> gemm_f32)
    def linear(self, name, x, bias=None):
        if self.precision == "fp32":
            w = self.f[name]
            if x.ndim != 2 or x.shape[0] != w.shape[1]:
                raise OracleError("shape", f"LinearOp expects [{w.shape[1]}, P] input, got {x.shape}")
            y = gemm_f32(w, x, self.tier)
            if bias is not None:
                y += self.f[bias][:, None]
            return y
        codes, sw = self.q[name]
        if x.ndim != 2 or x.shape[0] != codes.shape[1]:
            raise OracleError("shape", f"LinearOp expects [{codes.shape[1]}, P] input, got {x.shape}")
        xc, sx = quantize_activations(x)
        y = qgemm(codes, sw, xc, sx)
        if bias is not None:
            y += self.f[bias][:, None]
        return y

    # layers.py:170-181
    def gru_step(self, cell, x, h):
        t = self.tier
        lin = self.linear
        z = sigmoid(lin(f"{cell}.wz", x, f"{cell}.bz") + lin(f"{cell}.uz", h), t)
        r = sigmoid(lin(f"{cell}.wr", x, f"{cell}.br") + lin(f"{cell}.ur", h), t)
        cand = tanh(lin(f"{cell}.wc", x, f"{cell}.bc") + lin(f"{cell}.uc", r * h), t)
        return (F32(1.0) - z) * h + z * cand

    # layers.py:313-348
    def encode(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        if ids.size == 0:
            raise OracleError("empty", "cannot encode an empty sentence")
        if ids.min() < 0 or ids.max() >= self.dims.src_vocab:
            raise OracleError("vocab", "source id out of range")
        emb = np.ascontiguousarray(self.f["src_embed"][ids].T)
        length, hid = ids.size, self.dims.hidden
        fwd = np.empty((hid, length), dtype=F32)
        h = np.zeros((hid, 1), dtype=F32)
        for i in range(length):
            h = self.gru_step("enc_fwd", emb[:, i:i + 1], h)
            fwd[:, i:i + 1] = h
        bwd = np.empty((hid, length), dtype=F32)
        h = np.zeros((hid, 1), dtype=F32)
        for i in range(length - 1, -1, -1):
            h = self.gru_step("enc_bwd", emb[:, i:i + 1], h)
            bwd[:, i:i + 1] = h
        states = np.ascontiguousarray(np.vstack([bwd, fwd]))
        att_proj = self.linear("attn.w_enc", states, "attn.b_enc")
        if self.s0_mode == "zero":
            s0 = np.zeros((hid, 1), dtype=F32)
        else:
            s0 = tanh(self.linear("s0.w", np.ascontiguousarray(bwd[:, :1]), "s0.b"), self.tier)
        return states, att_proj, s0

    # layers.py:214-241
    def attend(self, s_query, states, att_proj):
        u = self.linear("attn.u_state", s_query)
        length, p = att_proj.shape[1], u.shape[1]
        scores = np.empty((length, p), dtype=F32)
        for j in range(p):
            t = tanh(att_proj + u[:, j:j + 1], self.tier)
            scores[:, j] = self.linear("attn.v", t)[0]
        alpha = softmax0(scores, self.tier)
        return context(states, alpha, self.tier), alpha

    # layers.py:255-266
    def logits(self, s, emb, ctx):
        readout = tanh(self.linear("out.w_state", s, "out.b_readout")
                       + self.linear("out.w_embed", emb)
                       + self.linear("out.w_ctx", ctx), self.tier)
        return self.linear("out.w_vocab", readout, "out.b_vocab")

    # layers.py:356-384
    def decoder_step(self, y_prev, s, s_prime, enc):
        """Returns (log_probs [V,P], s_new, s_intermediate, alpha)."""
        ids = np.asarray(y_prev, dtype=np.int64)
        if ids.min() < 0 or ids.max() >= self.dims.tgt_vocab:
            raise OracleError("vocab", "target id out of range")
        states, att_proj, _ = enc
        emb = np.ascontiguousarray(self.f["tgt_embed"][ids].T)
        s_int = self.gru_step("dec_r", emb, s)
        query = s_prime if self.attention_query == "previous" else s_int
        ctx, alpha = self.attend(query, states, att_proj)
        s_new = self.gru_step("dec_q", ctx, s_int)
        lp = log_softmax_cols(self.logits(s_new, emb, ctx), self.tier)
        return lp, s_new, s_int, alpha

    # decoder.py:88-160 (single model)
    def translate(self, src_ids, beam=5, max_ratio=3.0):
        """Returns (token ids without final EOS, log_prob)."""
        return translate_ensemble([self], [src_ids], beam, max_ratio)


def translate_ensemble(models, src_ids_per_member, beam=5, max_ratio=3.0):
    """decoder.py:88-160: beam search over one sentence; with several members the
    per-step log-probs are summed in member order in f32 and divided by
    f32(#members) (:115-120).  ``src_ids_per_member[i]``: the sentence under
    member i's source vocabulary (:99).  Returns (ids without final EOS, log_prob)."""
    srcs = [list(x) for x in src_ids_per_member]
    if not srcs[0]:
        raise OracleError("empty", "cannot translate an empty sentence")
    if beam < 1 or not max_ratio > 0:
        raise OracleError("config", "bad decode config")
    vocab = models[0].dims.tgt_vocab
    encs = [m.encode(x) for m, x in zip(models, srcs)]
    max_steps = math.ceil(max_ratio * len(srcs[0])) + 1
    live_tokens = [[]]
    live_scores = np.zeros(1, dtype=F64)
    states = [(e[2].copy(), e[2].copy()) for e in encs]        # (s, s_prime) per member
    y_prev = np.array([EOS_ID], dtype=np.int64)
    finished = []   # (tokens, score)
    for _ in range(max_steps):
        lps, nxt = None, []
        for m, enc, (s, sp) in zip(models, encs, states):
            lp, s_new, s_int, _ = m.decoder_step(y_prev, s, sp, enc)
            nxt.append((s_new, s_int))
            lps = lp if lps is None else lps + lp
        if len(models) > 1:
            lps = lps / F32(len(models))
        flat = (live_scores[:, None] + lps.T.astype(F64)).ravel()
        chosen = select_candidates(flat, beam, vocab)
        nt, ns, npar, nid = [], [], [], []
        for f in chosen:
            parent, tok = divmod(f, vocab)
            score = float(flat[f])
            if tok == EOS_ID:
                finished.append((live_tokens[parent] + [tok], score))
            else:
                nt.append(live_tokens[parent] + [tok])
                ns.append(score)
                npar.append(parent)
                nid.append(tok)
        if not nt:
            break
        live_tokens = nt
        live_scores = np.array(ns, dtype=F64)
        pidx = np.array(npar, dtype=np.int64)
        states = [(np.ascontiguousarray(a[:, pidx]), np.ascontiguousarray(b[:, pidx])) for a, b in nxt]
        y_prev = np.array(nid, dtype=np.int64)
        if finished and max(h[1] for h in finished) >= live_scores.max():
            break
    else:
        for toks, score in zip(live_tokens, live_scores):
            finished.append((list(toks), float(score)))
    best = min(finished, key=lambda h: (-h[1], h[0]))
    toks = best[0][:-1] if best[0] and best[0][-1] == EOS_ID else best[0]
    return toks, best[1]


def select_candidates(flat: np.ndarray, beam: int, vocab: int) -> list:
    """decoder.py:74-85: top-``beam`` under (score desc, token asc, parent asc)."""
    n = flat.size
    if n <= beam:
        idx = range(n)
    else:
        part = np.argpartition(-flat, beam - 1)[:beam]
        smin = flat[part].min()
        idx = np.nonzero(flat >= smin)[0].tolist()
    return sorted(idx, key=lambda f: (-flat[f], f % vocab, f // vocab))[:beam]


# ---------------------------------------------------------------------------
# synthetic inputs (BASELINE.json configs)
# ---------------------------------------------------------------------------

def synthetic_tensors(dims: Dims, seed: int, weight_std=0.05, bias_std=0.0,
                      eos_bias=0.0) -> dict:
    """Seeded default_rng: every 2-D tensor ~ N(0, weight_std) in
    tensor_specs order; 1-D biases zero (bias_std=0) or drawn after all
    weights with N(0, bias_std); ``eos_bias`` is added to b_vocab[EOS] (test
    models that terminate early)."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape in tensor_specs(dims):
        if len(shape) == 2:
            out[name] = rng.normal(0.0, weight_std, shape).astype(F32)
    for name, shape in tensor_specs(dims):
        if len(shape) == 1:
            out[name] = (rng.normal(0.0, bias_std, shape).astype(F32) if bias_std > 0
                         else np.zeros(shape, dtype=F32))
    if eos_bias:
        out["out.b_vocab"][EOS_ID] += F32(eos_bias)
    return out
