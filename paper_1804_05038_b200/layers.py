"""Model layers on B200 (drop-in for qnmt.layers).

Same objects and call signatures as the reference ``layers.py``; activations
keep the reference's ``[features, P]`` shape convention (layers.py:9-11).
Inputs may be numpy arrays (outputs are then numpy) or torch CUDA tensors
(outputs are torch views whose memory is the kernels' K-major ``[P][features]``
layout, i.e. ``y.t()`` is contiguous).

Two device compositions exist and are tested against the oracle:
* the per-op path (:meth:`LinearOp.apply`, :func:`gru_step`, :func:`attend`,
  :meth:`OutputNet.logits`) -- one C-ABI op per reference operation;
* the engine path (:meth:`Network.encode`, :meth:`Network.decoder_step`,
  and decoder.translate) -- csrc/engine.cu, the production path.
Both precisions run on B200: int8 LinearOps quantize + tcgen05/dp4a GEMM; float
LinearOps (the fp32 path, layers.py:138-145) use csrc/gemm_f32.cu, evaluated in
fp64 and rounded once (the Tier-B contract of gemm_f32).
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .engine import engine_pool
from .errors import ConfigError, ShapeError, VocabError, EmptyInputError
from .qmath import QuantizedMatrix, gemm_f32_kmajor, gemm_kmajor

F32 = np.float32


def _out(y_k: torch.Tensor, like):
    """K-major device result -> reference-shaped output of the caller's type."""
    y = y_k.t()
    return y.contiguous().cpu().numpy() if _dev.is_numpy(like) else y


def _quant_k(x_k: torch.Tensor, col_seg=None, nseg=1):
    """Segmented K1 on a contiguous device K-major [N][K] f32 -> (codes, scales)."""
    N, K = x_k.shape
    q = torch.empty((N, K), dtype=torch.int8, device=x_k.device)
    scales = torch.empty(nseg, dtype=torch.float32, device=x_k.device)
    bits = torch.empty(nseg, dtype=torch.int32, device=x_k.device)
    _lib.call("qnmt_quantize", x_k.data_ptr(), N, K, _dev.ld(x_k), _dev.ptr(col_seg), nseg,
              q.data_ptr(), K, scales.data_ptr(), bits.data_ptr(), 1, _dev.flag().data_ptr(),
              _dev.stream_ptr())
    return q, scales


# ---------------------------------------------------------------------------
# elementwise functions (layers.py:35-67), device versions (fp64-evaluated)
# ---------------------------------------------------------------------------

def tanh_f32(v):
    x = _dev.to_device(v)
    if x.dim() == 1:
        x = x[None, :]
    x = x.contiguous()
    y = torch.empty_like(x)
    f = _dev.reset_flag()
    _lib.call("qnmt_tanh", x.data_ptr(), x.shape[0], x.shape[1], _dev.ld(x), y.data_ptr(),
              _dev.ld(y), f.data_ptr(), _dev.stream_ptr())
    _dev.raise_flag(f, numeric_msg="tanh received non-finite input")
    y = y.reshape(np.shape(v)) if _dev.is_numpy(v) else y.reshape(v.shape)
    return y.cpu().numpy() if _dev.is_numpy(v) else y


def _log_softmax_cols(v):
    """Column log-softmax of [V, P] logits (layers.py:60-67)."""
    x = _dev.kmajor(v)
    lp = torch.empty_like(x)
    f = _dev.reset_flag()
    _lib.call("qnmt_log_softmax", x.data_ptr(), x.shape[0], x.shape[1], _dev.ld(x), lp.data_ptr(),
              _dev.ld(lp), f.data_ptr(), _dev.stream_ptr())
    _dev.raise_flag(f, numeric_msg="log_softmax received non-finite logits")
    return _out(lp, v)


# ---------------------------------------------------------------------------
# precision-generic linear operator (int8 on B200)
# ---------------------------------------------------------------------------

@dataclass(eq=False)
class LinearOp:
    """A trained linear transform ``y = W x (+ b)`` (layers.py:94-146): ``weight``
    is a :class:`QuantizedMatrix` (int8 path) or a float32 ``[out, in]`` matrix
    (fp32 path, numpy or device tensor)."""

    weight: object
    bias: object = None

    def _wdev(self) -> torch.Tensor:
        w = getattr(self, "_wd", None)
        if w is None:
            if len(np.shape(self.weight)) != 2 or min(np.shape(self.weight)) < 1:
                raise ShapeError(f"weight must be a non-empty 2-D matrix, got shape {tuple(np.shape(self.weight))}")
            w = _dev.to_device(self.weight).contiguous()
            self._wd = w
        return w

    @property
    def is_quantized(self) -> bool:
        return isinstance(self.weight, QuantizedMatrix)

    @property
    def out_dim(self) -> int:
        return self.weight.rows if self.is_quantized else self.weight.shape[0]

    @property
    def in_dim(self) -> int:
        return self.weight.cols if self.is_quantized else self.weight.shape[1]

    def _bias_dev(self):
        if self.bias is None:
            return None
        b = getattr(self, "_bdev", None)
        if b is None:
            b = _dev.to_device(self.bias).contiguous()
            self._bdev = b
        return b

    def apply_k(self, x_k: torch.Tensor, out: torch.Tensor | None = None, accumulate=False,
                col_seg=None, nseg=1) -> torch.Tensor:
        """K-major core: x_k [P][in] device f32 -> y_k [P][out] (quantize + GEMM + bias,
        or the fp32 product + bias)."""
        if not self.is_quantized:
            return gemm_f32_kmajor(self._wdev(), x_k, bias=self._bias_dev(), Y=out, accumulate=accumulate)
        if col_seg is None and nseg == 1 and out is None and x_k.shape[0] <= 8:
            return self._linear_small(x_k)
        q, sx = _quant_k(x_k, col_seg, nseg)
        return gemm_kmajor(self.weight.device_data(), self.weight.device_scale(), self.out_dim, q, sx,
                           col_seg=col_seg, bias=self._bias_dev(), Y=out, accumulate=accumulate,
                           w_static=True)

    def _linear_small(self, x_k: torch.Tensor) -> torch.Tensor:
        """Batch <= 8 (the latency path): quantize_activations + qgemm_panel + bias as the
        single qnmt_linear_i8 kernel."""
        N, K = x_k.shape
        M = self.out_dim
        x_k = x_k.contiguous()
        y = torch.empty((N, M), dtype=torch.float32, device=x_k.device)
        q = torch.empty((N, K), dtype=torch.int8, device=x_k.device)
        sx = torch.empty(1, dtype=torch.float32, device=x_k.device)
        bits = torch.empty(1, dtype=torch.int32, device=x_k.device)
        w = self.weight
        _lib.call("qnmt_linear_i8", w.device_data().data_ptr(), M, K, _dev.ld(w.device_data()),
                  w.device_scale().data_ptr(), M, x_k.data_ptr(), N, K, _dev.ptr(self._bias_dev()), y.data_ptr(), M,
                  q.data_ptr(), K, sx.data_ptr(), bits.data_ptr(), _lib.GEMM_W_STATIC, _dev.flag().data_ptr(),
                  _dev.stream_ptr())
        return y

    def apply(self, x, timer=None):
        if len(np.shape(x)) != 2 or np.shape(x)[0] != self.in_dim:
            raise ShapeError(f"LinearOp expects [{self.in_dim}, P] input, got {tuple(np.shape(x))}")
        f = _dev.reset_flag()
        y = self.apply_k(_dev.kmajor(x))
        _dev.raise_flag(f)
        return _out(y, x)


# ---------------------------------------------------------------------------
# GRU cell (layers.py:153-181)
# ---------------------------------------------------------------------------

@dataclass(eq=False)
class GruCell:
    update_in: LinearOp
    update_state: LinearOp
    reset_in: LinearOp
    reset_state: LinearOp
    cand_in: LinearOp
    cand_state: LinearOp
    hidden: int

    def __post_init__(self):
        for op in (self.update_in, self.update_state, self.reset_in,
                   self.reset_state, self.cand_in, self.cand_state):
            if op.out_dim != self.hidden:
                raise ShapeError("GRU sub-operator output does not match hidden size")

    def packed(self):
        """Stacked device weights: WX=[wz;wr;wc] (3 scales), BX, UZR=[uz;ur] (2 scales), UC."""
        p = getattr(self, "_packed", None)
        if p is None and not self.update_in.is_quantized:   # fp32: WX, BX, UZR, UC without scales
            ins = (self.update_in, self.reset_in, self.cand_in)
            wx = torch.cat([o._wdev() for o in ins]).contiguous()
            dev = wx.device
            bx = torch.cat([o._bias_dev() if o.bias is not None
                            else torch.zeros(self.hidden, dtype=torch.float32, device=dev) for o in ins])
            uzr = torch.cat([self.update_state._wdev(), self.reset_state._wdev()]).contiguous()
            p = (wx, None, bx.contiguous(), uzr, None, self.cand_state._wdev(), None)
            self._packed = p
        if p is None:
            ins = (self.update_in, self.reset_in, self.cand_in)
            wx = torch.cat([o.weight.device_data() for o in ins]).contiguous()
            wxs = torch.cat([o.weight.device_scale() for o in ins]).contiguous()
            dev = wx.device
            bx = torch.cat([o._bias_dev() if o.bias is not None
                            else torch.zeros(self.hidden, dtype=torch.float32, device=dev) for o in ins])
            uzr = torch.cat([self.update_state.weight.device_data(),
                             self.reset_state.weight.device_data()]).contiguous()
            uzrs = torch.cat([self.update_state.weight.device_scale(),
                              self.reset_state.weight.device_scale()]).contiguous()
            p = (wx, wxs, bx.contiguous(), uzr, uzrs, self.cand_state.weight.device_data(),
                 self.cand_state.weight.device_scale())
            self._packed = p
        return p


def gru_step_k(cell: GruCell, x_k: torch.Tensor, h_k: torch.Tensor, col_seg=None, nseg=1):
    """K-major GRU transition: x_k [P][in], h_k [P][H] -> h' [P][H]."""
    wx, wxs, bx, uzr, uzrs, uc, ucs = cell.packed()
    H = cell.hidden
    P = x_k.shape[0]
    f32 = wxs is None
    if f32:   # fp32 path: float products, no quantization
        gx = gemm_f32_kmajor(wx, x_k, bias=bx)
        gh = gemm_f32_kmajor(uzr, h_k)
    else:
        qx, sx = _quant_k(x_k, col_seg, nseg)
        qh, sh = _quant_k(h_k, col_seg, nseg)
        gx = gemm_kmajor(wx, wxs, H, qx, sx, col_seg=col_seg, bias=bx, w_static=True)   # [P][3H]
        gh = gemm_kmajor(uzr, uzrs, H, qh, sh, col_seg=col_seg, w_static=True)   # [P][2H]
    z = torch.empty((P, H), dtype=torch.float32, device=x_k.device)
    rh = torch.empty_like(z)
    flag = _dev.flag()
    st = _dev.stream_ptr()
    _lib.call("qnmt_gru_gates", gx.data_ptr(), 3 * H, None, gh.data_ptr(), 2 * H, h_k.data_ptr(),
              _dev.ld(h_k), P, H, z.data_ptr(), rh.data_ptr(), flag.data_ptr(), st)
    if f32:
        ghc = gemm_f32_kmajor(uc, rh)
    else:
        qr, sr = _quant_k(rh, col_seg, nseg)
        ghc = gemm_kmajor(uc, ucs, H, qr, sr, col_seg=col_seg, w_static=True)    # [P][H]
    out = torch.empty_like(z)
    _lib.call("qnmt_gru_combine", gx.data_ptr(), 3 * H, None, ghc.data_ptr(), H, z.data_ptr(),
              h_k.data_ptr(), _dev.ld(h_k), P, H, out.data_ptr(), H, None, 0, None, flag.data_ptr(), st)
    return out


def gru_step(cell: GruCell, x, h_prev, timer=None):
    """One GRU transition over a column batch (layers.py:170-181)."""
    if np.shape(h_prev)[0] != cell.hidden:
        raise ShapeError(f"state has {np.shape(h_prev)[0]} rows, cell expects {cell.hidden}")
    if np.shape(x)[0] != cell.update_in.in_dim:
        raise ShapeError(f"LinearOp expects [{cell.update_in.in_dim}, P] input, got {tuple(np.shape(x))}")
    f = _dev.reset_flag()
    out = gru_step_k(cell, _dev.kmajor(x), _dev.kmajor(h_prev))
    _dev.raise_flag(f)
    return _out(out, x)


# ---------------------------------------------------------------------------
# attention (layers.py:188-241)
# ---------------------------------------------------------------------------

@dataclass(eq=False)
class AttentionNet:
    enc_proj: LinearOp    # consumes the 2*hidden encoder states
    state_proj: LinearOp  # consumes the decoder query state
    scorer: LinearOp      # one real value per encoder state

    def __post_init__(self):
        if self.enc_proj.in_dim != 2 * self.state_proj.in_dim:
            raise ShapeError("encoder projection must consume twice the hidden size")
        if self.scorer.out_dim != 1:
            raise ShapeError("attention scorer must produce a single value")


class EncoderStates:
    """Per-sentence encoder output (layers.py:201-211).

    Device storage is position-major (``states_k`` [l][2H], ``att_proj_k``
    [l][A]); ``states`` / ``att_proj`` / ``s0`` give the reference's
    ``[features, l]`` views (numpy when constructed from numpy)."""

    def __init__(self, states, att_proj, s0, _kmajor=False):
        if _kmajor:
            self.states_k, self.att_proj_k, self.s0_k = states, att_proj, s0
            self._numpy = False
        else:
            self._numpy = _dev.is_numpy(states)
            self.states_k = _dev.kmajor(states)
            self.att_proj_k = _dev.kmajor(att_proj)
            self.s0_k = _dev.kmajor(s0)

    @property
    def states(self):
        s = self.states_k.t()
        return s.contiguous().cpu().numpy() if self._numpy else s

    @property
    def att_proj(self):
        s = self.att_proj_k.t()
        return s.contiguous().cpu().numpy() if self._numpy else s

    @property
    def s0(self):
        s = self.s0_k.t()
        return s.contiguous().cpu().numpy() if self._numpy else s

    @property
    def length(self) -> int:
        return int(self.states_k.shape[0])

    def att_exp_k(self) -> torch.Tensor:
        """fl32(e^(2 att_proj)) [l][A] for the one-MUFU attention scorer (computed once)."""
        e = getattr(self, "_att_exp", None)
        if e is None:
            ap = self.att_proj_k.contiguous()
            self.att_proj_k = ap
            e = torch.empty_like(ap)
            _lib.call("qnmt_attention_exp", ap.data_ptr(), ap.numel(), e.data_ptr(), _dev.stream_ptr())
            self._att_exp = e
        return e


def _one_sentence_meta(length, P, dev):
    sent_row = torch.zeros(1, dtype=torch.int64, device=dev)
    sent_len = torch.full((1,), length, dtype=torch.int32, device=dev)
    col_sent = torch.zeros(P, dtype=torch.int32, device=dev)
    return sent_row, sent_len, col_sent


def attend_k(att: AttentionNet, q_k: torch.Tensor, enc: EncoderStates):
    """K-major attention: q_k [P][H] -> (ctx [P][2H], alpha [P][l])."""
    u = att.state_proj.apply_k(q_k)                                          # [P][A]
    P, A = u.shape
    length = enc.length
    H2 = enc.states_k.shape[1]
    dev = u.device
    ctx = torch.empty((P, H2), dtype=torch.float32, device=dev)
    alpha = torch.empty((P, length), dtype=torch.float32, device=dev)
    v = att.scorer.weight
    # The kernels take up to 16 query columns of one sentence per call (a beam).  u above was
    # quantized over the whole [hidden, P] block as the reference does (layers.py:221); the scorer
    # quantizes every column's tanh block on its own (layers.py:225-226), so wider queries are
    # simply processed 16 columns at a time.
    for c0 in range(0, P, 16):
        pc = min(16, P - c0)
        sent_row, sent_len, _ = _one_sentence_meta(length, pc, dev)
        col_off = torch.zeros(1, dtype=torch.int32, device=dev)
        ncols = torch.full((1,), pc, dtype=torch.int32, device=dev)
        scratch = torch.empty(pc * (length + 4) + 2 * A + pc * A + 1024, dtype=torch.int32, device=dev)
        uc, cc, ac = u[c0:c0 + pc], ctx[c0:c0 + pc], alpha[c0:c0 + pc]
        if not att.scorer.is_quantized:   # fp32 scorer (layers.py:226 with a float LinearOp)
            _lib.call("qnmt_attention_f32", uc.data_ptr(), A, pc, col_off.data_ptr(), ncols.data_ptr(), 1,
                      enc.att_proj_k.data_ptr(), enc.states_k.data_ptr(), sent_row.data_ptr(), sent_len.data_ptr(),
                      length, A, H2, att.scorer._wdev().data_ptr(), cc.data_ptr(), H2, ac.data_ptr(), length,
                      scratch.data_ptr(), _dev.flag().data_ptr(), _dev.stream_ptr())
        else:
            _lib.call("qnmt_attention", uc.data_ptr(), A, pc, col_off.data_ptr(), ncols.data_ptr(), 1,
                      enc.att_proj_k.data_ptr(), None, enc.att_exp_k().data_ptr(),
                      enc.states_k.data_ptr(), sent_row.data_ptr(), sent_len.data_ptr(), length, A, H2,
                      v.device_data().data_ptr(), v.device_scale().data_ptr(), cc.data_ptr(), H2,
                      ac.data_ptr(), length, scratch.data_ptr(), _dev.flag().data_ptr(), _dev.stream_ptr())
    return ctx, alpha


def attend(att: AttentionNet, s_query, enc: EncoderStates, timer=None):
    """Attention weights and context for each query column (layers.py:214-241).

    Returns ``(context [2*hidden, P], alpha [l, P])``."""
    f = _dev.reset_flag()
    ctx, alpha = attend_k(att, _dev.kmajor(s_query), enc)
    _dev.raise_flag(f)
    return _out(ctx, s_query), _out(alpha, s_query)


# ---------------------------------------------------------------------------
# output network (layers.py:248-266)
# ---------------------------------------------------------------------------

@dataclass(eq=False)
class OutputNet:
    state_proj: LinearOp  # [readout, hidden], carries the readout bias
    embed_proj: LinearOp  # [readout, embed]
    ctx_proj: LinearOp    # [readout, 2*hidden]
    vocab_proj: LinearOp  # [vocab, readout]

    def logits_k(self, s_k, emb_k, ctx_k):
        ro = self.state_proj.apply_k(s_k)
        self.embed_proj.apply_k(emb_k, out=ro, accumulate=True)
        self.ctx_proj.apply_k(ctx_k, out=ro, accumulate=True)
        f = _dev.flag()
        _lib.call("qnmt_tanh", ro.data_ptr(), ro.shape[0], ro.shape[1], _dev.ld(ro), ro.data_ptr(),
                  _dev.ld(ro), f.data_ptr(), _dev.stream_ptr())
        return self.vocab_proj.apply_k(ro)

    def logits(self, s, prev_embed, context, timer=None):
        f = _dev.reset_flag()
        y = self.logits_k(_dev.kmajor(s), _dev.kmajor(prev_embed), _dev.kmajor(context))
        _dev.raise_flag(f)
        return _out(y, s)

    @property
    def vocab_size(self) -> int:
        return self.vocab_proj.out_dim


# ---------------------------------------------------------------------------
# assembled network (layers.py:273-435)
# ---------------------------------------------------------------------------

class DecoderState:
    """Recurrent decoder state (layers.py:273-282): one column per beam."""

    def __init__(self, s, s_prime):
        self.s = s
        self.s_prime = s_prime

    def select(self, idx) -> "DecoderState":
        if _dev.is_numpy(self.s):
            return DecoderState(np.ascontiguousarray(self.s[:, idx]),
                                np.ascontiguousarray(self.s_prime[:, idx]))
        i = torch.as_tensor(np.asarray(idx), device=self.s.device, dtype=torch.int64)
        return DecoderState(self.s[:, i], self.s_prime[:, i])


class Network:
    """Inference network for one quantized model (layers.py:285-384).

    ``encode`` and ``decoder_step`` run the C engine (csrc/engine.cu) -- the
    same code path as batched translation."""

    def __init__(self, qmodel, dims, src_embed, tgt_embed, enc_fwd, enc_bwd, dec_r, dec_q,
                 attention, output, s0_op, s0_mode, attention_query, precision, src_ids_fn,
                 tgt_tokens):
        self.qmodel = qmodel
        self.dims = dims
        self.src_embed = src_embed
        self.tgt_embed = tgt_embed
        self.enc_fwd, self.enc_bwd, self.dec_r, self.dec_q = enc_fwd, enc_bwd, dec_r, dec_q
        self.attention = attention
        self.output = output
        self.s0_op = s0_op
        self.s0_mode = s0_mode
        self.attention_query = attention_query
        self.precision = precision
        self.src_ids = src_ids_fn
        self.tgt_tokens = tgt_tokens

    @contextlib.contextmanager
    def engine(self, n=1, length=1, beam=1):
        """An engine of the model's pool, checked out for one call (networks are
        shared between threads, layers.py:285-290); the stream is synchronised
        before the engine goes back, so its scratch is free for the next caller."""
        pool = engine_pool(self.qmodel)
        e = pool.acquire(self.qmodel, n, length, min(max(beam, 8), 16))
        try:
            yield e
        finally:
            try:
                torch.cuda.current_stream().synchronize()
            finally:
                pool.release(e)

    def encode(self, src_ids, timer=None) -> EncoderStates:
        ids = np.asarray(src_ids, dtype=np.int64)
        if ids.size == 0:
            raise EmptyInputError("cannot encode an empty sentence")
        if ids.min() < 0 or ids.max() >= self.dims.src_vocab:
            raise VocabError(f"source id outside [0, {self.dims.src_vocab})")
        with self.engine(1, ids.size, 1) as e:
            states, att, s0, _, _ = e.encode_batch([ids])
        enc = EncoderStates(states, att, s0, _kmajor=True)
        enc._numpy = True
        return enc

    def initial_state(self, enc: EncoderStates, width: int = 1) -> DecoderState:
        s = enc.s0_k.repeat(width, 1)                  # [width][H]
        if enc._numpy:
            sn = s.t().contiguous().cpu().numpy()
            return DecoderState(sn, sn.copy())
        return DecoderState(s.t(), s.clone().t())

    def decoder_step(self, y_prev, state: DecoderState, enc: EncoderStates, timer=None):
        """One decode step over the live hypothesis columns (layers.py:356-384).

        Returns ``(log_probs [vocab, P], new_state, alpha [l, P])``."""
        ids = np.asarray(y_prev.cpu() if isinstance(y_prev, torch.Tensor) else y_prev, dtype=np.int64)
        if ids.min() < 0 or ids.max() >= self.dims.tgt_vocab:
            raise VocabError(f"target id outside [0, {self.dims.tgt_vocab})")
        P = ids.size
        s_k, sp_k = _dev.kmajor(state.s), _dev.kmajor(state.s_prime)
        dev = s_k.device
        y = torch.from_numpy(ids.astype(np.int32)).to(dev)
        sent_row, sent_len, col_sent = _one_sentence_meta(enc.length, P, dev)
        with self.engine(1, enc.length, P) as e:
            logits, s_int, s_new, alpha = e.decoder_step(y, s_k, sp_k, enc.states_k, enc.att_proj_k,
                                                         sent_row, sent_len, col_sent)
        lp = torch.empty_like(logits)
        f = _dev.reset_flag()
        _lib.call("qnmt_log_softmax", logits.data_ptr(), P, logits.shape[1], _dev.ld(logits),
                  lp.data_ptr(), _dev.ld(lp), f.data_ptr(), _dev.stream_ptr())
        _dev.raise_flag(f, numeric_msg="log_softmax received non-finite logits")
        like = state.s
        return _out(lp, like), DecoderState(_out(s_new, like), _out(s_int, like)), _out(alpha, like)


def encode(network: Network, src_ids, timer=None) -> EncoderStates:
    return network.encode(src_ids, timer)


def decoder_step(network: Network, y_prev, state, enc, timer=None):
    return network.decoder_step(y_prev, state, enc, timer)


def build_network(model, timer=None) -> Network:
    """Wrap a float (:class:`ModelParams`, fp32 path) or quantized parameter set
    in an inference network (layers.py:395-435)."""
    from .model import Float32Model, ModelParams, QuantizedModel, to_device_f32
    if isinstance(model, ModelParams):
        model = to_device_f32(model)
    if isinstance(model, Float32Model):
        f = model.f

        def lin(name, bias=None):
            return LinearOp(f[name], f[bias] if bias else None)
    elif isinstance(model, QuantizedModel):
        q, f = model.q, model.f

        def lin(name, bias=None):
            return LinearOp(q[name], f[bias] if bias else None)
    else:
        raise ConfigError("build_network needs ModelParams or a QuantizedModel")

    def cell(p) -> GruCell:
        return GruCell(update_in=lin(f"{p}.wz", f"{p}.bz"), update_state=lin(f"{p}.uz"),
                       reset_in=lin(f"{p}.wr", f"{p}.br"), reset_state=lin(f"{p}.ur"),
                       cand_in=lin(f"{p}.wc", f"{p}.bc"), cand_state=lin(f"{p}.uc"),
                       hidden=model.dims.hidden)

    att = AttentionNet(enc_proj=lin("attn.w_enc", "attn.b_enc"), state_proj=lin("attn.u_state"),
                       scorer=lin("attn.v"))
    out = OutputNet(state_proj=lin("out.w_state", "out.b_readout"), embed_proj=lin("out.w_embed"),
                    ctx_proj=lin("out.w_ctx"), vocab_proj=lin("out.w_vocab", "out.b_vocab"))
    return Network(model, model.dims, f["src_embed"], f["tgt_embed"], cell("enc_fwd"), cell("enc_bwd"),
                   cell("dec_r"), cell("dec_q"), att, out, lin("s0.w", "s0.b"), model.s0_mode,
                   model.attention_query, model.precision, model.src_ids, model.tgt_tokens)
