"""Python handle on the C engine (csrc/engine.cu): batched encode, decoder
step and device-resident translation of many sentences."""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _dev, _lib
from .errors import ConfigError, EmptyInputError, VocabError


class Engine:
    """Scratch for up to ``max_sentences`` sentences of length <= ``max_len``
    at beam <= ``max_beam`` for one :class:`QuantizedModel`."""

    def __init__(self, qmodel, max_sentences: int, max_len: int, max_beam: int):
        _dev.require_cuda()
        self.qmodel = qmodel
        self.max_sentences, self.max_len, self.max_beam = max_sentences, max_len, max_beam
        h = C.c_void_p()
        _lib.call("qnmt_engine_create", qmodel.handle(), max_sentences, max_len, max_beam, C.byref(h))
        self._h = h
        self.h2d_bytes = 0   # host<->device traffic of translate_ids calls (ids + metadata in, results out)
        self.d2h_bytes = 0

    def fits(self, n, length, beam) -> bool:
        return n <= self.max_sentences and length <= self.max_len and beam <= self.max_beam

    @property
    def device_bytes(self) -> int:
        return int(_lib.load().qnmt_engine_bytes(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None:
            _lib.load().qnmt_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- phase profiler (eager steps, CUDA events per phase group) -------------
    PHASE_GROUPS = ("encoder", "embedding", "quantize-activations", "matmul", "gru", "attention", "matmul-vocab",
                    "topk", "search", "gather", "other")

    def profile(self, enable: bool):
        """Enable (resetting the totals) or disable the engine's phase profiler;
        while enabled the decode loop runs eagerly (no CUDA graphs)."""
        _lib.call("qnmt_engine_profile", self._h, 1 if enable else 0)

    def profile_read(self) -> dict:
        """{group: milliseconds} accumulated since :meth:`profile` (True)."""
        ms, calls, ops, nb = ((C.c_double * 16)() for _ in range(4))
        n = _lib.load().qnmt_engine_profile_read(self._h, ms, calls, ops, nb)
        return {self.PHASE_GROUPS[i]: ms[i] for i in range(min(n, len(self.PHASE_GROUPS)))}

    # -- encoder -------------------------------------------------------------
    def encode_batch(self, id_lists):
        """Returns device (states [sum_l][2H], att_proj [sum_l][A], s0 [n][H], rows)."""
        d = self.qmodel.dims
        lens = np.array([len(x) for x in id_lists], dtype=np.int32)
        if len(lens) == 0 or (lens == 0).any():
            raise EmptyInputError("cannot encode an empty sentence")
        ids = np.concatenate([np.asarray(x, dtype=np.int64) for x in id_lists])
        if ids.min() < 0 or ids.max() >= d.src_vocab:
            raise VocabError(f"source id outside [0, {d.src_vocab})")
        dev = _dev.require_cuda()
        P = int(lens.sum())
        ids_d = torch.from_numpy(ids.astype(np.int32)).to(dev)
        states = torch.empty((P, 2 * d.hidden), dtype=torch.float32, device=dev)
        att = torch.empty((P, d.attn), dtype=torch.float32, device=dev)
        s0 = torch.empty((len(lens), d.hidden), dtype=torch.float32, device=dev)
        _lib.call("qnmt_encode_batch", self._h, ids_d.data_ptr(), lens.ctypes.data, len(lens),
                  states.data_ptr(), att.data_ptr(), s0.data_ptr(), _dev.stream_ptr())
        rows = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        return states, att, s0, rows, lens

    # -- one decoder step ----------------------------------------------------
    def decoder_step(self, y, s, sp, states, att_proj, sent_row, sent_len, col_sent, want_alpha=True):
        """All tensors device; s/sp K-major [N][H].  Returns (logits [N][V], s_int, s_new, alpha)."""
        d = self.qmodel.dims
        N = int(s.shape[0])
        dev = s.device
        max_len = int(sent_len.max().item()) if isinstance(sent_len, torch.Tensor) else int(max(sent_len))
        s_int = torch.empty((N, d.hidden), dtype=torch.float32, device=dev)
        s_new = torch.empty_like(s_int)
        logits = torch.empty((N, d.tgt_vocab), dtype=torch.float32, device=dev)
        alpha = torch.empty((N, max_len), dtype=torch.float32, device=dev) if want_alpha else None
        _lib.call("qnmt_decoder_step", self._h, N, col_sent.data_ptr(), int(sent_row.numel()),
                  y.data_ptr(), s.data_ptr(), sp.data_ptr(), states.data_ptr(), att_proj.data_ptr(),
                  sent_row.data_ptr(), sent_len.data_ptr(), max_len, s_int.data_ptr(), s_new.data_ptr(),
                  logits.data_ptr(), _dev.ptr(alpha), max_len if want_alpha else 0, _dev.stream_ptr())
        return logits, s_int, s_new, alpha

    # -- device-resident translation -----------------------------------------
    def translate_ids(self, id_lists, beam: int, max_ratio: float):
        """Translate many sentences (each exactly as decoder.translate).
        Returns (list of token-id lists without final EOS, list of log-probs)."""
        n = len(id_lists)
        if n == 0:
            return [], []
        lens = np.array([len(x) for x in id_lists], dtype=np.int32)
        if (lens == 0).any():
            raise EmptyInputError("cannot translate an empty sentence")
        if not self.fits(n, int(lens.max()), beam):
            raise ConfigError("batch exceeds engine capacity")
        ids = np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=np.int32) for x in id_lists]))
        stride = int(math.ceil(max_ratio * int(lens.max()))) + 1
        out_tok = np.zeros((n, stride), dtype=np.int32)
        out_len = np.zeros(n, dtype=np.int32)
        out_lp = np.zeros(n, dtype=np.float64)
        _lib.call("qnmt_translate_batch", self._h, ids.ctypes.data, lens.ctypes.data, n, beam,
                  float(max_ratio), out_tok.ctypes.data, stride, out_len.ctypes.data,
                  out_lp.ctypes.data, _dev.stream_ptr())
        # ids + per-sentence metadata (row, len, max_steps, P, col_off, col_sent, y, live) + encoder row maps
        self.h2d_bytes += ids.nbytes + n * 40 + 2 * 2 * n * int(lens.max()) * 4 + ids.nbytes + n * 4
        self.d2h_bytes += int(_lib.load().qnmt_last_d2h_bytes(self._h))
        toks = [out_tok[i, :out_len[i]].tolist() for i in range(n)]
        return toks, out_lp.tolist()


def translate_ensemble_ids(engines, id_lists_per_member, beam: int, max_ratio: float):
    """Ensemble translation (decoder.py:88-160, members averaged per step,
    :115-120) of many sentences; ``id_lists_per_member[i]`` are the source ids
    under member i's vocabulary.  Returns (token-id lists, log-probs)."""
    nm = len(engines)
    n = len(id_lists_per_member[0])
    if n == 0:
        return [], []
    lens = np.array([len(x) for x in id_lists_per_member[0]], dtype=np.int32)
    if (lens == 0).any():
        raise EmptyInputError("cannot translate an empty sentence")
    if any(not e.fits(n, int(lens.max()), beam) for e in engines):
        raise ConfigError("batch exceeds engine capacity")
    ids = np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=np.int32)
                                               for lists in id_lists_per_member for x in lists]))
    stride = int(math.ceil(max_ratio * int(lens.max()))) + 1
    out_tok = np.zeros((n, stride), dtype=np.int32)
    out_len = np.zeros(n, dtype=np.int32)
    out_lp = np.zeros(n, dtype=np.float64)
    hs = (C.c_void_p * nm)(*[e._h.value for e in engines])
    _lib.call("qnmt_translate_ensemble", C.cast(hs, C.c_void_p), nm, ids.ctypes.data, lens.ctypes.data, n, beam,
              float(max_ratio), out_tok.ctypes.data, stride, out_len.ctypes.data, out_lp.ctypes.data,
              _dev.stream_ptr())
    return [out_tok[i, :out_len[i]].tolist() for i in range(n)], out_lp.tolist()
