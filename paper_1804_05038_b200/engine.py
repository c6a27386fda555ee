"""Python handle on the C engine (csrc/engine.cu): batched encode, decoder
step and device-resident translation of many sentences."""

from __future__ import annotations

import ctypes as C
import math
import threading

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
        lib = _lib.load()   # byte counts of the copies the C engine issued for this batch
        self.h2d_bytes += int(lib.qnmt_last_h2d_bytes(self._h))
        self.d2h_bytes += int(lib.qnmt_last_d2h_bytes(self._h))
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


_POOL_LOCK = threading.Lock()


class EnginePool:
    """The engines of one device model, handed to one caller at a time.

    The reference's API is safe to call concurrently (bench.py:129-132 and
    cli.py:58-63 run ``translate`` from a thread pool on one model).  An engine
    owns device scratch, pinned staging and the search history of the batch it
    is decoding, so two threads must never share one: :meth:`acquire` checks an
    idle engine out (or creates one) under a lock and :meth:`release` returns
    it.  Engines are only closed while idle, so a decode in flight never loses
    its engine; an engine that is outgrown is closed when a larger one is made."""

    def __init__(self):
        self._lock = threading.Lock()
        self._idle: list = []
        self.all: list = []       # every live engine (per-engine traffic counters)

    def _cap(self, n, length, beam):
        big = self.all
        return (max([n] + [e.max_sentences for e in big]), max([length, 128] + [e.max_len for e in big]),
                max([beam] + [e.max_beam for e in big]))

    def capacity(self, n, length, beam):
        """The capacity a new engine for (n, length, beam) gets: at least every existing engine's."""
        with self._lock:
            return self._cap(n, length, beam)

    def acquire(self, qmodel, n: int, length: int, beam: int, exact=None) -> Engine:
        with self._lock:
            for i, e in enumerate(self._idle):
                ok = ((e.max_sentences, e.max_len, e.max_beam) == tuple(exact)) if exact else e.fits(n, length, beam)
                if ok:
                    return self._idle.pop(i)
            cap = tuple(exact) if exact else self._cap(n, length, beam)
            # idle engines that the new one covers are closed (bounded device memory)
            keep = []
            for e in self._idle:
                if e.max_sentences <= cap[0] and e.max_len <= cap[1] and e.max_beam <= cap[2]:
                    e.close()
                    self.all.remove(e)
                else:
                    keep.append(e)
            self._idle = keep
            e = Engine(qmodel, *cap)
            self.all.append(e)
            return e

    def release(self, e: Engine):
        with self._lock:
            if e._h is not None:
                self._idle.append(e)

    def close(self):
        with self._lock:
            for e in self._idle:
                e.close()
            self.all = [e for e in self.all if e not in self._idle]
            self._idle = []


def engine_pool(qmodel) -> EnginePool:
    """The model's engine pool (created once, thread-safe)."""
    pool = getattr(qmodel, "_engine_pool", None)
    if pool is None:
        with _POOL_LOCK:
            pool = getattr(qmodel, "_engine_pool", None)
            if pool is None:
                pool = EnginePool()
                qmodel._engine_pool = pool
    return pool
