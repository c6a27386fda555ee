"""Beam-search translation on B200 (drop-in for qnmt.decoder).

:func:`translate` keeps the reference signature (decoder.py:88-160) and runs
the device-resident engine for one sentence.  :func:`translate_batch` is the
B200-native bulk entry: many sentences per engine call, each one decoded
exactly as ``translate`` would (per-sentence activation scales, per-sentence
search state), so results are identical to a sentence-by-sentence loop.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, EmptyInputError
from .engine import Engine
from .model import EOS_ID, ModelParams, QuantizedModel, quantize_model


@dataclass
class DecodeConfig:
    beam: int = 5
    max_ratio: float = 3.0        # max output length = ceil(ratio * source len) + 1
    precision: str = "int8"       # the B200 path decodes int8 (fp32 is SURVEY 8(f) "next")

    def __post_init__(self):
        if self.beam < 1:
            raise ConfigError(f"beam must be >= 1, got {self.beam}")
        if not self.max_ratio > 0:
            raise ConfigError(f"max_ratio must be positive, got {self.max_ratio}")
        if self.precision not in ("fp32", "int8"):
            raise ConfigError(f"unknown precision {self.precision!r}")


@dataclass
class BeamHypothesis:
    """A partial translation: emitted ids, accumulated log-prob, decoder state."""

    tokens: list
    log_prob: float
    state: object = None
    finished: bool = False


def _single_model(models) -> QuantizedModel:
    if isinstance(models, (ModelParams, QuantizedModel)):
        members = [models]
    else:
        members = list(models)
    if not members:
        raise ConfigError("at least one model is required")
    if len(members) > 1:
        raise ConfigError("ensemble decoding is not implemented on the B200 path")
    m = members[0]
    if isinstance(m, ModelParams):
        m = _quantized_cache(m)
    return m


def _quantized_cache(params: ModelParams) -> QuantizedModel:
    qm = getattr(params, "_b200_quantized", None)
    if qm is None:
        qm = quantize_model(params)
        params._b200_quantized = qm
    return qm


def _engine_for(qm: QuantizedModel, n: int, length: int, beam: int) -> Engine:
    e = getattr(qm, "_engine", None)
    if e is None or not e.fits(n, length, beam):
        cap = (max(n, e.max_sentences if e else 0), max(length, 128, e.max_len if e else 0),
               max(beam, e.max_beam if e else 0))
        if e is not None:
            e.close()
        e = Engine(qm, *cap)
        qm._engine = e
    return e


def _check_cfg(cfg: DecodeConfig):
    if cfg.precision != "int8":
        raise ConfigError("the B200 path decodes int8 only (fp32 decoding is not implemented)")
    if cfg.beam > 16:
        raise ConfigError("beam > 16 is not supported by the device search")


def translate(models, source_tokens, cfg: DecodeConfig, timer=None):
    """Beam-search translation of one pre-tokenized sentence (decoder.py:88-160).

    Returns ``(target_tokens, log_prob)``: the token list excludes the final
    EOS; the score is the plain sum of per-step log-probs."""
    tokens = list(source_tokens)
    if not tokens:
        raise EmptyInputError("cannot translate an empty sentence")
    _check_cfg(cfg)
    qm = _single_model(models)
    ids = qm.src_ids(tokens)
    e = _engine_for(qm, 1, len(ids), cfg.beam)
    out, lps = e.translate_ids([ids], cfg.beam, cfg.max_ratio)
    return [qm.tgt_tokens[i] for i in out[0]], lps[0]


def translate_batch(model, sentences, cfg: DecodeConfig, max_batch: int = 256, return_ids=False):
    """Translate a corpus with batched device decoding (B200-native bulk path).

    ``sentences``: token lists / whitespace strings, or (``return_ids``) id
    lists.  Output order follows the input.  Each batch of up to
    ``max_batch`` sentences is one engine call."""
    _check_cfg(cfg)
    qm = _single_model(model)
    sents = [s.split() if isinstance(s, str) else list(s) for s in sentences]
    if not sents:
        return []
    if any(len(s) == 0 for s in sents):
        raise EmptyInputError("cannot translate an empty sentence")
    ids = [np.asarray(s, dtype=np.int64) if return_ids else qm.src_ids(s) for s in sents]
    max_len = max(len(x) for x in ids)
    e = _engine_for(qm, min(max_batch, len(ids)), max_len, cfg.beam)
    results = []
    for b0 in range(0, len(ids), max_batch):
        toks, lps = e.translate_ids(ids[b0:b0 + max_batch], cfg.beam, cfg.max_ratio)
        for t, lp in zip(toks, lps):
            results.append((t if return_ids else [qm.tgt_tokens[i] for i in t], lp))
    return results


def max_steps(length: int, max_ratio: float) -> int:
    """decoder.py:103."""
    return math.ceil(max_ratio * length) + 1


def bpe_merge(tokens) -> str:
    """Reassemble BPE subword units (decoder.py:163-177)."""
    words = []
    buf = ""
    for t in tokens:
        if t.endswith("@@"):
            buf += t[:-2]
        else:
            words.append(buf + t)
            buf = ""
    if buf:
        words.append(buf)
    return " ".join(words)


__all__ = ["DecodeConfig", "BeamHypothesis", "translate", "translate_batch", "bpe_merge",
           "max_steps", "EOS_ID"]
