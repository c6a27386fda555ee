"""Beam-search translation on B200 (drop-in for qnmt.decoder).

:func:`translate` keeps the reference signature (decoder.py:88-160) and runs
the device-resident engine for one sentence.  :func:`translate_batch` is the
B200-native bulk entry: many sentences per engine call, each one decoded
exactly as ``translate`` would (per-sentence activation scales, per-sentence
search state), so results are identical to a sentence-by-sentence loop.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass, field

import numpy as np

from .bleu import bleu
from .errors import ConfigError, EmptyInputError, QnmtError
from .engine import engine_pool, translate_ensemble_ids
from .model import EOS_ID, Float32Model, ModelParams, QuantizedModel, quantize_model, to_device_f32


@dataclass
class DecodeConfig:
    beam: int = 5
    max_ratio: float = 3.0        # max output length = ceil(ratio * source len) + 1
    precision: str = "fp32"       # "fp32" or "int8" (the B200 hot path; bulk callers pass it)

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


def _members(models, precision: str = "int8") -> list:
    """Ensemble members as device models (decoder.py:46-71): a single model or a
    non-empty list sharing one target vocabulary.  int8: float parameters are
    quantized once and cached; fp32: float parameters only (uploaded once)."""
    if isinstance(models, (ModelParams, QuantizedModel, Float32Model)):
        members = [models]
    else:
        members = list(models)
    if not members:
        raise ConfigError("at least one model is required")
    first = members[0].tgt_tokens
    for m in members[1:]:
        if m.tgt_tokens != first:
            raise ConfigError("ensemble members must share the target vocabulary")
    if len(members) > 8:
        raise ConfigError("ensembles of more than 8 members are not supported")
    if precision == "fp32":
        if any(isinstance(m, QuantizedModel) for m in members):
            raise ConfigError("fp32 decoding requires float parameters")
        return [to_device_f32(m) if isinstance(m, ModelParams) else m for m in members]
    if any(isinstance(m, Float32Model) for m in members):
        raise ConfigError("int8 decoding needs ModelParams or QuantizedModel members")
    return [_quantized_cache(m) if isinstance(m, ModelParams) else m for m in members]


_CACHE_LOCK = threading.Lock()


def _quantized_cache(params: ModelParams) -> QuantizedModel:
    qm = getattr(params, "_b200_quantized", None)
    if qm is None:
        with _CACHE_LOCK:   # concurrent translate() calls on one ModelParams quantize it once
            qm = getattr(params, "_b200_quantized", None)
            if qm is None:
                qm = quantize_model(params)
                params._b200_quantized = qm
    return qm


def _acquire(members, n: int, length: int, beam: int) -> list:
    """Check out one engine per member (a model listed twice gets two); an
    ensemble's engines share one capacity.  Release with :func:`_release`."""
    if len(members) == 1:
        return [engine_pool(members[0]).acquire(members[0], n, length, beam)]
    cap = (n, max(length, 128), beam)
    for m in members:
        c = engine_pool(m).capacity(n, length, beam)
        cap = tuple(max(a, b) for a, b in zip(cap, c))
    got = []
    try:
        for m in members:
            got.append(engine_pool(m).acquire(m, n, length, beam, exact=cap))
    except BaseException:
        _release(members, got)
        raise
    return got


def _release(members, engines):
    for m, e in zip(members, engines):
        engine_pool(m).release(e)


def _check_cfg(cfg: DecodeConfig):
    if cfg.beam > 16:
        raise ConfigError("beam > 16 is not supported by the device search")


_STREAMS: dict = {}


def _side_streams(k: int) -> list:
    """k CUDA streams of the current device, created once (one per pipelined engine)."""
    import torch
    dev = torch.cuda.current_device()
    lst = _STREAMS.setdefault(dev, [])
    while len(lst) < k:
        lst.append(torch.cuda.Stream(device=dev))
    return lst[:k]


# engine phase groups (csrc/engine.cu PG_*) -> reference phase names (bench.py:23-24)
GROUP_TO_PHASE = {"quantize-activations": "quantize-activations", "matmul": "matmul", "matmul-vocab": "matmul",
                  "gru": "transcendental", "attention": "transcendental", "embedding": "embedding",
                  "topk": "search-overhead", "search": "search-overhead", "gather": "search-overhead",
                  "encoder": "encoder", "other": "other"}


def _charge_timer(timer, phases: dict):
    """Add device-measured phase seconds to a reference PhaseTimer (its
    ``seconds`` dict, bench.py:27-57)."""
    sec = getattr(timer, "seconds", None)
    if not isinstance(sec, dict):
        raise ConfigError("timer must be a PhaseTimer (an object with a 'seconds' dict)")
    for k, v in phases.items():
        sec[k] = sec.get(k, 0.0) + v


def _decode_ids(members, per_member_ids, cfg: DecodeConfig, max_batch: int, streams: int = 1, sort: bool = False,
                phases: dict = None):
    """Batched device decode of id lists (one list per member).  Returns [(ids, logp)]
    in input order.

    ``sort``: batches are cut from the length-sorted corpus (stable), so the
    sentences of one engine call need similar step counts (ceil(ratio*l)+1) and
    the device runs full-width steps instead of a long tail of a few live
    sentences.  ``streams`` > 1 (single model): that many engines, each on its
    own CUDA stream driven by its own host thread, take batches from a shared
    queue -- one engine's host-side turnaround (polls, result fetch, graph
    launches) and its small latency-bound kernels overlap the other engines'
    device work.  Every sentence is still decoded exactly as decoder.translate
    would (results do not depend on batching).  The queue hands out the longest
    batches first.

    ``phases`` (a dict): the decode runs with the engine's device phase
    profiler (eager steps, CUDA events per phase group, one stream) and adds
    {reference phase name: seconds} into it."""
    n_all = len(per_member_ids[0])
    order = sorted(range(n_all), key=lambda i: (len(per_member_ids[0][i]), i)) if sort else list(range(n_all))
    batches = [order[b0:b0 + max_batch] for b0 in range(0, n_all, max_batch)]
    max_len = max(len(x) for x in per_member_ids[0])
    nb = min(max_batch, n_all)
    out = [None] * n_all

    def put(idx, toks, lps):
        for i, t, lp in zip(idx, toks, lps):
            out[i] = (t, lp)

    if len(members) > 1:
        engines = _acquire(members, nb, max_len, cfg.beam)
        try:
            for idx in batches:
                put(idx, *translate_ensemble_ids(engines, [[ids[i] for i in idx] for ids in per_member_ids],
                                                 cfg.beam, cfg.max_ratio))
        finally:
            _release(members, engines)
        return out
    ids0 = per_member_ids[0]
    k = max(1, min(streams, len(batches)))
    pool = engine_pool(members[0])
    engines = []
    try:
        if phases is not None:
            k = 1
        for _ in range(k):
            engines.append(pool.acquire(members[0], nb, max_len, cfg.beam))
        if phases is not None:
            e = engines[0]
            e.profile(True)
            try:
                for idx in batches:
                    put(idx, *e.translate_ids([ids0[i] for i in idx], cfg.beam, cfg.max_ratio))
                groups = e.profile_read()
            finally:
                e.profile(False)
            for g, ms in groups.items():
                ph = GROUP_TO_PHASE.get(g, "other")
                phases[ph] = phases.get(ph, 0.0) + ms * 1e-3
            return out
        if k == 1:
            for idx in batches:
                put(idx, *engines[0].translate_ids([ids0[i] for i in idx], cfg.beam, cfg.max_ratio))
            return out
        _run_streams(engines, batches, ids0, cfg, put)
    finally:
        for e in engines:
            pool.release(e)
    return out


def _run_streams(engines, batches, ids0, cfg, put):
    """Engines on their own CUDA streams and host threads take batches from a
    shared queue (see _decode_ids)."""
    import torch
    k = len(engines)
    # longest batches first (LPT): the engines drain the short ones together at the end
    # instead of one engine finishing the longest batch alone
    queue = sorted(range(len(batches)), key=lambda b: (-max(len(ids0[i]) for i in batches[b]), b))
    lock = threading.Lock()
    errors = []
    main = torch.cuda.current_stream()
    sides = _side_streams(k)

    def worker(j):
        try:
            sides[j].wait_stream(main)
            with torch.cuda.stream(sides[j]):
                while True:
                    with lock:
                        if not queue or errors:
                            return
                        b = queue.pop(0)
                    idx = batches[b]
                    put(idx, *engines[j].translate_ids([ids0[i] for i in idx], cfg.beam, cfg.max_ratio))
        except BaseException as exc:   # noqa: BLE001 -- re-raised in the caller's thread
            with lock:
                errors.append(exc)

    threads = [threading.Thread(target=worker, args=(j,)) for j in range(k)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for s in sides:
        main.wait_stream(s)
    if errors:
        raise errors[0]


def translate(models, source_tokens, cfg: DecodeConfig, timer=None):
    """Beam-search translation of one pre-tokenized sentence (decoder.py:88-160).

    Returns ``(target_tokens, log_prob)``: the token list excludes the final
    EOS; the score is the plain sum of per-step log-probs (ensemble members
    contribute the arithmetic mean of their log-probs per step).

    ``timer`` (a reference PhaseTimer): the decode runs with the engine's
    device phase profiler and the measured seconds are added to the timer's
    phases (device time per phase group instead of host wall-clock spans)."""
    tokens = list(source_tokens)
    if not tokens:
        raise EmptyInputError("cannot translate an empty sentence")
    _check_cfg(cfg)
    members = _members(models, cfg.precision)
    ids = [[m.src_ids(tokens)] for m in members]
    phases = {} if timer is not None and len(members) == 1 else None
    if timer is not None and phases is None:
        raise ConfigError("phase timing of ensemble decodes is not supported")
    out, lp = _decode_ids(members, ids, cfg, 1, phases=phases)[0]
    if timer is not None:
        _charge_timer(timer, phases)
    return [members[0].tgt_tokens[i] for i in out], lp


def shard_batches(lengths, max_batch: int, world: int) -> list:
    """Sentence sharding of the bulk path over ``world`` devices:
    the corpus is sorted by length (stable), cut into batches of ``max_batch``
    sentences, and the batches are dealt to the devices in snake order
    (0..W-1, W-1..0, ...), so every device sees the whole length range and the
    devices' decode work is balanced.  Returns, per device, its list of batches
    (lists of corpus indices).  No data moves between devices: each decodes
    its own sentences against its own replica of the weights."""
    order = sorted(range(len(lengths)), key=lambda i: (lengths[i], i))
    batches = [order[i:i + max_batch] for i in range(0, len(order), max_batch)]
    out = [[] for _ in range(world)]
    for k, b in enumerate(batches):
        r = k % world if (k // world) % 2 == 0 else world - 1 - k % world
        out[r].append(b)
    return out


def _translate_devices(members, ids, cfg, max_batch, streams, devices):
    """translate_batch over several GPUs: one host thread per device decodes the
    device's shard (shard_batches) with its own replica of the model and its
    own engines/streams; results are reassembled in input order.  The
    reference's fan-out this replaces is bench.py:129-132 / cli.py:58-63
    (sentences over a thread pool)."""
    import torch
    from .model import replicate
    if len(members) > 1:
        raise ConfigError("multi-device decoding of ensembles is not supported")
    lens = [len(x) for x in ids[0]]
    shards = shard_batches(lens, max_batch, len(devices))
    out = [None] * len(lens)
    reps = [replicate(members[0], d) for d in devices]
    errors = []

    def worker(r):
        try:
            torch.cuda.set_device(devices[r])
            flat = [i for b in shards[r] for i in b]
            if not flat:
                return
            res = _decode_ids([reps[r]], [[ids[0][i] for i in flat]], cfg, max_batch, streams=streams, sort=True)
            for i, v in zip(flat, res):
                out[i] = v
        except BaseException as exc:   # noqa: BLE001 -- re-raised in the caller's thread
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(len(devices))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out


def translate_batch(models, sentences, cfg: DecodeConfig, max_batch: int = 256, return_ids=False,
                    streams: int = 3, sort: bool = True, devices=None):
    """Translate a corpus with batched device decoding (B200-native bulk path).

    ``models``: one model or an ensemble list.  ``sentences``: token lists /
    whitespace strings, or (``return_ids``) id lists.  Output order follows
    the input.  Each batch of up to ``max_batch`` sentences is one engine call;
    batches are cut from the length-sorted corpus and pipelined over
    ``streams`` engines (see ``_decode_ids``).  ``devices`` (a list of CUDA
    device indices): the sorted batches are sharded over those GPUs
    (``shard_batches``), each decoding its shard against its own replica of
    the weights with no collective.  Results are identical to
    sentence-by-sentence ``translate`` on any device count."""
    _check_cfg(cfg)
    members = _members(models, cfg.precision)
    if return_ids:   # id arrays pass through untouched (no per-token Python objects on the bulk path)
        sents = [s if isinstance(s, np.ndarray) and s.ndim == 1 else np.asarray(list(s), dtype=np.int64)
                 for s in sentences]
    else:
        sents = [s.split() if isinstance(s, str) else list(s) for s in sentences]
    if not sents:
        return []
    if any(len(s) == 0 for s in sents):
        raise EmptyInputError("cannot translate an empty sentence")
    if return_ids:
        ids = [sents] * len(members)
    else:
        ids = [[m.src_ids(s) for s in sents] for m in members]
    tgt = members[0].tgt_tokens
    if devices is not None and len(devices) > 0:
        res = _translate_devices(members, ids, cfg, max_batch, streams, list(devices))
    else:
        res = _decode_ids(members, ids, cfg, max_batch, streams=streams, sort=sort)
    return [(t if return_ids else [tgt[i] for i in t], lp) for t, lp in res]


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


def edit_distance(a, b) -> int:
    """Levenshtein distance between two token sequences (decoder.py:180-190)."""
    if len(a) < len(b):
        a, b = b, a
    row = list(range(len(b) + 1))
    for i, x in enumerate(a, 1):
        prev_diag, row[0] = row[0], i
        for j, y in enumerate(b, 1):
            cur = min(row[j] + 1, row[j - 1] + 1, prev_diag + (x != y))
            prev_diag, row[j] = row[j], cur
    return row[-1]


@dataclass
class ParityReport:
    """Output agreement between the two precision modes on one corpus (decoder.py:193-213)."""

    sentences: int
    identical: int
    identical_fraction: float
    edit_distances: list
    mean_edit_distance: float
    bleu_int8_vs_fp32: float
    fp32_outputs: list = field(repr=False, default_factory=list)
    int8_outputs: list = field(repr=False, default_factory=list)

    def to_dict(self) -> dict:
        return {"sentences": self.sentences, "identical": self.identical,
                "identical_fraction": self.identical_fraction, "mean_edit_distance": self.mean_edit_distance,
                "bleu_int8_vs_fp32": self.bleu_int8_vs_fp32, "edit_distances": list(self.edit_distances)}


def compare_precisions(model: ModelParams, sentences, cfg: DecodeConfig, max_batch: int = 256) -> ParityReport:
    """Decode every sentence under fp32 and int8 and measure agreement
    (decoder.py:216-248).  Both precisions run batched on the device; results
    are identical to the reference's sentence-by-sentence loop."""
    sents = [s.split() if isinstance(s, str) else list(s) for s in sentences]
    if not sents:
        raise EmptyInputError("no sentences to compare")
    for i, s in enumerate(sents):
        if not s:
            raise EmptyInputError(f"sentence {i}: cannot translate an empty sentence")
    if not isinstance(model, ModelParams):
        raise ConfigError("compare_precisions needs float parameters")
    cfg32 = DecodeConfig(cfg.beam, cfg.max_ratio, "fp32")
    cfg8 = DecodeConfig(cfg.beam, cfg.max_ratio, "int8")
    try:
        out32 = translate_batch(model, sents, cfg32, max_batch)
        out8 = translate_batch(model, sents, cfg8, max_batch)
    except QnmtError:
        # a batch failed: find the sentence as the reference's per-sentence loop would
        # and name it (decoder.py:227-232)
        for i, s in enumerate(sents):
            try:
                translate(model, s, cfg32)
                translate(model, s, cfg8)
            except QnmtError as exc:
                raise type(exc)(f"sentence {i}: {exc}") from exc
        raise
    d = [edit_distance(a[0], b[0]) for a, b in zip(out32, out8)]
    same = sum(a[0] == b[0] for a, b in zip(out32, out8))
    f32_txt = [bpe_merge(a[0]) for a in out32]
    i8_txt = [bpe_merge(b[0]) for b in out8]
    return ParityReport(sentences=len(sents), identical=same, identical_fraction=same / len(sents),
                        edit_distances=d, mean_edit_distance=float(np.mean(d)),
                        bleu_int8_vs_fp32=bleu(i8_txt, f32_txt), fp32_outputs=f32_txt, int8_outputs=i8_txt)


__all__ = ["DecodeConfig", "BeamHypothesis", "translate", "translate_batch", "bpe_merge",
           "max_steps", "EOS_ID", "edit_distance", "ParityReport", "compare_precisions"]
