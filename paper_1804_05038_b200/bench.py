"""Throughput measurement and phase profiling of the B200 decode paths
(drop-in for qnmt.bench).

Same report as the reference (bench.py:60-92): words per second (WPS, target
tokens excluding EOS) over the corpus, words per core-second (WPCS = WPS /
workers), wall time = median of an odd number of repeats after one untimed
warm-up.  On B200 one host thread drives batched device decoding
(:func:`translate_batch`, up to ``batch`` sentences per engine call), so
``workers`` is the number of host threads (1) and WPCS = WPS.

Phase accounting: the reference instruments its timed runs with a host
PhaseTimer.  Here the timed runs stay uninstrumented (CUDA-graph decode) and
``instrument=True`` adds one extra pass with the engine's device phase profiler
(CUDA events per phase group, eager steps); its shares fill ``phase_seconds``
/ ``phase_fractions`` under the reference's phase names.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

from .decoder import DecodeConfig, _decode_ids, _members, translate_batch
from .errors import ConfigError
from .model import ModelParams, QuantizedModel

PHASES = ("quantize-activations", "matmul", "transcendental", "embedding", "search-overhead", "other")

class PhaseTimer:
    """Wall-clock accumulator per named phase (bench.py:27-57): phases nest and
    time goes to the innermost open phase.  One timer per thread."""

    def __init__(self):
        self.seconds: dict = {}
        self._stack: list = []

    def _charge(self, now):
        if self._stack:
            name, since = self._stack[-1]
            self.seconds[name] = self.seconds.get(name, 0.0) + (now - since)

    def push(self, name: str):
        now = time.perf_counter()
        self._charge(now)
        self._stack.append([name, now])

    def pop(self):
        now = time.perf_counter()
        self._charge(now)
        self._stack.pop()
        if self._stack:
            self._stack[-1][1] = now

    def merge(self, other: "PhaseTimer"):
        for name, sec in other.seconds.items():
            self.seconds[name] = self.seconds.get(name, 0.0) + sec

    def tracked_total(self) -> float:
        return sum(self.seconds.values())


@dataclass
class BenchReport:
    """Result of one benchmark run in one precision mode (bench.py:60-92)."""

    precision: str
    sentences: int
    total_words: int
    workers: int
    repeats: int
    run_seconds: list
    median_seconds: float
    wps: float
    wpcs: float
    phase_seconds: dict = field(default_factory=dict)
    phase_fractions: dict = field(default_factory=dict)  # percent of busy time

    def to_dict(self) -> dict:
        return {"precision": self.precision, "sentences": self.sentences, "total_words": self.total_words,
                "workers": self.workers, "repeats": self.repeats, "run_seconds": list(self.run_seconds),
                "median_seconds": self.median_seconds, "wps": self.wps, "wpcs": self.wpcs,
                "phase_seconds": dict(self.phase_seconds), "phase_fractions": dict(self.phase_fractions)}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2, sort_keys=True)


def _normalize_corpus(sentences) -> list:
    return [s.split() if isinstance(s, str) else list(s) for s in sentences]


def _prepare_model(model, precision: str):
    """bench.py:99-104: int8 quantizes float parameters (on the device); fp32
    needs float parameters."""
    if precision == "fp32" and isinstance(model, QuantizedModel):
        raise ConfigError("fp32 benchmark requires float parameters")
    return model


def _device_phases(model, corpus, cfg: DecodeConfig, batch: int) -> dict:
    """One decode pass with the engine phase profiler on: {reference phase: seconds}."""
    members = _members(model, cfg.precision)
    if len(members) != 1:
        return {}
    m = members[0]
    ids = [[m.src_ids(s) for s in corpus]]
    out: dict = {}
    _decode_ids(members, ids, cfg, batch, sort=True, phases=out)
    return out


def run_benchmark(model, sentences, cfg: DecodeConfig, workers: int = 1, repeats: int = 9,
                  instrument: bool = True, batch: int = 256) -> BenchReport:
    """Translate the corpus ``repeats`` times and report median-run speed
    (bench.py:135-191).  Model preparation (device upload, quantization, engine
    and CUDA-graph creation) happens in the untimed warm-up pass."""
    if repeats < 1 or repeats % 2 == 0:
        raise ConfigError(f"repeats must be odd and >= 1, got {repeats}")
    if workers < 1:
        raise ConfigError(f"workers must be >= 1, got {workers}")
    corpus = _normalize_corpus(sentences)
    prepared = _prepare_model(model, cfg.precision)
    outputs = translate_batch(prepared, corpus, cfg, max_batch=batch) if corpus else []   # warm-up
    run_seconds = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        outputs = translate_batch(prepared, corpus, cfg, max_batch=batch) if corpus else []
        run_seconds.append(time.perf_counter() - t0)
    total_words = sum(len(toks) for toks, _ in outputs)
    median = sorted(run_seconds)[len(run_seconds) // 2]
    wps = total_words / median if median > 0 else 0.0
    phase_seconds: dict = {}
    phase_fractions: dict = {}
    if instrument and corpus:
        t0 = time.perf_counter()
        phase_seconds = _device_phases(prepared, corpus, cfg, batch)
        wall = time.perf_counter() - t0
        phase_seconds["other"] = phase_seconds.get("other", 0.0) + max(0.0, wall - sum(phase_seconds.values()))
        if wall > 0:
            phase_fractions = {k: 100.0 * v / wall for k, v in phase_seconds.items()}
    return BenchReport(precision=cfg.precision, sentences=len(corpus), total_words=total_words, workers=1,
                       repeats=repeats, run_seconds=run_seconds, median_seconds=median, wps=wps, wpcs=wps,
                       phase_seconds=phase_seconds, phase_fractions=phase_fractions)


def profile_phases(model, sentences, cfg: DecodeConfig) -> list:
    """One profiled pass over the corpus; ``[(phase, percent of wall)]`` by
    descending share (bench.py:194-215).  Empty input yields an empty table."""
    corpus = _normalize_corpus(sentences)
    if not corpus:
        return []
    prepared = _prepare_model(model, cfg.precision)
    translate_batch(prepared, corpus, cfg)   # warm-up
    t0 = time.perf_counter()
    sec = _device_phases(prepared, corpus, cfg, 256)
    wall = time.perf_counter() - t0
    if wall <= 0:
        return []
    sec["other"] = sec.get("other", 0.0) + max(0.0, wall - sum(sec.values()))
    return sorted(((k, 100.0 * v / wall) for k, v in sec.items()), key=lambda kv: -kv[1])


__all__ = ["PHASES", "PhaseTimer", "BenchReport", "run_benchmark", "profile_phases", "ModelParams"]
