"""Checked engines (QNMT_CANARY=1): every device buffer of the engine is followed
by a 256-byte guard band of 0xA5; after decodes of many shapes the guard bands
must be intact (no kernel wrote past a buffer into its neighbour).  This is the
write-side memcheck the GPU pool allows (compute-sanitizer is refused there).
Outputs must also equal those of an unchecked engine."""

import os

import numpy as np
import pytest
import torch

from qnmt_test_helpers import model_pair, translate_specs

pytestmark = pytest.mark.gpu
pb = pytest.importorskip("paper_1804_05038_b200")
from paper_1804_05038_b200 import _lib  # noqa: E402


def _checked_engine(qm, S, L, B):
    old = os.environ.get("QNMT_CANARY")
    os.environ["QNMT_CANARY"] = "1"
    try:
        return pb.Engine(qm, S, L, B)
    finally:
        if old is None:
            del os.environ["QNMT_CANARY"]
        else:
            os.environ["QNMT_CANARY"] = old


def _canaries(e):
    return int(_lib.load().qnmt_engine_check_canaries(e._h, torch.cuda.current_stream().cuda_stream))


@pytest.mark.parametrize("tag", ["small", "med", "eos", "eosmed", "flags"])
def test_guard_bands_intact_small_models(tag):
    tr = translate_specs()
    params, _ = model_pair(tr["models"][tag])
    qm = pb.quantize_model(params)
    e = _checked_engine(qm, 24, 20, 16)
    ref = pb.Engine(qm, 24, 20, 16)
    assert _canaries(e) == 0 and _canaries(ref) == -1
    rng = np.random.default_rng(len(tag))
    for beam in (1, 2, 5, 16):
        for n in (1, 7, 24):
            sents = [rng.integers(3, params.dims.src_vocab, int(rng.integers(1, 21))).tolist() for _ in range(n)]
            got = e.translate_ids(sents, beam, 1.5)
            assert _canaries(e) == 0, (beam, n)
            assert got == ref.translate_ids(sents, beam, 1.5)


def test_guard_bands_intact_baseline_dims():
    """BASELINE cfg5 dims (V = 50000, H = 1024, A = 2048): batched beam-5 decode
    with graph-captured steps, the persistent greedy path, the op-level encoder
    and decoder step."""
    d = pb.Dims(32000, 50000, 512, 1024, 2048, 512)
    params = pb.synthetic_model(d, 1804)
    qm = pb.quantize_model(params)
    e = _checked_engine(qm, 64, 100, 5)
    rng = np.random.default_rng(5)
    sents = [rng.integers(3, 32000, int(rng.integers(5, 101))).tolist() for _ in range(64)]
    e.translate_ids(sents, 5, 1.5)
    assert _canaries(e) == 0
    e.translate_ids(sents[:3], 5, 1.5)
    assert _canaries(e) == 0
    e.translate_ids([sents[0]], 1, 1.5)          # persistent batch-1 greedy kernel
    assert _canaries(e) == 0
    states, att, s0, rows, lens = e.encode_batch([sents[1], sents[2]])
    assert _canaries(e) == 0
    assert states.shape[0] == len(sents[1]) + len(sents[2])
