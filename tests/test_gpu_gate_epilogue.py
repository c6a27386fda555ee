"""GRU gate nonlinearities in the tcgen05 GEMM epilogues (gemm_tcgen05.cu
EPI_GATES / EPI_COMBINE, engine.cu gru_cell; layers.py:170-181).

Batched decode steps with more than 8 columns compute z = sigmoid(W_z x + U_z h)
and r * h on the accumulators of the cell's input GEMM and h' = (1 - z) h +
z tanh(W_c x + U_c (r * h)) on those of the candidate GEMM, with the
per-sentence max |.| for the next quantization reduced there too.  The
results must equal the oracle's (Tier B) and those of the separate fused
elementwise + quantize kernels (qnmt_set_gate_epi(0)) bit for bit: tokens
and f64 log-probs of whole decodes, on hidden sizes that are / are not a
multiple of the 128-row tile, with both attention-query / s0 flag settings,
early-EOS models, and every tile width of the two epilogue GEMMs."""

import numpy as np
import pytest

from oracle import qnmt_oracle as O

pytestmark = pytest.mark.gpu
pb = pytest.importorskip("paper_1804_05038_b200")
from paper_1804_05038_b200 import _lib  # noqa: E402

# (dims, s0_mode, attention_query, eos_bias)
MODELS = {
    "h64": (dict(src_vocab=90, tgt_vocab=83, embed=32, hidden=64, attn=48, readout=32), "transform", "current", 0.0),
    "h160": (dict(src_vocab=120, tgt_vocab=131, embed=48, hidden=160, attn=64, readout=48), "transform", "current",
             0.0),
    "h128flags": (dict(src_vocab=70, tgt_vocab=67, embed=16, hidden=128, attn=32, readout=16), "zero", "previous",
                  0.0),
    "h96eos": (dict(src_vocab=90, tgt_vocab=83, embed=32, hidden=96, attn=48, readout=32), "transform", "current",
               1.5),
}
_cache = {}


def _model(tag):
    if tag not in _cache:
        dims, s0, aq, eos = MODELS[tag]
        params = pb.synthetic_model(pb.Dims(**dims), 4242 + len(tag), 0.3, 0.1, eos, s0, aq)
        om = O.QModel(O.Dims(**dims), params.tensors, s0_mode=s0, attention_query=aq, tier="B")
        _cache[tag] = (params, pb.quantize_model(params), om)
    return _cache[tag]


def _decode(qm, sents, beam, gate, bn=(0, 0)):
    lib = _lib.load()
    old = lib.qnmt_set_gate_epi(gate)
    old_bn = lib.qnmt_set_gru_epi_bn(bn[0], bn[1])
    try:
        cfg = pb.DecodeConfig(beam=beam, max_ratio=1.5, precision="int8")
        return pb.translate_batch(qm, sents, cfg, max_batch=16, return_ids=True)
    finally:
        lib.qnmt_set_gate_epi(old)
        lib.qnmt_set_gru_epi_bn(0, 0)
        assert old_bn in (0, bn[0])


@pytest.mark.parametrize("tag", sorted(MODELS))
@pytest.mark.parametrize("beam", [1, 3, 5])
def test_gate_epilogue_equals_oracle_and_fused_kernels(tag, beam):
    params, qm, om = _model(tag)
    rng = np.random.default_rng(beam * 17 + len(tag))
    sents = [rng.integers(3, params.dims.src_vocab, int(rng.integers(1, 16))).tolist() for _ in range(21)]
    on = _decode(qm, sents, beam, 1)
    off = _decode(qm, sents, beam, 0)
    assert on == off
    for s, (toks, lp) in zip(sents, on):
        et, elp = om.translate(s, beam, 1.5)
        assert toks == et and lp == elp, (tag, beam, s, toks, et)


@pytest.mark.parametrize("bn", [(64, 64), (96, 128), (128, 96), (160, 192), (192, 224), (224, 160), (256, 256)])
def test_gate_epilogue_tile_widths(bn):
    params, qm, om = _model("h160")
    rng = np.random.default_rng(bn[0])
    sents = [rng.integers(3, params.dims.src_vocab, int(rng.integers(2, 12))).tolist() for _ in range(40)]
    ref = _decode(qm, sents, 5, 0)
    assert _decode(qm, sents, 5, 1, bn) == ref


@pytest.mark.parametrize("key", ["dec_r.bz", "dec_r.br", "dec_q.bc"])
def test_gate_epilogue_flags_non_finite(key):
    """A non-finite pre-activation raises NumericError from the epilogue as from k_gates_q / k_combine_q."""
    bad = pb.synthetic_model(pb.Dims(**MODELS["h64"][0]), 4245, 0.3, 0.1, 0.0, "transform", "current")
    t = bad.tensors[key].copy()
    t.flat[3] = np.inf   # W x + b is +inf in that row
    bad.tensors[key] = t
    qb = pb.quantize_model(bad)
    sents = [[5, 6, 7]] * 12
    for gate in (0, 1):
        with pytest.raises(pb.errors.NumericError):
            _decode(qb, sents, 3, gate)
