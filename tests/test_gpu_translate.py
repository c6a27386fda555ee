"""End-to-end parity of the device-resident greedy / beam search against the
reference goldens (Tier B): identical token ids and identical f64 log-probs."""

import math

import numpy as np
import pytest

from oracle import qnmt_oracle as O
from qnmt_test_helpers import F32, golden, model_pair, sha, translate_specs

pytestmark = pytest.mark.gpu
pb = pytest.importorskip("paper_1804_05038_b200")

_q = {}


def qmodel(spec, tag):
    if tag not in _q:
        params, om = model_pair(spec)
        _q[tag] = (pb.quantize_model(params), om, params)
    return _q[tag]


def test_translate_golden_cases():
    tr = translate_specs()
    for c in tr["cases"]:
        qm, _, params = qmodel(tr["models"][c["model"]], c["model"])
        toks = [params.src_tokens[i] for i in c["src"]]
        cfg = pb.DecodeConfig(beam=c["beam"], max_ratio=c["max_ratio"], precision="int8")
        words, logp = pb.translate(qm, toks, cfg)
        idx = {t: i for i, t in enumerate(params.tgt_tokens)}
        assert [idx[w] for w in words] == c["out_B"], c
        assert logp == c["logp_B"], c


@pytest.mark.parametrize("tag", ["small", "med", "eos", "eosmed", "flags"])
@pytest.mark.parametrize("beam", [1, 3, 5])
def test_batch_equals_sentence_by_sentence(tag, beam):
    """translate_batch (one engine call, segmented scales) == oracle per sentence."""
    tr = translate_specs()
    qm, om, params = qmodel(tr["models"][tag], tag)
    rng = np.random.default_rng(beam * 31 + len(tag))
    sents = [rng.integers(3, params.dims.src_vocab, int(rng.integers(1, 14))).tolist() for _ in range(23)]
    cfg = pb.DecodeConfig(beam=beam, max_ratio=1.5)
    got = pb.translate_batch(qm, sents, cfg, max_batch=16, return_ids=True)
    for s, (toks, lp) in zip(sents, got):
        et, elp = om.translate(s, beam, 1.5)
        assert toks == et and lp == elp, (s, toks, et)


def test_errors():
    tr = translate_specs()
    qm, _, params = qmodel(tr["models"]["small"], "small")
    with pytest.raises(pb.errors.EmptyInputError):
        pb.translate(qm, [], pb.DecodeConfig())
    with pytest.raises(pb.errors.ConfigError):
        pb.translate(qm, ["w0001"], pb.DecodeConfig(precision="fp32"))
    # unknown source tokens map to UNK (model.py:110-115) and decode fine
    words, lp = pb.translate(qm, ["nope", "w0003"], pb.DecodeConfig(beam=2))
    assert isinstance(words, list) and math.isfinite(lp)


@pytest.fixture(scope="module")
def base():
    d = pb.Dims(32000, 32000, 512, 1024, 2048, 512)
    params = pb.synthetic_model(d, 1804)
    return params, pb.quantize_model(params), golden("baseline_dims.npz")


def test_baseline_weight_scales(base):
    params, qm, g = base
    for n, s in zip([str(x) for x in g["w_scale_names"]], g["w_scales"]):
        assert qm.q[n].scale == float(s), n


def test_cfg2_encoder_bit_exact(base):
    """BASELINE cfg2: l = 50 encoder states [50 x 2048] bit-exact."""
    params, qm, g = base
    net = pb.build_network(qm)
    enc = net.encode(g["src50"])
    assert sha(enc.states) == str(g["B_states_sha"])
    assert sha(enc.att_proj) == str(g["B_att_proj_sha"])
    assert np.array_equal(enc.s0, g["B_s0"])


def test_cfg3_greedy_bit_exact(base):
    """BASELINE cfg3: encoder + 50 greedy steps, V = 32000 (latency path)."""
    params, qm, g = base
    toks = [params.src_tokens[i] for i in g["src50"]]
    words, logp = pb.translate(qm, toks, pb.DecodeConfig(beam=1, max_ratio=0.98))
    idx = {t: i for i, t in enumerate(params.tgt_tokens)}
    assert [idx[w] for w in words] == g["B_greedy50"].tolist()
    assert logp == float(g["B_greedy50_logp"])
    net = pb.build_network(qm)
    enc = net.encode(g["src50"])
    lp, st, alpha = net.decoder_step(np.array([2]), net.initial_state(enc, 1), enc)
    assert sha(lp) == str(g["B_step1_lp_sha"])
    assert np.array_equal(alpha, g["B_step1_alpha"])


def test_beam5_baseline_dims(base):
    params, qm, g = base
    toks = [params.src_tokens[i] for i in g["B_beam5_src"]]
    words, logp = pb.translate(qm, toks, pb.DecodeConfig(beam=5, max_ratio=1.5))
    idx = {t: i for i, t in enumerate(params.tgt_tokens)}
    assert [idx[w] for w in words] == g["B_beam5"].tolist()
    assert logp == float(g["B_beam5_logp"])
