"""Ensemble decoding (decoder.py:88-160 with several models,
log-probs averaged per step at :115-120).  Goldens: the REFERENCE's translate()
over lists of models (tests/golden/make_golden.py gen_ensemble), Tier A and B."""

import json
import os

import numpy as np
import pytest

from oracle import qnmt_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "ensemble_small.json")) as fh:
        return json.load(fh)


def _oracle_members(spec_list, tier="B"):
    out = []
    for sp in spec_list:
        d = O.Dims(**sp["dims"])
        t = O.synthetic_tensors(d, sp["seed"], sp["weight_std"], sp["bias_std"], sp["eos_bias"])
        out.append(O.QModel(d, t, s0_mode=sp["s0_mode"], attention_query=sp["attention_query"], tier=tier))
    return out


def _ids(tokens, src_vocab):
    """synthetic vocab: 'w%04d' -> id k+2; unknown -> UNK (model.py:110-115)."""
    out = []
    for t in tokens:
        k = int(t[1:]) + 2
        out.append(k if k < src_vocab else 1)
    return out


def test_oracle_ensembles_match_reference(gold):
    members = {tag: _oracle_members(specs) for tag, specs in gold["ensembles"].items()}
    for c in gold["cases"]:
        ms = members[c["ensemble"]]
        srcs = [_ids(c["src_tokens"], m.dims.src_vocab) for m in ms]
        toks, lp = O.translate_ensemble(ms, srcs, c["beam"], c["max_ratio"])
        assert toks == c["out_B"], c
        assert lp == c["logp_B"], c


def test_ensemble_api_errors():
    import paper_1804_05038_b200 as pb
    from paper_1804_05038_b200 import errors
    a = pb.synthetic_model(pb.Dims(20, 17, 8, 8, 8, 8), 1)
    b = pb.synthetic_model(pb.Dims(20, 18, 8, 8, 8, 8), 2)
    with pytest.raises(errors.ConfigError):
        pb.translate([a, b], ["w0001"], pb.DecodeConfig(2, 1.5))   # different target vocabularies
    with pytest.raises(errors.ConfigError):
        pb.translate([], ["w0001"], pb.DecodeConfig(2, 1.5))


@pytest.mark.gpu
def test_gpu_ensembles_match_reference(gold):
    import paper_1804_05038_b200 as pb
    models = {}
    for tag, specs in gold["ensembles"].items():
        ms = []
        cache = {}
        for sp in specs:
            key = (sp["tag"])
            if key not in cache:   # "ensdup" lists one model object twice
                p = pb.synthetic_model(pb.Dims(**sp["dims"]), sp["seed"], sp["weight_std"], sp["bias_std"],
                                       sp["eos_bias"], sp["s0_mode"], sp["attention_query"])
                cache[key] = pb.quantize_model(p)
            ms.append(cache[key])
        models[tag] = ms
    for c in gold["cases"]:
        words, lp = pb.translate(models[c["ensemble"]], c["src_tokens"], pb.DecodeConfig(c["beam"], c["max_ratio"], "int8"))
        ids = [int(w[1:]) + 2 if w.startswith("w") else {"<pad>": 0, "<unk>": 1, "</s>": 2}[w] for w in words]
        assert ids == c["out_B"], c
        assert lp == c["logp_B"], c


@pytest.mark.gpu
def test_gpu_ensemble_batch_equals_oracle():
    """Batched ensemble decode (many sentences per engine call) == the oracle's
    sentence-by-sentence ensemble, at a model size where the tcgen05 path runs."""
    import paper_1804_05038_b200 as pb
    d = pb.Dims(300, 251, 32, 48, 40, 32)
    specs = [(31, 0.3, 0.1, 0.6), (32, 0.3, 0.1, 0.6)]
    ps = [pb.synthetic_model(d, s, w, b, e) for s, w, b, e in specs]
    qms = [pb.quantize_model(p) for p in ps]
    oms = [O.QModel(O.Dims(**d.as_dict()), p.tensors) for p in ps]
    rng = np.random.default_rng(9)
    srcs = [rng.integers(3, 300, int(rng.integers(1, 20))).tolist() for _ in range(24)]
    got = pb.translate_batch(qms, srcs, pb.DecodeConfig(beam=4, max_ratio=1.5, precision="int8"), max_batch=16, return_ids=True)
    for s, g in zip(srcs, got):
        want = O.translate_ensemble(oms, [s, s], 4, 1.5)
        assert g[0] == want[0] and g[1] == want[1], s
