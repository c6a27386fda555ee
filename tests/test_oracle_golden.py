"""Pin the CPU oracle against goldens produced by running the reference
itself (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import qnmt_oracle as O
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

F32 = np.float32


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def kat():
    return np.load(os.path.join(GOLDEN, "qmath_kat.npz"))


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLDEN, "small_model.npz"))


def test_quantize_known_answers(kat):
    names = sorted({k[2:-3] for k in kat.files if k.startswith("q_") and k.endswith("_in")})
    assert "halfulp" in names and "ties" in names
    for n in names:
        codes, scale = O.quantize(kat[f"q_{n}_in"])
        assert np.array_equal(codes, kat[f"q_{n}_codes"]), n
        assert scale == float(kat[f"q_{n}_scale"]), n
    # restated from pkg/tests/test_qmath.py:48-75 and SURVEY 8(c)
    assert O.quantize(np.array([[2, 1, -1]], F32))[0].tolist() == [[127, 64, -64]]
    assert O.quantize(np.array([[127, 0.49999997]], F32))[0].tolist() == [[127, 1]]
    c, s = O.quantize(np.array([[10.0]], F32))
    assert c[0, 0] == 127 and abs(s - 12.7) < 1e-5
    c, s = O.quantize(np.zeros((3, 3), F32))
    assert s == 1.0 and not c.any()


def test_quantize_errors():
    with pytest.raises(O.OracleError) as e:
        O.quantize(np.array([[1.0, np.nan]], F32))
    assert e.value.kind == "invalid-input"
    with pytest.raises(O.OracleError) as e:
        O.quantize_activations(np.array([[np.inf]], F32))
    assert e.value.kind == "numeric"


def test_qgemm_known_answers(kat):
    for i in range(int(kat["g_count"])):
        y = O.qgemm(kat[f"g{i}_a"], float(kat[f"g{i}_sa"]), kat[f"g{i}_b"], float(kat[f"g{i}_sb"]))
        assert np.array_equal(y, kat[f"g{i}_y"]), i


def test_cfg1_hashes(kat):
    w = np.random.default_rng(1804).normal(0, 0.05, (3072, 1024)).astype(F32)
    wc, ws = O.quantize(w)
    assert ws == float(kat["cfg1_w_scale"])
    assert sha(wc) == str(kat["cfg1_w_codes_sha"])
    for b in (1, 64):
        x = np.random.default_rng(5038 + b).normal(0, 1, (1024, b)).astype(F32)
        xc, xs = O.quantize_activations(x)
        assert xs == float(kat[f"cfg1_b{b}_x_scale"])
        assert sha(xc) == str(kat[f"cfg1_b{b}_x_codes_sha"])
        acc = O.int_product(wc, xc)
        assert sha(acc.astype(np.int32)) == str(kat[f"cfg1_b{b}_acc_sha"])
        y = O.scale_output(acc, ws, xs)
        assert sha(y) == str(kat[f"cfg1_b{b}_y_sha"])


def _specs():
    with open(os.path.join(GOLDEN, "translate_small.json")) as fh:
        return json.load(fh)


def _model(spec, tier):
    d = O.Dims(**spec["dims"])
    t = O.synthetic_tensors(d, spec["seed"], spec["weight_std"], spec["bias_std"],
                            spec["eos_bias"])
    return O.QModel(d, t, s0_mode=spec["s0_mode"], attention_query=spec["attention_query"],
                    tier=tier)


@pytest.mark.parametrize("tag", ["small", "med", "eos", "eosmed", "flags"])
@pytest.mark.parametrize("tier", ["A", "B"])
def test_op_level(small, tag, tier):
    m = _model(_specs()["models"][tag], tier)
    p = f"{tag}{tier}"
    g = small
    states, att_proj, s0 = m.encode(g[f"{p}_src"])
    exact = tier == "B"

    def check(a, b, what):
        if exact:
            assert np.array_equal(a, b), what
        else:
            den = max(float(np.max(np.abs(b))), 1e-30)
            assert float(np.max(np.abs(a - b))) / den <= 1e-4, what

    check(states, g[f"{p}_states"], "states")
    check(att_proj, g[f"{p}_att_proj"], "att_proj")
    check(s0, g[f"{p}_s0"], "s0")
    lp, snew, sint, alpha = m.decoder_step(g[f"{p}_step_y"], g[f"{p}_step_s"],
                                           g[f"{p}_step_sp"], (states, att_proj, s0))
    check(lp, g[f"{p}_step_lp"], "lp")
    check(snew, g[f"{p}_step_snew"], "snew")
    check(sint, g[f"{p}_step_sint"], "sint")
    check(alpha, g[f"{p}_step_alpha"], "alpha")
    check(m.gru_step("dec_r", g[f"{p}_gru_x"], g[f"{p}_gru_h"]), g[f"{p}_gru_out"], "gru")
    ctx, al = m.attend(g[f"{p}_gru_h"], states, att_proj)
    check(ctx, g[f"{p}_att_ctx"], "ctx")
    check(al, g[f"{p}_att_alpha"], "alpha2")
    check(m.linear("dec_r.wz", g[f"{p}_gru_x"], "dec_r.bz"), g[f"{p}_lin_out"], "lin")


def test_translate_tier_b_exact():
    tr = _specs()
    models = {}
    for c in tr["cases"]:
        key = c["model"]
        if key not in models:
            models[key] = _model(tr["models"][key], "B")
        toks, logp = models[key].translate(c["src"], c["beam"], c["max_ratio"])
        assert toks == c["out_B"], c
        assert logp == c["logp_B"], c
    # some cases must exercise EOS and early termination
    early = sum(len(c["out_B"]) < int(np.ceil(c["max_ratio"] * len(c["src"]))) + 1
                for c in tr["cases"])
    assert early >= 10, early


@pytest.mark.slow
def test_baseline_dims_tier_b():
    g = np.load(os.path.join(GOLDEN, "baseline_dims.npz"))
    d = O.Dims(32000, 32000, 512, 1024, 2048, 512)
    m = O.QModel(d, O.synthetic_tensors(d, 1804), tier="B")
    names = [str(n) for n in g["w_scale_names"]]
    for n, s in zip(names, g["w_scales"]):
        assert m.q[n][1] == float(s), n
    states, att_proj, s0 = m.encode(g["src50"])
    assert sha(states) == str(g["B_states_sha"])
    assert sha(att_proj) == str(g["B_att_proj_sha"])
    assert np.array_equal(s0, g["B_s0"])
    toks, logp = m.translate(g["src50"].tolist(), beam=1, max_ratio=0.98)
    assert toks == g["B_greedy50"].tolist()
    assert logp == float(g["B_greedy50_logp"])
