"""fp32 precision path: LinearOp's float branch
(layers.py:138-145), gemm_f32 (qmath.py:434-440), fp32 translate and
compare_precisions (decoder.py:216-248).  Goldens: the REFERENCE run with
precision="fp32" (tests/golden/make_golden.py gen_fp32); Tier B evaluates
gemm_f32 in fp64 and rounds once, like the other four elementwise functions."""

import json
import os

import numpy as np
import pytest

from oracle import qnmt_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F32, F64 = np.float32, np.float64


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "fp32_small.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def ops():
    return np.load(os.path.join(GOLDEN, "fp32_ops.npz"))


def _oracle(spec, tier="B"):
    d = O.Dims(**spec["dims"])
    t = O.synthetic_tensors(d, spec["seed"], spec["weight_std"], spec["bias_std"], spec["eos_bias"])
    return O.QModel(d, t, s0_mode=spec["s0_mode"], attention_query=spec["attention_query"], tier=tier,
                    precision="fp32")


def _params(spec):
    import paper_1804_05038_b200 as pb
    return pb.synthetic_model(pb.Dims(**spec["dims"]), spec["seed"], spec["weight_std"], spec["bias_std"],
                              spec["eos_bias"], spec["s0_mode"], spec["attention_query"])


def test_oracle_fp32_translations_match_reference(gold):
    models = {k: _oracle(v) for k, v in gold["models"].items()}
    for c in gold["cases"]:
        toks, lp = models[c["model"]].translate(c["src"], c["beam"], c["max_ratio"])
        assert toks == c["out_B"] and lp == c["logp_B"], c


def test_oracle_fp32_ops_match_reference(gold, ops):
    for tag, spec in gold["models"].items():
        om = _oracle(spec)
        states, att, s0 = om.encode(ops[f"{tag}_src"])
        assert np.array_equal(states, ops[f"{tag}_states"]), tag
        assert np.array_equal(att, ops[f"{tag}_att_proj"]), tag
        assert np.array_equal(s0, ops[f"{tag}_s0"]), tag
        s = np.repeat(s0, 3, axis=1)
        lp, s_new, s_int, alpha = om.decoder_step(ops[f"{tag}_y"], s, s.copy(), (states, att, s0))
        assert np.array_equal(lp, ops[f"{tag}_lp"]), tag
        assert np.array_equal(s_new, ops[f"{tag}_s_new"]) and np.array_equal(s_int, ops[f"{tag}_s_int"]), tag
        assert np.array_equal(alpha, ops[f"{tag}_alpha"]), tag
        assert np.array_equal(om.linear("dec_r.wz", ops[f"{tag}_x"], "dec_r.bz"), ops[f"{tag}_lin_wz"]), tag


def test_tier_a_fp32_close(gold):
    """Unpatched reference (numpy/OpenBLAS f32): the Tier-B oracle's fp32 decodes agree
    except at near-ties; log-probs within the north-star 1e-4 where tokens agree."""
    models = {k: _oracle(v) for k, v in gold["models"].items()}
    same = 0
    for c in gold["cases"]:
        if c["out_A"] == c["out_B"]:
            same += 1
            assert abs(c["logp_A"] - c["logp_B"]) <= 1e-4 * max(1.0, abs(c["logp_B"]))
    assert same >= 0.9 * len(gold["cases"])


def test_bleu_and_edit_distance_known_answers(gold):
    import paper_1804_05038_b200 as pb
    for c in gold["bleu"]:
        h = [" ".join(x) for x in c["hyps"]]
        r = [" ".join(x) for x in c["refs"]]
        if isinstance(c["bleu"], str):
            with pytest.raises(Exception) as ei:
                pb.bleu(h, r)
            assert type(ei.value).__name__ == c["bleu"]
        else:
            assert pb.bleu(h, r) == c["bleu"]
    for c in gold["edit"]:
        assert pb.edit_distance(c["a"], c["b"]) == c["d"]


def test_fp32_config_errors():
    import paper_1804_05038_b200 as pb
    from paper_1804_05038_b200 import errors
    p = pb.synthetic_model(pb.Dims(20, 17, 8, 8, 8, 8), 1)
    with pytest.raises(errors.ConfigError):   # decoder.py:64-66: a quantized model cannot decode fp32
        pb.translate(pb.QuantizedModel(p.dims, {}, {}, p.src_tokens, p.tgt_tokens), ["w0001"],
                     pb.DecodeConfig(2, 1.5, "fp32"))
    with pytest.raises(errors.ConfigError):
        pb.DecodeConfig(2, 1.5, "fp16")
    with pytest.raises(errors.EmptyInputError):
        pb.compare_precisions(p, [], pb.DecodeConfig(2, 1.5))


@pytest.mark.gpu
def test_gpu_gemm_f32_exact():
    import paper_1804_05038_b200 as pb
    rng = np.random.default_rng(3)
    for M, K, N in [(1, 1, 1), (7, 5, 3), (64, 33, 8), (130, 70, 9), (257, 512, 65), (3072, 1024, 64), (50, 3, 200)]:
        a = rng.normal(0, 0.05, (M, K)).astype(F32)
        b = rng.normal(0, 1, (K, N)).astype(F32)
        got = pb.gemm_f32(a, b)
        want = (a.astype(F64) @ b.astype(F64)).astype(F32)
        assert np.array_equal(got, want), (M, K, N)


@pytest.mark.gpu
def test_gpu_fp32_translations_match_reference(gold):
    import paper_1804_05038_b200 as pb
    params = {k: _params(v) for k, v in gold["models"].items()}
    for c in gold["cases"]:
        got = pb.translate_batch(params[c["model"]], [c["src"]], pb.DecodeConfig(c["beam"], c["max_ratio"], "fp32"),
                                 return_ids=True)[0]
        assert got[0] == c["out_B"] and got[1] == c["logp_B"], c


@pytest.mark.gpu
def test_gpu_fp32_ops_match_reference(gold, ops):
    import paper_1804_05038_b200 as pb
    for tag, spec in gold["models"].items():
        net = pb.build_network(_params(spec))
        assert net.precision == "fp32"
        enc = net.encode(ops[f"{tag}_src"])
        assert np.array_equal(enc.states, ops[f"{tag}_states"]), tag
        assert np.array_equal(enc.att_proj, ops[f"{tag}_att_proj"]), tag
        assert np.array_equal(enc.s0, ops[f"{tag}_s0"]), tag
        lp, st, alpha = net.decoder_step(ops[f"{tag}_y"], net.initial_state(enc, 3), enc)
        assert np.array_equal(lp, ops[f"{tag}_lp"]), tag
        assert np.array_equal(st.s, ops[f"{tag}_s_new"]) and np.array_equal(st.s_prime, ops[f"{tag}_s_int"]), tag
        assert np.array_equal(alpha, ops[f"{tag}_alpha"]), tag
        assert np.array_equal(net.dec_r.update_in.apply(ops[f"{tag}_x"]), ops[f"{tag}_lin_wz"]), tag
        # per-op composition (gru_step / attend / OutputNet.logits) equals the oracle's
        om = _oracle(spec)
        x = ops[f"{tag}_x"][:, :2]
        h = np.asarray(ops[f"{tag}_s_new"][:, :2])
        assert np.array_equal(pb.gru_step(net.dec_r, x, h), om.gru_step("dec_r", x, h)), tag
        ctx, al = pb.attend(net.attention, h, enc)
        octx, oal = om.attend(h, enc.states, enc.att_proj)
        assert np.array_equal(ctx, octx) and np.array_equal(al, oal), tag


@pytest.mark.gpu
def test_gpu_compare_precisions_matches_reference(gold):
    import paper_1804_05038_b200 as pb
    for tag, ref in gold["parity"].items():
        rep = pb.compare_precisions(_params(gold["models"][tag]), ref["corpus"], pb.DecodeConfig(3, 1.5))
        assert rep.to_dict() == ref["report"], tag
        assert rep.fp32_outputs == ref["fp32"] and rep.int8_outputs == ref["int8"], tag


@pytest.mark.gpu
def test_gpu_fp32_batch_and_ensemble_equal_oracle():
    """Batched fp32 decode (tiled f64 GEMM path, N > 8) and an fp32 ensemble."""
    import paper_1804_05038_b200 as pb
    d = pb.Dims(300, 251, 32, 48, 40, 32)
    ps = [pb.synthetic_model(d, s, 0.3, 0.1, 0.6) for s in (41, 42)]
    oms = [O.QModel(O.Dims(**d.as_dict()), p.tensors, precision="fp32") for p in ps]
    rng = np.random.default_rng(11)
    srcs = [rng.integers(3, 300, int(rng.integers(1, 16))).tolist() for _ in range(20)]
    cfg = pb.DecodeConfig(beam=4, max_ratio=1.5, precision="fp32")
    got = pb.translate_batch(ps[0], srcs, cfg, max_batch=16, return_ids=True)
    for s, g in zip(srcs, got):
        want = oms[0].translate(s, 4, 1.5)
        assert g[0] == want[0] and g[1] == want[1], s
    got = pb.translate_batch(ps, srcs[:6], cfg, return_ids=True)
    for s, g in zip(srcs[:6], got):
        want = O.translate_ensemble(oms, [s, s], 4, 1.5)
        assert g[0] == want[0] and g[1] == want[1], s
