"""GPU parity of the layer ops and the engine's encode / decoder_step against
the Tier-B oracle (itself pinned bit-exactly to the patched reference).
Expected: bit-identical outputs."""

import numpy as np
import pytest
import torch

from qnmt_test_helpers import F32, golden, model_pair, translate_specs

pytestmark = pytest.mark.gpu
pb = pytest.importorskip("paper_1804_05038_b200")

MODELS = ["small", "med", "eos", "eosmed", "flags"]


@pytest.fixture(scope="module")
def specs():
    return translate_specs()["models"]


@pytest.fixture(scope="module")
def small():
    return golden("small_model.npz")


_cache = {}


def net_and_oracle(specs, tag):
    if tag not in _cache:
        params, om = model_pair(specs[tag])
        qm = pb.quantize_model(params)
        _cache[tag] = (pb.build_network(qm), om, qm, params)
    return _cache[tag]


@pytest.mark.parametrize("tag", MODELS)
def test_weights_quantized_like_reference(specs, tag):
    net, om, qm, _ = net_and_oracle(specs, tag)
    for name, (codes, scale) in om.q.items():
        assert qm.q[name].scale == scale, name
        assert np.array_equal(qm.q[name].device_data().cpu().numpy(), codes), name


@pytest.mark.parametrize("tag", MODELS)
def test_ops_vs_oracle(specs, small, tag):
    net, om, qm, _ = net_and_oracle(specs, tag)
    g = small
    p = f"{tag}B"
    x, h = g[f"{p}_gru_x"], g[f"{p}_gru_h"]
    # LinearOp (layers.py:118-146) -- exact vs the patched reference golden
    assert np.array_equal(net.dec_r.update_in.apply(x), g[f"{p}_lin_out"])
    # gru_step (layers.py:170-181)
    assert np.array_equal(pb.gru_step(net.dec_r, x, h), g[f"{p}_gru_out"])
    assert np.array_equal(pb.gru_step(net.dec_r, x, h), om.gru_step("dec_r", x, h))
    # encoder (layers.py:313-348)
    enc = net.encode(g[f"{p}_src"])
    assert np.array_equal(enc.states, g[f"{p}_states"])
    assert np.array_equal(enc.att_proj, g[f"{p}_att_proj"])
    assert np.array_equal(enc.s0, g[f"{p}_s0"])
    # attend (layers.py:214-241)
    ctx, alpha = pb.attend(net.attention, h, enc)
    assert np.array_equal(alpha, g[f"{p}_att_alpha"])
    assert np.array_equal(ctx, g[f"{p}_att_ctx"])
    # decoder_step teacher-forced (layers.py:356-384)
    st = pb.DecoderState(g[f"{p}_step_s"], g[f"{p}_step_sp"])
    lp, st2, al = net.decoder_step(g[f"{p}_step_y"], st, enc)
    assert np.array_equal(st2.s_prime, g[f"{p}_step_sint"])
    assert np.array_equal(st2.s, g[f"{p}_step_snew"])
    assert np.array_equal(al, g[f"{p}_step_alpha"])
    assert np.array_equal(lp, g[f"{p}_step_lp"])


@pytest.mark.parametrize("scale", [1e-7, 1e-4, 1e-2, 1.0, 40.0])
@pytest.mark.parametrize("P", [1, 5, 16])
def test_attention_magnitudes(specs, small, scale, P):
    """Attention over query / att_proj magnitudes that drive the per-hypothesis
    scale from ~1e9 (every code from the exact fp64 path) to saturation, and
    1..16 hypotheses per sentence: bit-identical to the oracle."""
    net, om, qm, _ = net_and_oracle(specs, "med")
    g = small
    enc = net.encode(g["medB_src"])
    rng = np.random.default_rng(int(P * 1000 + np.log10(scale) * 10 + 500))
    h = (rng.normal(0, 0.5, (om.dims.hidden, P)) * scale).astype(F32)
    att_proj = (enc.att_proj * F32(scale)).astype(F32)
    enc2 = pb.EncoderStates(enc.states, att_proj, enc.s0)
    ctx, alpha = pb.attend(net.attention, h, enc2)
    ctx_o, alpha_o = om.attend(h, enc.states, att_proj)
    assert np.array_equal(alpha, alpha_o)
    assert np.array_equal(ctx, ctx_o)


@pytest.mark.parametrize("tag", MODELS)
def test_output_net_per_op_path(specs, tag):
    """OutputNet.logits via the per-op path equals the oracle (layers.py:255-266)."""
    net, om, qm, _ = net_and_oracle(specs, tag)
    d = om.dims
    rng = np.random.default_rng(3)
    s = rng.normal(0, 0.5, (d.hidden, 4)).astype(F32)
    e = rng.normal(0, 0.05, (d.embed, 4)).astype(F32)
    c = rng.normal(0, 0.5, (2 * d.hidden, 4)).astype(F32)
    assert np.array_equal(net.output.logits(s, e, c), om.logits(s, e, c))


def test_tier_a_tolerance(specs, small):
    """Against the UNPATCHED reference (numpy f32 transcendentals) the
    teacher-forced step agrees within the north-star op-level bound."""
    net, om, qm, _ = net_and_oracle(specs, "med")
    g = small
    p = "medA"
    enc = net.encode(g[f"{p}_src"])
    st = pb.DecoderState(g[f"{p}_step_s"], g[f"{p}_step_sp"])
    lp, st2, al = net.decoder_step(g[f"{p}_step_y"], st, enc)
    ref = g[f"{p}_step_lp"]
    assert np.max(np.abs(lp - ref)) / np.max(np.abs(ref)) < 1e-4
    ref = g[f"{p}_gru_out"]
    out = pb.gru_step(net.dec_r, g[f"{p}_gru_x"], g[f"{p}_gru_h"])
    assert np.max(np.abs(out - ref)) / np.max(np.abs(ref)) < 1e-4


def test_torch_inputs_stay_on_device(specs, small):
    net, om, qm, _ = net_and_oracle(specs, "small")
    x = torch.from_numpy(small["smallB_gru_x"]).cuda()
    h = torch.from_numpy(small["smallB_gru_h"]).cuda()
    y = pb.gru_step(net.dec_r, x, h)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    assert np.array_equal(y.cpu().numpy(), small["smallB_gru_out"])


def test_errors(specs):
    net, om, qm, _ = net_and_oracle(specs, "small")
    with pytest.raises(pb.errors.ShapeError):
        net.dec_r.update_in.apply(np.zeros((3, 2), F32))
    with pytest.raises(pb.errors.EmptyInputError):
        net.encode([])
    with pytest.raises(pb.errors.VocabError):
        net.encode([1, 10_000])
    bad = np.zeros((om.dims.embed, 1), F32)
    bad[0, 0] = np.nan
    with pytest.raises(pb.errors.NumericError):
        net.dec_r.update_in.apply(bad)


@pytest.mark.parametrize("P", [17, 33, 40])
def test_attend_more_than_16_query_columns(specs, P):
    """attend on wider query blocks than one beam (the kernels take 16 columns per call; the
    state projection is quantized over the whole block as layers.py:221 does)."""
    net, om, qm, params = net_and_oracle(specs, "med")
    rng = np.random.default_rng(P)
    src = rng.integers(3, params.dims.src_vocab, 11).tolist()
    enc = net.encode(np.asarray(src))
    ost, oatt, os0 = om.encode(src)
    q = (rng.normal(0, 1, (params.dims.hidden, P)) * 0.7).astype(F32)
    ctx, alpha = pb.attend(net.attention, q, enc)
    octx, oalpha = om.attend(q, ost, oatt)
    assert np.array_equal(alpha, oalpha) and np.array_equal(ctx, octx)
