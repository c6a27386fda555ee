"""End-to-end parity of the device-resident greedy / beam search against the
reference goldens (Tier B): identical token ids and identical f64 log-probs."""

import math

import numpy as np
import torch
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
    cfg = pb.DecodeConfig(beam=beam, max_ratio=1.5, precision="int8")
    got = pb.translate_batch(qm, sents, cfg, max_batch=16, return_ids=True)
    for s, (toks, lp) in zip(sents, got):
        et, elp = om.translate(s, beam, 1.5)
        assert toks == et and lp == elp, (s, toks, et)


def test_errors():
    tr = translate_specs()
    qm, _, params = qmodel(tr["models"]["small"], "small")
    with pytest.raises(pb.errors.EmptyInputError):
        pb.translate(qm, [], pb.DecodeConfig(precision="int8"))
    with pytest.raises(pb.errors.ConfigError):
        pb.translate(qm, ["w0001"], pb.DecodeConfig(precision="fp32"))
    # unknown source tokens map to UNK (model.py:110-115) and decode fine
    words, lp = pb.translate(qm, ["nope", "w0003"], pb.DecodeConfig(beam=2, precision="int8"))
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
    words, logp = pb.translate(qm, toks, pb.DecodeConfig(beam=1, max_ratio=0.98, precision="int8"))
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
    words, logp = pb.translate(qm, toks, pb.DecodeConfig(beam=5, max_ratio=1.5, precision="int8"))
    idx = {t: i for i, t in enumerate(params.tgt_tokens)}
    assert [idx[w] for w in words] == g["B_beam5"].tolist()
    assert logp == float(g["B_beam5_logp"])


@pytest.mark.parametrize("beam", [1, 4])
def test_graph_mode_equals_eager_and_oracle(beam):
    """CUDA-graph decode (device-side live count) == eager per-step loop == oracle,
    on a 16-aligned model that terminates early (EOS) for some sentences."""
    from paper_1804_05038_b200 import _lib
    d = pb.Dims(300, 411, 64, 128, 96, 48)
    params = pb.synthetic_model(d, 21, weight_std=0.25, bias_std=0.1, eos_bias=0.6)
    qm = pb.quantize_model(params)
    om = O.QModel(O.Dims(**d.as_dict()), params.tensors)
    rng = np.random.default_rng(beam)
    sents = [rng.integers(3, 300, int(rng.integers(1, 40))).tolist() for _ in range(37)]
    eng = pb.Engine(qm, 64, 64, 8)
    lib = _lib.load()
    lib.qnmt_engine_set_graphs(eng._h, 1)
    g_out = eng.translate_ids(sents, beam, 2.0)
    g_out2 = eng.translate_ids(sents[:20], beam, 2.0)       # re-capture for a different batch size
    lib.qnmt_engine_set_graphs(eng._h, 0)
    e_out = eng.translate_ids(sents, beam, 2.0)
    assert g_out == e_out
    assert g_out2[0] == e_out[0][:20] and g_out2[1] == e_out[1][:20]
    early = 0
    for i, s in enumerate(sents):
        toks, lp = om.translate(s, beam, 2.0)
        assert g_out[0][i] == toks and g_out[1][i] == lp, i
        early += len(toks) < int(np.ceil(2.0 * len(s)))
    assert early > 0


@pytest.mark.parametrize("V,k,ties", [(50000, 5, False), (50000, 5, True), (37, 8, True), (7, 5, True),
                                      (32000, 1, True), (1000, 12, True), (2048, 16, False)])
def test_candidate_kernels_exact(V, k, ties):
    """Single-pass candidates == three-pass kernel == numpy restatement of
    decoder.py:125 + :74-85 per parent, including heavy logit ties."""
    import torch
    from paper_1804_05038_b200 import _lib, _dev
    rng = np.random.default_rng(V + k)
    N = 37
    x = rng.normal(0, 2, (N, V)).astype(np.float32)
    if ties:
        x = (np.round(x * 4) / 4).astype(np.float32)
    live = rng.normal(-20, 5, N)
    lib = _lib.load()

    def run(exact):
        old = lib.qnmt_set_topk_exact(exact)
        xs, lv = torch.from_numpy(x).cuda(), torch.from_numpy(live).cuda()
        cs = torch.empty((N, k), dtype=torch.float64, device="cuda")
        ct = torch.empty((N, k), dtype=torch.int32, device="cuda")
        f = _dev.reset_flag()
        _lib.call("qnmt_topk_candidates", xs.data_ptr(), N, V, V, lv.data_ptr(), k, cs.data_ptr(), ct.data_ptr(),
                  f.data_ptr(), _dev.stream_ptr())
        lib.qnmt_set_topk_exact(old)
        return cs.cpu().numpy(), ct.cpu().numpy()

    s1, t1 = run(0)
    s3, t3 = run(1)
    lp = O.log_softmax_cols(x.T).T          # [N, V] f32 (Tier B)
    for n in range(N):
        sc = live[n] + lp[n].astype(np.float64)
        order = sorted(range(V), key=lambda v: (-sc[v], v))[:k]
        assert t1[n].tolist() == order and t3[n].tolist() == order, n
        assert np.array_equal(s1[n], sc[order]) and np.array_equal(s3[n], sc[order])


def _fused_pair(eng, sents, beam, ratio):
    from paper_1804_05038_b200 import _lib
    lib = _lib.load()
    old = lib.qnmt_set_vocab_fused(1)
    try:
        fused = eng.translate_ids(sents, beam, ratio)
        lib.qnmt_set_vocab_fused(0)
        plain = eng.translate_ids(sents, beam, ratio)
    finally:
        lib.qnmt_set_vocab_fused(old)
    return fused, plain


@pytest.mark.parametrize("beam", [1, 5, 12])
def test_vocab_fused_equals_unfused_and_oracle(beam):
    """Fused vocab projection + softmax statistics + candidates (vocab_topk.cu)
    == vocab GEMM + candidate kernel == oracle, V not a multiple of the tile."""
    d = pb.Dims(200, 1333, 64, 64, 64, 48)
    params = pb.synthetic_model(d, 5, weight_std=0.3, bias_std=0.2, eos_bias=0.5)
    qm = pb.quantize_model(params)
    om = O.QModel(O.Dims(**d.as_dict()), params.tensors)
    rng = np.random.default_rng(beam + 100)
    sents = [rng.integers(3, 200, int(rng.integers(1, 20))).tolist() for _ in range(19)]
    eng = pb.Engine(qm, 32, 32, 16)
    fused, plain = _fused_pair(eng, sents, beam, 1.5)
    assert fused == plain
    for i, s in enumerate(sents[:8]):
        toks, lp = om.translate(s, beam, 1.5)
        assert fused[0][i] == toks and fused[1][i] == lp, i


@pytest.mark.parametrize("dup", [3, 40])
def test_vocab_fused_ties(dup):
    """Tie-heavy vocabularies: W_vocab rows repeat every `dup` tokens, so whole
    groups of tokens share one logit.  Exercises the fused merge's exact rescan
    of half-tiles (many equal logits in one 128-token half) and its full-row
    fallback (ties across the candidate boundary)."""
    d = pb.Dims(120, 700, 32, 32, 32, 32)
    params = pb.synthetic_model(d, 9, weight_std=0.4, bias_std=0.0, eos_bias=0.3)
    w = params.tensors["out.w_vocab"]
    params.tensors["out.w_vocab"] = np.ascontiguousarray(w[np.arange(d.tgt_vocab) % dup]).astype(F32)
    qm = pb.quantize_model(params)
    om = O.QModel(O.Dims(**d.as_dict()), params.tensors)
    rng = np.random.default_rng(dup)
    sents = [rng.integers(3, 120, int(rng.integers(1, 9))).tolist() for _ in range(6)]
    eng = pb.Engine(qm, 8, 16, 8)
    fused, plain = _fused_pair(eng, sents, 5, 1.5)
    assert fused == plain
    for i, s in enumerate(sents):
        toks, lp = om.translate(s, 5, 1.5)
        assert fused[0][i] == toks and fused[1][i] == lp, i


@pytest.mark.parametrize("V,k,dup,N", [(50000, 5, 0, 37), (50000, 5, 97, 37), (3001, 8, 7, 37), (700, 16, 0, 37),
                                       (300, 12, 2, 37), (20, 5, 0, 37), (50000, 5, 0, 300), (50000, 3, 5000, 300),
                                       (50000, 6, 11, 1280), (5000, 1, 2, 700), (1, 1, 0, 9)])
def test_vocab_candidates_abi(V, k, dup, N):
    """qnmt_vocab_candidates (fused) == qnmt_gemm_i8 + qnmt_topk_candidates on
    the same codes, including vocabularies with repeated rows (exact ties), over
    1..10 row blocks of the fused kernel."""
    _vocab_candidates_case(V, k, dup, N, 900.0)


@pytest.mark.parametrize("ws", [0.5, 3e-3])
def test_vocab_candidates_wide_logits(ws):
    """Logit ranges far beyond 700 (tiny weight scale): the fused kernel's
    range-guarded exp path (no narrow-tile bound) against GEMM + candidates.
    Tokens must agree exactly. Scores are compared to 4 f64 ulps: when the top
    logit leads the rest by > ~36, lse = log(1 + eps) with eps < 2^-52, so the
    top token's log-prob (~ -eps, a tiny f32) carries the fp64 rounding of
    1 + eps, which depends on summation order."""
    _vocab_candidates_case(5000, 5, 0, 300, ws, score_ulps=4)
    _vocab_candidates_case(5000, 5, 13, 37, ws, score_ulps=4)


def _vocab_candidates_case(V, k, dup, N, wscale, score_ulps=0):
    import torch
    from paper_1804_05038_b200 import _lib, _dev
    rng = np.random.default_rng(V + 31 * k + dup + N)
    K = 64
    w = rng.integers(-127, 128, (V, K)).astype(np.int8)
    if dup:
        w = w[np.arange(V) % dup]
    W = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    X = torch.from_numpy(rng.integers(-127, 128, (N, K)).astype(np.int8)).cuda()
    ws = torch.full((1,), wscale, device="cuda")
    seg = torch.from_numpy((np.arange(N) // 5).astype(np.int32)).cuda()
    xs = torch.from_numpy(rng.uniform(300, 900, N // 5 + 1).astype(np.float32)).cuda()
    bias = torch.from_numpy((np.round(rng.normal(0, 0.5, V) * 8) / 8).astype(np.float32)).cuda()
    live = torch.from_numpy(rng.normal(-10, 3, N)).cuda()
    Y = pb.qmath.gemm_kmajor(W, ws, V, X, xs, col_seg=seg, bias=bias)
    cs0 = torch.empty((N, k), dtype=torch.float64, device="cuda")
    ct0 = torch.empty((N, k), dtype=torch.int32, device="cuda")
    f = _dev.reset_flag()
    _lib.call("qnmt_topk_candidates", Y.data_ptr(), N, V, V, live.data_ptr(), k, cs0.data_ptr(), ct0.data_ptr(),
              f.data_ptr(), _dev.stream_ptr())
    cs1 = torch.empty_like(cs0)
    ct1 = torch.empty_like(ct0)
    scratch = torch.empty(int(_lib.load().qnmt_vocab_candidates_scratch(N, V)), dtype=torch.uint8, device="cuda")
    _lib.call("qnmt_vocab_candidates", X.data_ptr(), N, K, xs.data_ptr(), seg.data_ptr(), W.data_ptr(), V, K, K,
              ws.data_ptr(), V, bias.data_ptr(), live.data_ptr(), k, scratch.data_ptr(), cs1.data_ptr(),
              ct1.data_ptr(), f.data_ptr(), _dev.stream_ptr())
    _dev.raise_flag(f)
    assert torch.equal(ct0, ct1)
    if score_ulps == 0:
        assert torch.equal(cs0, cs1)
    else:
        a, b = cs0.cpu().numpy(), cs1.cpu().numpy()
        assert np.all(np.abs(a - b) <= score_ulps * np.spacing(np.abs(a)))


@pytest.mark.parametrize("query,s0", [("previous", "transform"), ("current", "zero"), ("previous", "zero")])
def test_engine_variants_stacked(query, s0):
    """Engine paths with stacked GEMMs (16-aligned dims): previous-state attention
    query (W_x stacks only) and zero initial state, against the oracle."""
    d = pb.Dims(150, 333, 48, 64, 80, 32)
    params = pb.synthetic_model(d, 13, weight_std=0.3, bias_std=0.2, eos_bias=0.4, s0_mode=s0,
                                attention_query=query)
    qm = pb.quantize_model(params)
    om = O.QModel(O.Dims(**d.as_dict()), params.tensors, s0_mode=s0, attention_query=query)
    rng = np.random.default_rng(len(query) + len(s0))
    sents = [rng.integers(3, 150, int(rng.integers(1, 18))).tolist() for _ in range(15)]
    eng = pb.Engine(qm, 16, 32, 6)
    out = eng.translate_ids(sents, 4, 1.5)
    for i, s in enumerate(sents):
        toks, lp = om.translate(s, 4, 1.5)
        assert out[0][i] == toks and out[1][i] == lp, i


@pytest.mark.gpu
def test_gpu_persistent_greedy_matches_oracle_and_step_graphs():
    """Batch-1 greedy translations through the persistent decode kernel (persistent.cu)
    == the oracle == the step-graph engine, incl. sentences that end on EOS."""
    import paper_1804_05038_b200 as pb
    from paper_1804_05038_b200 import _lib
    lib = _lib.load()
    for seed, ws, bs, eb, s0m in ((61, 0.3, 0.1, 0.6, "transform"), (62, 0.05, 0.0, 0.0, "transform"),
                                  (63, 0.5, 0.1, 1.0, "transform"), (64, 0.3, 0.1, 0.6, "zero")):
        d = pb.Dims(300, 251, 32, 48, 64, 32)
        params = pb.synthetic_model(d, seed, ws, bs, eb, s0_mode=s0m)
        qm = pb.quantize_model(params)
        om = O.QModel(O.Dims(**d.as_dict()), params.tensors, s0_mode=s0m)
        rng = np.random.default_rng(seed)
        for k in range(6):
            src = rng.integers(3, 300, 1 if k == 0 else int(rng.integers(1, 30))).tolist()
            ratio = float(rng.choice([0.5, 1.5, 3.0]))
            old = lib.qnmt_set_greedy1(1)
            got = pb.translate_batch(qm, [src], pb.DecodeConfig(1, ratio, "int8"), return_ids=True)[0]
            lib.qnmt_set_greedy1(0)
            ref = pb.translate_batch(qm, [src], pb.DecodeConfig(1, ratio, "int8"), return_ids=True)[0]
            lib.qnmt_set_greedy1(old)
            want = om.translate(src, 1, ratio)
            assert got[0] == want[0] and got[1] == want[1], (seed, src)
            assert got == ref



@pytest.mark.gpu
def test_gpu_persistent_encoder_matches_batched_encoder():
    """One-sentence encodes (persistent recurrence kernel) == the batched encoder's states,
    att_proj and s0 for the same sentence inside a multi-sentence batch, and == the oracle."""
    import paper_1804_05038_b200 as pb
    d = pb.Dims(300, 251, 32, 48, 64, 32)
    params = pb.synthetic_model(d, 71, 0.3, 0.1, 0.6)
    qm = pb.quantize_model(params)
    om = O.QModel(O.Dims(**d.as_dict()), params.tensors)
    eng = pb.Engine(qm, 8, 64, 4)
    rng = np.random.default_rng(71)
    sents = [rng.integers(3, 300, n).tolist() for n in (1, 2, 7, 33, 64)]
    st_b, att_b, s0_b, rows, lens = eng.encode_batch(sents)
    for k, src in enumerate(sents):
        st1, att1, s01, _, _ = eng.encode_batch([src])
        r0, l = int(rows[k]), len(src)
        assert torch.equal(st1, st_b[r0:r0 + l]) and torch.equal(att1, att_b[r0:r0 + l])
        assert torch.equal(s01[0], s0_b[k])
        ost, oatt, os0 = om.encode(src)
        assert np.array_equal(st1.t().cpu().numpy(), ost) and np.array_equal(att1.t().cpu().numpy(), oatt)
        assert np.array_equal(s01.t().cpu().numpy(), os0)


@pytest.mark.gpu
@pytest.mark.parametrize("hidden", [64, 128, 192, 320])
def test_gpu_cluster_resident_encoder_matches_batched_encoder_and_oracle(hidden):
    """Hidden sizes that are a multiple of 64 take k_enc1c (persistent.cu): the recurrent weights
    resident in the shared memory of one 16-CTA cluster per direction, two cluster barriers and
    two distributed-shared-memory all-gathers per position.  States, att_proj and s0 of
    one-sentence encodes == the batched encoder's (per-step kernels) == the oracle, for lengths
    1 .. 64; the BASELINE-dims cfg2 golden (H = 1024) goes through the same kernel."""
    import paper_1804_05038_b200 as pb
    d = pb.Dims(300, 251, 32, hidden, 64, 32)
    params = pb.synthetic_model(d, 90 + hidden, 0.2, 0.1, 0.6)
    qm = pb.quantize_model(params)
    om = O.QModel(O.Dims(**d.as_dict()), params.tensors)
    eng = pb.Engine(qm, 8, 64, 4)
    rng = np.random.default_rng(hidden)
    sents = [rng.integers(3, 300, n).tolist() for n in (1, 2, 5, 31, 64)]
    st_b, att_b, s0_b, rows, lens = eng.encode_batch(sents)
    for k, src in enumerate(sents):
        st1, att1, s01, _, _ = eng.encode_batch([src])
        r0, l = int(rows[k]), len(src)
        assert torch.equal(st1, st_b[r0:r0 + l]) and torch.equal(att1, att_b[r0:r0 + l])
        assert torch.equal(s01[0], s0_b[k])
        ost, oatt, os0 = om.encode(src)
        assert np.array_equal(st1.t().cpu().numpy(), ost) and np.array_equal(att1.t().cpu().numpy(), oatt)
        assert np.array_equal(s01.t().cpu().numpy(), os0)


@pytest.mark.gpu
@pytest.mark.parametrize("vocab,attn", [(297, 16), (40, 32), (700, 16), (1297, 64)])
def test_gpu_persistent_greedy_small_vocabulary(vocab, attn):
    """Regression: the persistent batch-1 greedy kernel writes one (max, sum) pair per CTA into the
    engine's vocabulary-partials buffer; sized for the fused kernel's partials of one row it was too
    small for vocabularies under ~6000 tokens, and the overflow corrupted the attention scores of
    the same step (NumericError on finite models; found by benchmarks/stress_parity.py)."""
    import paper_1804_05038_b200 as pb
    d = pb.Dims(188, vocab, 16, 128, attn, 48)
    params = pb.synthetic_model(d, 169549767, 0.2, 0.1, 1.5, "transform", "current")
    qm = pb.quantize_model(params)
    om = O.QModel(O.Dims(**d.as_dict()), params.tensors)
    rng = np.random.default_rng(vocab)
    for _ in range(4):
        s = rng.integers(3, 188, int(rng.integers(1, 20))).tolist()
        got = pb.translate_batch(qm, [s], pb.DecodeConfig(1, 1.0, "int8"), return_ids=True)[0]
        want = om.translate(s, 1, 1.0)
        assert got[0] == want[0] and got[1] == want[1], (vocab, attn, s)
