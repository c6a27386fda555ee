"""The attention scorer's variants give identical codes, scores, alpha and
context (attention.cu):

* two-MUFU scorer (k_att_score5): t = 1 - 2 / (1 + 2^(2x log2 e)) per element,
  with its per-hypothesis scales from k_att_scale or computed in its own CTAs
  (k_att_score5f, the default);
* one-MUFU scorer (k_att_score6): e^(2(ap+u)) = E_ap * E_u from per-batch /
  per-step fp64 exps, rounding-window elements queued and resolved exactly
  by the CTA's last warp;
* k_att_score8: the two-MUFU scorer with its att_proj tile staged by one bulk
  copy before the PDL wait, branch-free position loop and dp4a code sums;
* k_att_score7: the one-MUFU scorer with its tile staged by one bulk copy
  before the PDL wait, branch-free position loop and dp4a code dot products;
* score6 / score7 with the fixup queue disabled (every window hit goes
  through the queue-overflow rescan of the whole CTA).

The two-MUFU scorer is pinned against the oracle by test_gpu_layers.py and the
decode goldens; here the variants are compared at BASELINE attention size (A =
2048, 2H = 2048) over a batch with l ~ U[5, 100], beams 1..16, and inputs
scaled so that part of the batch is beyond the one-MUFU path's |x| <= 20
eligibility bound (those sentences take the two-MUFU path inside score6)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
pb = pytest.importorskip("paper_1804_05038_b200")
from paper_1804_05038_b200 import _dev, _lib  # noqa: E402

# (scorer variant, fixup queue length, scale fused into the two-MUFU scorer, bulk-staged two-MUFU scorer)
MODES = [(0, 512, 0, 0), (0, 512, 0, 1), (0, 512, 1, 0), (1, 512, 0, 0), (1, 0, 0, 0), (2, 512, 0, 0),
         (2, 0, 0, 0)]


def _run(lib, mode, inp):
    old_e = lib.qnmt_set_att_exp(mode[0])
    old_c = lib.qnmt_set_att_fixcap(mode[1])
    old_f = lib.qnmt_set_att_fused_scale(mode[2])
    old_8 = lib.qnmt_set_att_score8(mode[3])
    try:
        (att, ex, states, u, v, vs, off, cnt, rows_d, lens_d, S, N, A, H2, max_len) = inp
        mm = torch.empty((S, 2, A), device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        _lib.call("qnmt_attention_stats", att.data_ptr(), rows_d.data_ptr(), lens_d.data_ptr(), S, A,
                  mm.data_ptr(), st)
        ctx = torch.empty((N, H2), device="cuda")
        alpha = torch.zeros((N, max_len), device="cuda")   # (entries past a sentence's length stay 0)
        scratch = torch.empty(N * (104 + A) + 4 * N * max_len + 1024, dtype=torch.int32, device="cuda")
        f = _dev.reset_flag()
        _lib.call("qnmt_attention", u.data_ptr(), A, N, off.data_ptr(), cnt.data_ptr(), S, att.data_ptr(),
                  mm.data_ptr(), ex.data_ptr(), states.data_ptr(), rows_d.data_ptr(), lens_d.data_ptr(), max_len,
                  A, H2, v.data_ptr(), vs.data_ptr(), ctx.data_ptr(), H2, alpha.data_ptr(), max_len,
                  scratch.data_ptr(), f.data_ptr(), st)
        torch.cuda.synchronize()
        assert not bool(f.any())
        return ctx.cpu().numpy(), alpha.cpu().numpy()
    finally:
        lib.qnmt_set_att_exp(old_e)
        lib.qnmt_set_att_fixcap(old_c)
        lib.qnmt_set_att_fused_scale(old_f)
        lib.qnmt_set_att_score8(old_8)


def _inputs(seed, beams, scale_u, scale_ap, A=2048, H2=2048):
    rng = np.random.default_rng(seed)
    S = len(beams)
    lens = rng.integers(5, 101, S).astype(np.int32)
    rows = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    Pn = int(lens.sum())
    N = int(sum(beams))
    g = torch.Generator(device="cuda").manual_seed(seed)
    att = torch.randn((Pn, A), device="cuda", generator=g) * scale_ap
    states = torch.randn((Pn, H2), device="cuda", generator=g) * 0.5
    u = torch.randn((N, A), device="cuda", generator=g) * scale_u
    v = torch.randint(-127, 128, (A,), dtype=torch.int8, device="cuda", generator=g)
    vs = torch.full((1,), 90.0, device="cuda")
    off = torch.from_numpy(np.concatenate([[0], np.cumsum(beams)[:-1]]).astype(np.int32)).cuda()
    cnt = torch.from_numpy(np.asarray(beams, np.int32)).cuda()
    ex = torch.empty_like(att)
    _lib.call("qnmt_attention_exp", att.data_ptr(), att.numel(), ex.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    return (att, ex, states, u, v, vs, off, cnt, torch.from_numpy(rows).cuda(), torch.from_numpy(lens).cuda(),
            S, N, A, H2, int(lens.max()))


@pytest.mark.parametrize("case", [
    ("beam5", 11, [5] * 24, 0.5, 0.5),
    ("ragged_beams", 12, [1, 2, 3, 4, 5, 8, 16, 7, 5, 1, 16, 3], 0.5, 0.5),
    ("wide", 13, [5] * 12, 6.0, 6.0),          # |ap| / |u| partly beyond 20: mixed eligibility
    ("tiny", 14, [5] * 8, 1e-4, 1e-4),         # large per-hypothesis scales
    ("small_A", 15, [5, 3, 1, 5], 0.5, 0.5, 40, 96),    # A, 2H below one CTA's quads
    ("mid_A", 16, [5] * 6, 0.5, 0.5, 1000, 512),
    ("small_x", 17, [5] * 12, 0.09, 0.09),     # |x| <= 0.75 throughout (the decode's own range)
    ("small_x_mixed", 18, [5, 3, 5, 1] * 4, 0.12, 0.12),
])
def test_scorer_variants_identical(case):
    _, seed, beams, su, sa = case[:5]
    lib = _lib.load()
    inp = _inputs(seed, beams, su, sa, *case[5:])
    ref_ctx, ref_alpha = _run(lib, MODES[0], inp)
    for mode in MODES[1:]:
        ctx, alpha = _run(lib, mode, inp)
        bad = np.argwhere(alpha != ref_alpha)
        assert np.array_equal(alpha, ref_alpha), (mode, len(bad), bad[:6].tolist(),
                                                  [(float(alpha[tuple(b)]), float(ref_alpha[tuple(b)])) for b in bad[:3]])
        assert np.array_equal(ctx, ref_ctx), mode


@pytest.mark.parametrize("A", [2052, 2304, 4096])
def test_attention_dims_beyond_2048_match_the_oracle(A):
    """Attention dims past the register-resident scorers (A > 2048) take the strided
    kernels (k_att_scale_wide / k_att_score_wide): attend, a teacher-free beam decode and a
    batch decode are bit-identical to the oracle."""
    from oracle import qnmt_oracle as O
    d = pb.Dims(64, 61, 16, 32, A, 16)
    params = pb.synthetic_model(d, 21, weight_std=0.3, bias_std=0.1, eos_bias=0.5)
    qm = pb.quantize_model(params)
    om = O.QModel(O.Dims(**d.as_dict()), params.tensors)
    net = pb.build_network(qm)
    src = [5, 9, 17, 33, 40, 8, 2, 11]
    enc = net.encode(src)
    rng = np.random.default_rng(A)
    for P, scale in ((1, 1.0), (5, 1.0), (16, 1.0), (3, 1e-5), (4, 30.0)):
        h = (rng.normal(0, 0.5, (d.hidden, P)) * scale).astype(np.float32)
        att_proj = (enc.att_proj * np.float32(scale)).astype(np.float32)
        ctx, alpha = pb.attend(net.attention, h, pb.EncoderStates(enc.states, att_proj, enc.s0))
        ctx_o, alpha_o = om.attend(h, enc.states, att_proj)
        assert np.array_equal(alpha, alpha_o), (P, scale)
        assert np.array_equal(ctx, ctx_o), (P, scale)
    srcs = [src, [3, 4], list(range(10, 31))]
    got = pb.translate_batch(qm, srcs, pb.DecodeConfig(beam=3, max_ratio=2.0, precision="int8"), return_ids=True)
    for sr, g in zip(srcs, got):
        want = om.translate(sr, beam=3, max_ratio=2.0)
        assert g[0] == want[0] and g[1] == want[1], (sr, g, want)
    one = pb.translate_batch(qm, [src], pb.DecodeConfig(beam=1, max_ratio=1.5, precision="int8"), return_ids=True)[0]
    want = om.translate(src, beam=1, max_ratio=1.5)
    assert one[0] == want[0] and one[1] == want[1]
