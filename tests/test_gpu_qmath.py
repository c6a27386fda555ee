"""GPU parity of K1 (quantize) and K2/K3 (int8 GEMM + dequant) against the
reference goldens and the oracle: bit-exact for codes, scales, int32/int64
accumulators and dequantized f32 outputs."""

import numpy as np
import pytest
import torch

from oracle import qnmt_oracle as O
from qnmt_test_helpers import F32, golden, sha

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_1804_05038_b200")
from paper_1804_05038_b200 import _lib  # noqa: E402
from paper_1804_05038_b200.errors import InvalidInputError, NumericError, ShapeError  # noqa: E402


@pytest.fixture(scope="module")
def kat():
    return golden("qmath_kat.npz")


def rand_q(rng, rows, cols):
    codes = rng.integers(-127, 128, (rows, cols)).astype(np.int8)
    return pb.QuantizedMatrix(codes, float(np.float32(rng.uniform(0.5, 200.0))))


def test_quantize_known_answers(kat):
    names = sorted({k[2:-3] for k in kat.files if k.startswith("q_") and k.endswith("_in")})
    for n in names:
        q = pb.quantize(kat[f"q_{n}_in"])
        assert np.array_equal(q.data, kat[f"q_{n}_codes"]), n
        assert q.scale == float(kat[f"q_{n}_scale"]), n
        qa = pb.quantize_activations(kat[f"q_{n}_in"])
        assert np.array_equal(qa.data, kat[f"q_{n}_codes"]), n
    assert pb.quantize(np.array([[2, 1, -1]], F32)).data.tolist() == [[127, 64, -64]]
    assert pb.quantize(np.array([[127, 0.49999997]], F32)).data.tolist() == [[127, 1]]
    q = pb.quantize(np.array([[10.0]], F32))
    assert q.data[0, 0] == 127 and q.scale == pytest.approx(12.7, abs=1e-5)
    z = pb.quantize(np.zeros((3, 3), F32))
    assert z.scale == 1.0 and not z.data.any()


def test_quantize_errors():
    with pytest.raises(InvalidInputError):
        pb.quantize(np.array([[1.0, np.nan]], F32))
    with pytest.raises(InvalidInputError):
        pb.quantize(np.array([[np.inf]], F32))
    with pytest.raises(NumericError):
        pb.quantize_activations(np.array([[1.0], [np.nan]], F32))
    with pytest.raises(ShapeError):
        pb.quantize(np.zeros((0, 3), F32))


@pytest.mark.parametrize("seed", range(40))
def test_quantize_random_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    shape = (int(rng.integers(1, 70)), int(rng.integers(1, 300)))
    scale = [1e-3, 1.0, 50.0, 1e6][seed % 4]
    m = (rng.normal(0, 1, shape) * scale).astype(F32)
    if seed % 5 == 0:
        m[rng.integers(0, shape[0]), rng.integers(0, shape[1])] = 0.5 / F32(127) * m.max()
    q = pb.quantize(m)
    oc, os_ = O.quantize(m)
    assert np.array_equal(q.data, oc) and q.scale == os_
    # symmetry and idempotence (test_qmath.py:84-103)
    qn = pb.quantize(-m)
    assert np.array_equal(qn.data, -q.data) and qn.scale == q.scale
    q2 = pb.quantize(pb.dequantize(q))
    assert np.array_equal(q2.data, q.data)


def test_dequantize():
    q = pb.QuantizedMatrix(np.array([[127]], dtype=np.int8), 12.7)
    assert pb.dequantize(q)[0, 0] == pytest.approx(10.0, abs=1e-5)
    rng = np.random.default_rng(0)
    q = rand_q(rng, 7, 9)
    assert np.array_equal(pb.dequantize(q), O.dequantize(q.data, q.scale))


def test_qgemm_known_answers(kat):
    for i in range(int(kat["g_count"])):
        a = pb.QuantizedMatrix(kat[f"g{i}_a"], float(kat[f"g{i}_sa"]))
        b = pb.QuantizedMatrix(kat[f"g{i}_b"], float(kat[f"g{i}_sb"]))
        y = pb.qgemm_panel(a, b)
        assert np.array_equal(y, kat[f"g{i}_y"]), i
        assert np.array_equal(pb.qgemm(a, b), kat[f"g{i}_y"]), i


@pytest.mark.parametrize("seed", range(60))
def test_qgemm_random_bit_exact(seed):
    """test_qmath.py:153-163 property, extended to the tiled shapes (N up to 300)."""
    rng = np.random.default_rng(1000 + seed)
    if seed < 30:
        m, k, p = int(rng.integers(1, 65)), int(rng.integers(1, 65)), int(rng.integers(1, 9))
    else:
        m = int(rng.integers(1, 400))
        k = int(16 * rng.integers(1, 80)) if seed % 2 else int(64 * rng.integers(1, 20))
        p = int(rng.integers(1, 300))
    a, b = rand_q(rng, m, k), rand_q(rng, k, p)
    expect = O.qgemm(a.data, a.scale, b.data, b.scale)
    assert np.array_equal(pb.qgemm(a, b), expect)
    acc = pb.qmath.qgemm_acc(a, b).cpu().numpy()
    assert np.array_equal(acc, O.int_product(a.data, b.data))


def test_int64_widening_beyond_safe_k():
    rng = np.random.default_rng(5)
    k = pb.INT32_SAFE_K + 64
    a = pb.QuantizedMatrix(rng.integers(-127, 128, (2, k)).astype(np.int8), 1.0)
    b = pb.QuantizedMatrix(rng.integers(-127, 128, (k, 2)).astype(np.int8), 1.0)
    expect = O.qgemm(a.data, 1.0, b.data, 1.0)
    assert np.array_equal(pb.qgemm(a, b), expect)
    big = pb.QuantizedMatrix(np.full((1, k), 127, np.int8), 1.0)
    bb = pb.QuantizedMatrix(np.full((k, 1), 127, np.int8), 1.0)
    assert pb.qmath.qgemm_acc(big, bb).item() == 127 * 127 * k   # > 2^31


def test_shape_errors():
    rng = np.random.default_rng(0)
    with pytest.raises(ShapeError):
        pb.qgemm(rand_q(rng, 3, 4), rand_q(rng, 5, 2))
    with pytest.raises(InvalidInputError):
        pb.qgemm(np.zeros((2, 2), np.int8), rand_q(rng, 2, 2))


@pytest.mark.parametrize("bsz", [1, 64])
def test_cfg1_bit_exact(kat, bsz):
    """BASELINE cfg1: W [3072x1024] N(0,0.05), X [1024xB] N(0,1)."""
    w = np.random.default_rng(1804).normal(0, 0.05, (3072, 1024)).astype(F32)
    wq = pb.quantize(w)
    assert wq.scale == float(kat["cfg1_w_scale"]) and sha(wq.data) == str(kat["cfg1_w_codes_sha"])
    x = np.random.default_rng(5038 + bsz).normal(0, 1, (1024, bsz)).astype(F32)
    xq = pb.quantize_activations(x)
    assert xq.scale == float(kat[f"cfg1_b{bsz}_x_scale"])
    assert sha(xq.data) == str(kat[f"cfg1_b{bsz}_x_codes_sha"])
    acc = pb.qmath.qgemm_acc(wq, xq).cpu().numpy()
    assert sha(acc.astype(np.int32)) == str(kat[f"cfg1_b{bsz}_acc_sha"])
    y = pb.qgemm_panel(wq, xq)
    assert sha(y) == str(kat[f"cfg1_b{bsz}_y_sha"])
    # the same through torch tensors (device-resident API)
    yt = pb.qgemm(pb.quantize(torch.from_numpy(w).cuda()), pb.quantize_activations(torch.from_numpy(x).cuda()))
    assert isinstance(yt, torch.Tensor) and np.array_equal(yt.cpu().numpy(), y)


@pytest.mark.parametrize("seed", range(8))
def test_segmented_quantize_vs_oracle(seed):
    """Per-segment scales (batched decode): each segment equals an independent
    quantize_activations of that segment's columns."""
    rng = np.random.default_rng(77 + seed)
    K = int(rng.choice([12, 512, 1024, 2048]))
    nseg = int(rng.integers(1, 9))
    widths = rng.integers(1, 6, nseg)
    cols = []
    seg = []
    for s, w in enumerate(widths):
        cols.append((rng.normal(0, 1, (w, K)) * 10.0 ** rng.uniform(-3, 3)).astype(F32))
        seg += [s] * int(w)
    x = np.concatenate(cols)
    from paper_1804_05038_b200.layers import _quant_k
    xd = torch.from_numpy(x).cuda()
    segd = torch.tensor(seg, dtype=torch.int32, device="cuda")
    q, sc = _quant_k(xd, segd, nseg)
    q, sc = q.cpu().numpy(), sc.cpu().numpy()
    r = 0
    for s, w in enumerate(widths):
        oc, os_ = O.quantize_activations(cols[s].T)
        assert sc[s] == np.float32(os_)
        assert np.array_equal(q[r:r + w].T, oc)
        r += w


def test_library_loaded_from_tree():
    import os
    assert os.path.exists(_lib.LIB_PATH)
    maps = open("/proc/self/maps").read()
    assert "libqnmt_b200.so" in maps


SHAPES_TC = [(128, 128, 16), (128, 128, 64), (130, 256, 9), (3072, 1024, 1280), (50000 // 7, 512, 333),
             (2048, 1024, 256), (1024, 2048, 1000), (77, 80, 300), (512, 96, 17), (1000, 1024, 64),
             (256, 2048, 2), (384, 512, 1)]


@pytest.mark.parametrize("shape", SHAPES_TC)
def test_tcgen05_gemm_bit_exact(shape):
    """K3 (tcgen05.mma kind::i8) == CUDA-core path == oracle, incl. M/N/K tails."""
    M, K, N = shape
    rng = np.random.default_rng(M * 7 + K + N)
    W = pb.QuantizedMatrix(rng.integers(-127, 128, (M, K)).astype(np.int8), float(np.float32(rng.uniform(1, 300))))
    X = pb.QuantizedMatrix(rng.integers(-127, 128, (K, N)).astype(np.int8), float(np.float32(rng.uniform(1, 300))))
    expect = O.qgemm(W.data, W.scale, X.data, X.scale)
    lib = _lib.load()
    old = lib.qnmt_set_gemm_impl(2)
    try:
        y_tc = pb.qgemm(W, X)
        acc_tc = pb.qmath.qgemm_acc(W, X).cpu().numpy()
        lib.qnmt_set_gemm_impl(1)
        y_dp = pb.qgemm(W, X)
    finally:
        lib.qnmt_set_gemm_impl(old)
    assert np.array_equal(acc_tc, O.int_product(W.data, X.data))
    assert np.array_equal(y_tc, expect)
    assert np.array_equal(y_dp, expect)


def test_tcgen05_segmented_bias_accumulate():
    """Segmented activation scales + bias + ACCUMULATE epilogue on the tensor-core path."""
    import torch
    rng = np.random.default_rng(9)
    M, K, N, S = 640, 1024, 700, 37
    Wc = rng.integers(-127, 128, (M, K)).astype(np.int8)
    Xc = rng.integers(-127, 128, (N, K)).astype(np.int8)
    seg = np.sort(rng.integers(0, S, N)).astype(np.int32)
    ws = np.float32(rng.uniform(10, 200, 2))          # two row blocks of 320
    xs = np.float32(rng.uniform(10, 200, S))
    bias = rng.normal(0, 1, M).astype(np.float32)
    y0 = rng.normal(0, 1, (N, M)).astype(np.float32)
    d = lambda a: torch.from_numpy(a).cuda()
    Y = d(y0.copy())
    lib = _lib.load()
    old = lib.qnmt_set_gemm_impl(2)
    try:
        pb.qmath.gemm_kmajor(d(Wc), d(ws), 320, d(Xc), d(xs), col_seg=d(seg), bias=d(bias), Y=Y, accumulate=True)
    finally:
        lib.qnmt_set_gemm_impl(old)
    acc = O.int_product(Wc, Xc.T)                       # [M, N]
    ref = np.empty((N, M), np.float32)
    for n in range(N):
        for blk in range(2):
            rows = slice(320 * blk, 320 * (blk + 1))
            yv = O.scale_output(acc[rows, n], ws[blk], xs[seg[n]])
            ref[n, rows] = y0[n, rows] + (yv + bias[rows])
    assert np.array_equal(Y.cpu().numpy(), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("M,K,N", [(4096, 1024, 2560), (4100, 1040, 2600), (8192, 512, 4864)])
def test_gpu_tc_pair_kernel_matches_single_cta(M, K, N):
    """CTA-pair tcgen05 GEMM (cta_group::2, M = 256 tiles) == single-CTA kernel and the
    exact integer product (torch._int_mm on the device, int32), incl. M/N/K tails."""
    import torch
    from paper_1804_05038_b200 import _lib
    import paper_1804_05038_b200 as pb
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    W = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda", generator=g)
    X = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda", generator=g)
    ws = torch.rand(1, device="cuda", generator=g) * 100 + 1
    xs = torch.rand(16, device="cuda", generator=g) * 100 + 1
    seg = (torch.arange(N, device="cuda", dtype=torch.int32) * 16) // N
    bias = torch.randn(M, device="cuda", generator=g)
    lib = _lib.load()
    outs = []
    for pair in (1, 0):
        old = lib.qnmt_set_tc_pair(pair)
        acc = torch.empty((N, M), dtype=torch.int64, device="cuda")
        Y = pb.qmath.gemm_kmajor(W, ws, M, X, xs, col_seg=seg, bias=bias, acc_out=acc,
                                 Y=torch.empty((N, M), dtype=torch.float32, device="cuda"))
        lib.qnmt_set_tc_pair(old)
        outs.append((acc, Y))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    if K % 8 == 0 and N % 8 == 0 and M % 8 == 0:
        ref = torch._int_mm(X, W.t())
        assert torch.equal(outs[0][0], ref.to(torch.int64))


SHAPES_SPLIT = [(3072, 1024, 64), (3072, 1024, 9), (512, 4096, 33), (1000, 2048, 100), (128, 8192, 16),
                (2048, 512, 128), (77, 1024, 300), (6000, 1024, 20)]


@pytest.mark.parametrize("shape", SHAPES_SPLIT)
def test_tcgen05_split_k_bit_exact(shape):
    """Tile-starved tcgen05 products split K over more CTAs (int32 partials added in a
    workspace, the last split runs the epilogue): results identical with and without
    the split and to the oracle, repeated calls included (the workspace is left zeroed),
    with segmented scales, bias and ACCUMULATE."""
    import torch
    M, K, N = shape
    rng = np.random.default_rng(M + 3 * K + 7 * N)
    Wc = rng.integers(-127, 128, (M, K)).astype(np.int8)
    Xc = rng.integers(-127, 128, (N, K)).astype(np.int8)
    S = max(1, N // 5)
    seg = np.sort(rng.integers(0, S, N)).astype(np.int32)
    ws = np.float32(rng.uniform(50, 300))
    xs = rng.uniform(50, 300, S).astype(np.float32)
    bias = rng.normal(0, 1, M).astype(np.float32)
    y0 = rng.normal(0, 1, (N, M)).astype(np.float32)
    W, X = torch.from_numpy(Wc).cuda(), torch.from_numpy(Xc).cuda()
    wsd = torch.tensor([ws], device="cuda")
    xsd, segd = torch.from_numpy(xs).cuda(), torch.from_numpy(seg).cuda()
    bd = torch.from_numpy(bias).cuda()
    lib = _lib.load()
    outs = []
    old_i = lib.qnmt_set_gemm_impl(2)
    try:
        for split in (1, 0, 1):   # (split on, off, on again: the workspace is reused)
            old = lib.qnmt_set_tc_split(split)
            try:
                Y = torch.from_numpy(y0.copy()).cuda()
                pb.qmath.gemm_kmajor(W, wsd, M, X, xsd, col_seg=segd, bias=bd, Y=Y, accumulate=True)
                acc = torch.empty((N, M), dtype=torch.int64, device="cuda")
                pb.qmath.gemm_kmajor(W, wsd, M, X, xsd, col_seg=segd, acc_out=acc)
                outs.append((Y.cpu().numpy(), acc.cpu().numpy()))
            finally:
                lib.qnmt_set_tc_split(old)
    finally:
        lib.qnmt_set_gemm_impl(old_i)
    exact = Xc.astype(np.int64) @ Wc.astype(np.int64).T
    for Y, acc in outs:
        assert np.array_equal(acc, exact)
        assert np.array_equal(Y, outs[1][0])
    # against the oracle: y = Y + (fl32(acc / (sw * sx)) + b) (qmath.py:379-381, layers.py:144-145)
    dq = (exact.astype(np.float64) / (np.float64(ws) * xs[seg].astype(np.float64)[:, None])).astype(np.float32)
    assert np.array_equal(outs[0][0], y0 + (dq + bias[None, :]))


@pytest.mark.parametrize("N,K,M", [(1, 1024, 3072), (2, 512, 1000), (5, 2048, 513), (8, 4096, 256), (3, 16, 7),
                                   (1, 8192, 64), (9, 1024, 300), (64, 1024, 3072)])
def test_linear_i8_matches_oracle(N, K, M):
    """qnmt_linear_i8 (LinearOp.apply, layers.py:124-146: quantize_activations +
    qgemm_panel + bias; one kernel for N <= 8, quantize + GEMM beyond) == oracle:
    codes, scale and outputs bit-exact."""
    import torch
    from paper_1804_05038_b200 import _dev
    rng = np.random.default_rng(N * 1000 + K + M)
    w = rng.normal(0, 0.05, (M, K)).astype(np.float32)
    x = (rng.normal(0, 1, (K, N)) * rng.uniform(0.01, 10)).astype(np.float32)
    b = rng.normal(0, 0.1, M).astype(np.float32)
    wq = pb.quantize(w)
    xq_c, xq_s = O.quantize_activations(x)
    expect = O.qgemm(wq.data, wq.scale, xq_c, xq_s) + b[:, None]
    op = pb.LinearOp(wq, b)
    y = op.apply(x)
    assert np.array_equal(y, expect)
    # raw ABI: codes and scale
    Xk = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    W = wq.device_data()
    Y = torch.empty((N, M), device="cuda")
    q = torch.empty((N, K), dtype=torch.int8, device="cuda")
    sx = torch.empty(1, device="cuda")
    bits = torch.empty(1, dtype=torch.int32, device="cuda")
    f = _dev.reset_flag()
    _lib.call("qnmt_linear_i8", W.data_ptr(), M, K, K, wq.device_scale().data_ptr(), M, Xk.data_ptr(), N, K,
              torch.from_numpy(b).cuda().data_ptr(), Y.data_ptr(), M, q.data_ptr(), K, sx.data_ptr(), bits.data_ptr(),
              _lib.GEMM_W_STATIC, f.data_ptr(), _dev.stream_ptr())
    _dev.raise_flag(f)
    assert float(sx.item()) == xq_s
    assert np.array_equal(q.cpu().numpy().T, xq_c)
    assert np.array_equal(Y.cpu().numpy().T, expect)


def test_linear_i8_nonfinite_raises():
    rng = np.random.default_rng(3)
    wq = pb.quantize(rng.normal(0, 0.05, (64, 32)).astype(np.float32))
    x = rng.normal(0, 1, (32, 1)).astype(np.float32)
    x[5, 0] = np.inf
    with pytest.raises(pb.errors.NumericError):
        pb.LinearOp(wq, None).apply(x)


@pytest.mark.parametrize("shape", [(1, 4), (1, 16), (3, 1364), (8, 1024), (63, 1040), (64, 1024), (16, 4096),
                                   (64, 1028), (65, 1024), (9, 7)])
def test_cluster_quantize_small_matrices(shape):
    """One-launch quantization of small single-segment matrices (k_quant_cluster: 8 CTAs, values in
    registers, maxima through distributed shared memory) and its neighbours just beyond the
    65536-value capacity / with a length that is not a multiple of 4 (two-pass kernels): codes
    and scale == the oracle's quantize_activations, incl. all-zero input and a huge dynamic range."""
    from paper_1804_05038_b200.layers import _quant_k
    n, K = shape
    rng = np.random.default_rng(n * 10007 + K)
    for kind in ("normal", "zero", "range", "tiny"):
        if kind == "normal":
            x = rng.normal(0, 1, (n, K)).astype(F32)
        elif kind == "zero":
            x = np.zeros((n, K), F32)
        elif kind == "range":
            x = (rng.normal(0, 1, (n, K)) * 10.0 ** rng.uniform(-6, 6, (n, K))).astype(F32)
        else:
            x = (rng.normal(0, 1, (n, K)) * 1e-30).astype(F32)
        q, sc = _quant_k(torch.from_numpy(x).cuda())
        oc, os_ = O.quantize_activations(x.T)
        assert sc.cpu().numpy()[0] == np.float32(os_), (shape, kind)
        assert np.array_equal(q.cpu().numpy().T, oc), (shape, kind)


def test_cluster_quantize_non_finite_raises():
    x = np.ones((64, 1024), F32)
    x[17, 333] = np.inf
    with pytest.raises(pb.errors.NumericError):
        pb.quantize_activations(torch.from_numpy(np.ascontiguousarray(x.T)).cuda())
    x[17, 333] = np.nan
    with pytest.raises(pb.errors.NumericError):
        pb.quantize_activations(torch.from_numpy(np.ascontiguousarray(x.T)).cuda())
