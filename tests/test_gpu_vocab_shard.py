"""K7, the vocabulary-sharded output projection (paper_1804_05038_b200/vocab_shard.py,
SURVEY 8(e)): W_vocab split over G shards, per-shard (max, sum exp, top-8 logits)
partials, combined into the step's candidates.  On one GPU the shards are emulated
one after another -- the same partial / combine kernels and the same bytes the NCCL
all-gather carries under torchrun.  Candidates must equal the unsharded fused path
(qnmt_vocab_candidates, itself pinned to the GEMM + candidate kernel and the
oracle) bit for bit, for any shard count, including tie-heavy vocabularies."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
pb = pytest.importorskip("paper_1804_05038_b200")
from paper_1804_05038_b200 import vocab_shard as VS  # noqa: E402


def _case(V, K, N, k, dup, seed, wscale=900.0):
    rng = np.random.default_rng(seed)
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
    return X, xs, seg, W, ws, bias, live


@pytest.mark.parametrize("V,K,N,k,dup", [(50000, 512, 300, 5, 0), (50000, 64, 1280, 5, 0), (32000, 512, 37, 1, 0),
                                         (5000, 64, 100, 8, 0), (3001, 64, 37, 5, 7), (50000, 64, 37, 5, 97)])
@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_sharded_equals_unsharded(V, K, N, k, dup, G):
    X, xs, seg, W, ws, bias, live = _case(V, K, N, k, dup, V + K + N + G)
    cs0, ct0 = VS.unsharded(X, xs, seg, W, ws, bias, live, k)
    cs1, ct1 = VS.candidates(X, xs, seg, W, ws, bias, live, k, shards=G)
    assert torch.equal(ct0, ct1)
    assert torch.equal(cs0, cs1)


def test_shard_partials_content():
    """One shard's partial: M = max logit, S = sum exp(x - M), top-8 by (logit desc,
    token asc) with global ids -- checked against the materialised logits."""
    V, K, N = 4000, 64, 21
    X, xs, seg, W, ws, bias, live = _case(V, K, N, 5, 0, 3)
    lo, hi = 1152, 2304
    parts = VS.shard_partials(X, xs, seg, W, ws, bias, lo, hi).cpu().numpy()
    Y = pb.qmath.gemm_kmajor(W, ws, V, X, xs, col_seg=seg, bias=bias).cpu().numpy()   # [N][V] exact logits
    for n in range(N):
        rec = parts[n]
        S = rec[0:8].view(np.float64)[0]
        M = rec[8:12].view(np.float32)[0]
        cnt = rec[12:16].view(np.int32)[0]
        xsv = rec[16:48].view(np.float32)
        tok = rec[48:80].view(np.int32)
        row = Y[n, lo:hi]
        assert M == row.max() and cnt == 8
        order = sorted(range(hi - lo), key=lambda v: (-row[v], v))[:8]
        assert tok.tolist() == [lo + v for v in order]
        assert np.array_equal(xsv, row[order])
        ref = np.sum(np.exp(row.astype(np.float64) - np.float64(M)))
        assert abs(S - ref) <= 1e-12 * ref


def test_shard_bounds_cover():
    for V in (1, 191, 192, 50000, 32000):
        for G in (1, 2, 3, 8, 16):
            b = VS.shard_bounds(V, G)
            assert b[0][0] == 0 and b[-1][1] == V and len(b) == G
            assert all(b[i][1] == b[i + 1][0] for i in range(G - 1))
            assert all(lo % VS.TILE == 0 or lo == V for lo, _ in b)


_NCCL_CHILD = r"""
import os, sys
sys.path.insert(0, {root!r})
sys.path.insert(0, os.path.join({root!r}, "tests"))
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", {port!r})
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
from paper_1804_05038_b200 import vocab_shard as VS
from test_gpu_vocab_shard import _case
ok = True
for (V, K, N, k, dup) in [(50000, 64, 300, 5, 0), (3001, 64, 37, 5, 7)]:
    X, xs, seg, W, ws, bias, live = _case(V, K, N, k, dup, V + K + N)
    cs0, ct0 = VS.unsharded(X, xs, seg, W, ws, bias, live, k)
    cs1, ct1 = VS.candidates(X, xs, seg, W, ws, bias, live, k, group=dist.group.WORLD)
    ok &= bool(torch.equal(ct0, ct1)) and bool(torch.equal(cs0, cs1))
dist.barrier()
dist.destroy_process_group()
print("NCCL_K7_OK" if ok else "NCCL_K7_MISMATCH")
"""


def test_nccl_group_path_world_size_1(tmp_path):
    """The NCCL branch of candidates() (all_gather_into_tensor of the partials, combine) on a
    one-rank NCCL group: the only multi-GPU code path of the project, exercised on the one GPU
    of the box (a real exchange needs more GPUs; the bytes and the combine are the same)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "k7_nccl_child.py"
    script.write_text(_NCCL_CHILD.format(root=root, port=str(29500 + os.getpid() % 2000)))
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "NCCL_K7_OK" in r.stdout, (r.stdout + r.stderr)[-3000:]
