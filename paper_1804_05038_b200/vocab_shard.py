"""K7: the vocabulary-sharded output projection (BASELINE cfg5's
optional variant) -- the B200 restatement of layers.py:266 (vocab LinearOp),
:60-67 (_log_softmax_cols) and decoder.py:74-85/:125 (candidates per parent)
with W_vocab split row-wise over G shards.

Each shard (one GPU, or one emulated slice on a single GPU) runs the fused
tcgen05 vocab kernel over its rows and reduces every hypothesis row to an
80-byte partial: its max logit M_g, S_g = sum exp(x - M_g) (fp64) and its
top-8 logits (qnmt_vocab_shard_partials).  The partials are exchanged
(NCCL all-gather over NVLink when ``group`` is a process group: N * 80 bytes
per rank per step) and every rank combines them into the same candidates
(qnmt_vocab_shard_combine): M = max M_g, lse = log sum_g S_g e^(M_g - M),
scores live + fl32((x - M) - lse) over the union of the shards' lists.  The
union holds the global top-k unless a shard's 8th candidate ties into the
top-k (f32 score ties); those steps are recomputed unsharded
(QNMT_FLAG_SHARD_TIE).

Replicated weights (58 MB int8 per GPU) remain the default design: the
per-step exchange is a latency-bound collective on a step that is already
device-bound at N = 1280 (DESIGN.md section 7 has the measurement)."""

from __future__ import annotations

import torch

from . import _dev, _lib
from .errors import ConfigError

FLAG_SHARD_TIE = 8
TILE = 192   # shard boundaries on the fused kernel's token tiles (vocab_topk.cu VT_BN)


def shard_bounds(V: int, G: int) -> list:
    """Contiguous token ranges [lo, hi) of G shards, tile-aligned, covering V."""
    if G < 1 or G > 16:
        raise ConfigError("1 <= shards <= 16")
    per = -(-V // G)
    per = -(-per // TILE) * TILE
    out = []
    for g in range(G):
        lo, hi = min(V, g * per), min(V, (g + 1) * per)
        out.append((lo, hi))
    return out


def part_bytes() -> int:
    return int(_lib.load().qnmt_vocab_shard_part_bytes())


def shard_partials(X, x_scales, row_seg, W, w_scale, bias, lo: int, hi: int, out=None, scratch=None):
    """The shard [lo, hi) of the vocabulary: [N] partials (uint8 [N, 80]).  X: int8
    [N][K] codes (K-major), W: int8 [V][K] codes (the full matrix or any view
    containing rows lo..hi-1 at their global offsets), w_scale: device f32[1]."""
    N, K = X.shape
    Vs = hi - lo
    if out is None:
        out = torch.empty((N, part_bytes()), dtype=torch.uint8, device=X.device)
    if N == 0:
        return out
    if Vs <= 0:
        raise ConfigError("empty vocabulary shard")
    if scratch is None:
        scratch = torch.empty(int(_lib.load().qnmt_vocab_candidates_scratch(N, Vs)), dtype=torch.uint8,
                              device=X.device)
    f = _dev.reset_flag()
    Wp = W.data_ptr() + lo * _dev.ld(W)
    bp = bias.data_ptr() + 4 * lo if bias is not None else None
    _lib.call("qnmt_vocab_shard_partials", X.data_ptr(), N, _dev.ld(X), x_scales.data_ptr(), _dev.ptr(row_seg), Wp,
              Vs, K, _dev.ld(W), w_scale.data_ptr(), max(Vs, 1 << 30), bp, lo, scratch.data_ptr(), out.data_ptr(),
              f.data_ptr(), _dev.stream_ptr())
    _dev.raise_flag(f)
    return out


def combine(parts, N: int, live, k: int):
    """parts: uint8 [G * N, 80] (shard-major) -> (cand_score f64 [N][k], cand_tok i32
    [N][k], tie flag)."""
    G = parts.shape[0] // max(N, 1)
    cs = torch.empty((N, k), dtype=torch.float64, device=parts.device)
    ct = torch.empty((N, k), dtype=torch.int32, device=parts.device)
    f = _dev.reset_flag()
    _lib.call("qnmt_vocab_shard_combine", parts.data_ptr(), G, N, _dev.ptr(live), k, cs.data_ptr(), ct.data_ptr(),
              f.data_ptr(), _dev.stream_ptr())
    tie = bool((f[0] & FLAG_SHARD_TIE).item())
    _dev.raise_flag(f)
    return cs, ct, tie


def candidates(X, x_scales, row_seg, W, w_scale, bias, live, k: int, shards: int = 1, group=None):
    """Beam candidates of the vocabulary step with W_vocab sharded.

    ``group`` None: ``shards`` slices emulated one after another on this GPU
    (the partial / combine arithmetic of the multi-GPU path, for parity).
    ``group`` a torch.distributed process group (NCCL): this rank computes the
    shard ``group.rank()`` of ``group.size()``, all-gathers the partials and
    combines them (every rank obtains the same candidates).  A step whose
    union may miss a tied token is recomputed unsharded."""
    import torch.distributed as dist
    N = X.shape[0]
    V = W.shape[0]
    if group is None:
        bounds = shard_bounds(V, shards)
        parts = torch.empty((len(bounds) * N, part_bytes()), dtype=torch.uint8, device=X.device)
        for g, (lo, hi) in enumerate(bounds):
            if hi > lo:
                shard_partials(X, x_scales, row_seg, W, w_scale, bias, lo, hi, out=parts[g * N:(g + 1) * N])
            else:
                parts[g * N:(g + 1) * N].zero_()
    else:
        G, r = dist.get_world_size(group), dist.get_rank(group)
        lo, hi = shard_bounds(V, G)[r]
        mine = torch.zeros((N, part_bytes()), dtype=torch.uint8, device=X.device)
        if hi > lo:
            shard_partials(X, x_scales, row_seg, W, w_scale, bias, lo, hi, out=mine)
        parts = torch.empty((G * N, part_bytes()), dtype=torch.uint8, device=X.device)
        dist.all_gather_into_tensor(parts, mine, group=group)
    cs, ct, tie = combine(parts, N, live, k)
    if tie:   # rare f32 score ties at the list boundary: the unsharded fused path
        return unsharded(X, x_scales, row_seg, W, w_scale, bias, live, k)
    return cs, ct


def unsharded(X, x_scales, row_seg, W, w_scale, bias, live, k: int):
    """qnmt_vocab_candidates over the whole vocabulary (the replicated design)."""
    N, K = X.shape
    V = W.shape[0]
    cs = torch.empty((N, k), dtype=torch.float64, device=X.device)
    ct = torch.empty((N, k), dtype=torch.int32, device=X.device)
    scratch = torch.empty(int(_lib.load().qnmt_vocab_candidates_scratch(N, V)), dtype=torch.uint8, device=X.device)
    f = _dev.reset_flag()
    _lib.call("qnmt_vocab_candidates", X.data_ptr(), N, _dev.ld(X), x_scales.data_ptr(), _dev.ptr(row_seg),
              W.data_ptr(), V, K, _dev.ld(W), w_scale.data_ptr(), V, _dev.ptr(bias), _dev.ptr(live), k,
              scratch.data_ptr(), cs.data_ptr(), ct.data_ptr(), f.data_ptr(), _dev.stream_ptr())
    _dev.raise_flag(f)
    return cs, ct
