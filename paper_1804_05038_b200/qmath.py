"""8-bit symmetric quantization and integer GEMMs on B200 (drop-in for qnmt.qmath).

Same names and semantics as the reference ``qmath.py``:

* :class:`QuantizedMatrix` -- int8 codes in [-127, 127] plus a positive f32
  scale (qmath.py:59-90).  ``data`` keeps the caller's array type: numpy in ->
  numpy out (a device copy is cached), torch CUDA tensor in -> tensor out.
* :func:`quantize` / :func:`quantize_activations` -- scale = 127/max|x|,
  round half away from zero in f32 (qmath.py:119-182) -- kernel ``K1``
  (csrc/quantize.cu).
* :func:`qgemm` / :func:`qgemm_panel` -- exact integer products with the f64
  dequantization epilogue (qmath.py:379-427) -- kernels ``K2``/``K3``
  (csrc/gemm_dp4a.cu, csrc/gemm_tcgen05.cu).  Both schedules are one device
  code path, so they are bit-identical by construction.

Nothing here computes on the CPU: every call launches the CUDA library and
raises if it is unavailable.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .errors import InvalidInputError, NumericError, ShapeError

INT8_MAX = 127
INT32_SAFE_K = _lib.INT32_SAFE_K


class QuantizedMatrix:
    """Signed 8-bit matrix plus the scale (quantized units per real unit)."""

    def __init__(self, data, scale: float):
        if isinstance(data, np.ndarray):
            ok = data.dtype == np.int8 and data.ndim == 2
        elif isinstance(data, torch.Tensor):
            ok = data.dtype == torch.int8 and data.dim() == 2
        else:
            ok = False
        if not ok:
            raise InvalidInputError("QuantizedMatrix requires a 2-D int8 array")
        scale = float(scale)
        if not (scale > 0 and np.isfinite(scale)):
            raise InvalidInputError(f"scale must be positive and finite, got {scale}")
        self.data = data
        self.scale = scale
        self._dev = data.contiguous() if isinstance(data, torch.Tensor) and data.is_cuda else None
        self._scale_dev = None
        self._shadow = None   # API parity with the reference's VNNI shadow (unused on GPU)

    @property
    def rows(self) -> int:
        return int(self.data.shape[0])

    @property
    def cols(self) -> int:
        return int(self.data.shape[1])

    def device_data(self) -> torch.Tensor:
        """Contiguous device int8 codes [rows][cols] (cached)."""
        if self._dev is None:
            self._dev = _dev.to_device(self.data, torch.int8).contiguous()
        return self._dev

    def device_scale(self) -> torch.Tensor:
        if self._scale_dev is None:
            self._scale_dev = torch.tensor([self.scale], dtype=torch.float32, device=_dev.require_cuda())
        return self._scale_dev

    def __repr__(self):
        return f"QuantizedMatrix(rows={self.rows}, cols={self.cols}, scale={self.scale!r})"


@dataclass
class QuantizationStats:
    """Round-trip error record for one quantized tensor (qmath.py:93-101)."""

    name: str
    scale: float
    max_abs: float
    rms_error: float
    max_error: float


def _as_f32_matrix(m, name):
    if isinstance(m, torch.Tensor):
        if m.dim() != 2 or m.shape[0] < 1 or m.shape[1] < 1:
            raise ShapeError(f"{name} must be a non-empty 2-D matrix, got shape {tuple(m.shape)}")
        return _dev.to_device(m).contiguous()
    m = np.asarray(m, dtype=np.float32)
    if m.ndim != 2 or m.shape[0] < 1 or m.shape[1] < 1:
        raise ShapeError(f"{name} must be a non-empty 2-D matrix, got shape {m.shape}")
    return _dev.to_device(m).contiguous()


def _quantize_dev(x: torch.Tensor, mode: int):
    """One-segment K1 over a contiguous device f32 matrix -> (codes, scale tensor)."""
    rows, cols = x.shape
    q = torch.empty((rows, cols), dtype=torch.int8, device=x.device)
    scales = torch.empty(1, dtype=torch.float32, device=x.device)
    bits = torch.empty(1, dtype=torch.int32, device=x.device)
    f = _dev.reset_flag()
    _lib.call("qnmt_quantize", x.data_ptr(), rows, cols, cols, None, 1, q.data_ptr(), cols,
              scales.data_ptr(), bits.data_ptr(), mode, f.data_ptr(), _dev.stream_ptr())
    return q, scales, f


def _wrap(codes: torch.Tensor, scale: float, like) -> QuantizedMatrix:
    if _dev.is_numpy(like) or not isinstance(like, torch.Tensor):
        qm = QuantizedMatrix(codes.cpu().numpy(), scale)
        qm._dev = codes
    else:
        qm = QuantizedMatrix(codes, scale)
    return qm


def quantize(m) -> QuantizedMatrix:
    """Quantize a float32 matrix to int8 codes in [-127, 127] (qmath.py:145-154).

    scale = 127 / max|m| (1.0 for an all-zero matrix); codes are
    round-to-nearest with ties away from zero, computed in float32.
    Non-finite input raises InvalidInputError.
    """
    x = _as_f32_matrix(m, "input")
    q, scales, f = _quantize_dev(x, 0)
    _dev.raise_flag(f, invalid_msg="cannot quantize non-finite values")
    qm = _wrap(q, float(scales.item()), m)
    qm._scale_dev = scales
    return qm


def quantize_activations(x) -> QuantizedMatrix:
    """Per-call activation quantization (qmath.py:172-182); non-finite -> NumericError."""
    if isinstance(x, torch.Tensor):
        xd = _dev.to_device(x).contiguous()
    else:
        xd = _dev.to_device(np.asarray(x, dtype=np.float32)).contiguous()
    if xd.dim() != 2:
        raise ShapeError(f"activations must be 2-D, got shape {tuple(xd.shape)}")
    q, scales, f = _quantize_dev(xd, 1)
    _dev.raise_flag(f, numeric_msg="activations contain non-finite values")
    qm = _wrap(q, float(scales.item()), x)
    qm._scale_dev = scales
    return qm


def dequantize(q: QuantizedMatrix):
    """Reconstruct float32 values as code / scale (qmath.py:185-187)."""
    d = q.device_data()
    y = torch.empty(d.shape, dtype=torch.float32, device=d.device)
    _lib.call("qnmt_dequantize", d.data_ptr(), d.numel(), float(np.float32(q.scale)), y.data_ptr(),
              _dev.stream_ptr())
    return y.cpu().numpy() if _dev.is_numpy(q.data) else y


def quantization_stats(name: str, m, q: QuantizedMatrix) -> QuantizationStats:
    """qmath.py:190-198 (diagnostic, not on the decode path)."""
    md = _dev.to_device(m).double()
    err = md - _dev.to_device(dequantize(q)).double()
    return QuantizationStats(name=name, scale=q.scale, max_abs=float(md.abs().max()),
                             rms_error=float(torch.sqrt(torch.mean(err * err))),
                             max_error=float(err.abs().max()))


def _check_pair(a, b):
    if not isinstance(a, QuantizedMatrix) or not isinstance(b, QuantizedMatrix):
        raise InvalidInputError("qgemm operands must be QuantizedMatrix")
    if a.cols != b.rows:
        raise ShapeError(f"inner dimensions disagree: {a.rows}x{a.cols} @ {b.rows}x{b.cols}")
    if b.cols < 1:
        raise ShapeError("right-hand operand must have at least one column")


def gemm_kmajor(W: torch.Tensor, w_scales: torch.Tensor, rows_per_scale: int, X: torch.Tensor,
                x_scales: torch.Tensor, col_seg=None, bias=None, Y=None, accumulate=False,
                acc_out=None, w_static=False) -> torch.Tensor:
    """Device GEMM in kernel layout: Y[N][M] from W[M][K] and K-major X[N][K].
    ``w_static``: W is a model weight (not produced by the preceding kernels), so
    the GEMV may prefetch it before its programmatic-dependent-launch wait."""
    M, K = W.shape
    N = X.shape[0]
    if X.shape[1] != K:
        raise ShapeError(f"inner dimensions disagree: {M}x{K} @ {X.shape[1]}x{N}")
    if Y is None and acc_out is None:
        Y = torch.empty((N, M), dtype=torch.float32, device=W.device)
    _lib.call("qnmt_gemm_i8", W.data_ptr(), M, K, _dev.ld(W), w_scales.data_ptr(), rows_per_scale,
              X.data_ptr(), N, _dev.ld(X), x_scales.data_ptr(), _dev.ptr(col_seg), _dev.ptr(bias),
              _dev.ptr(Y), _dev.ld(Y) if Y is not None else M, _dev.ptr(acc_out),
              (_lib.GEMM_ACCUMULATE if accumulate else 0) | (_lib.GEMM_W_STATIC if w_static else 0),
              _dev.stream_ptr())
    return Y


def gemm_f32_kmajor(W: torch.Tensor, X: torch.Tensor, bias=None, Y=None, accumulate=False) -> torch.Tensor:
    """fp32-path product in kernel layout: Y[N][M] = fl32(W[M][K] . X[N][K]) (fp64
    evaluation, csrc/gemm_f32.cu) (+ bias) (+ Y)."""
    M, K = W.shape
    N = X.shape[0]
    if X.shape[1] != K:
        raise ShapeError(f"inner dimensions disagree: {M}x{K} @ {X.shape[1]}x{N}")
    if Y is None:
        Y = torch.empty((N, M), dtype=torch.float32, device=W.device)
    _lib.call("qnmt_gemm_f32", W.data_ptr(), M, K, _dev.ld(W), X.data_ptr(), N, _dev.ld(X), _dev.ptr(bias),
              Y.data_ptr(), _dev.ld(Y), _lib.GEMM_ACCUMULATE if accumulate else 0, _dev.stream_ptr())
    return Y


def gemm_f32(a, b):
    """Standard float32 product (qmath.py:434-440), on the device: fp64-evaluated,
    rounded once (numpy in -> numpy out)."""
    for name, m in (("a", a), ("b", b)):
        if len(np.shape(m)) != 2 or min(np.shape(m)) < 1:
            raise ShapeError(f"{name} must be a non-empty 2-D matrix, got shape {tuple(np.shape(m))}")
    if np.shape(a)[1] != np.shape(b)[0]:
        raise ShapeError(f"inner dimensions disagree: {tuple(np.shape(a))} @ {tuple(np.shape(b))}")
    W = _dev.to_device(a).contiguous()
    X = _dev.kmajor(b)
    Y = gemm_f32_kmajor(W, X).t()
    return Y.contiguous().cpu().numpy() if _dev.is_numpy(a) or _dev.is_numpy(b) else Y


def gemm_f32_blocked(a, b):
    """The reference's cache-blocked schedule (qmath.py:462-474) exists to show that
    blocking buys nothing on narrow panels; it equals :func:`gemm_f32` up to
    reassociation.  The device has one fp64-evaluated schedule, so this is that call."""
    return gemm_f32(a, b)


def qgemm(a: QuantizedMatrix, b: QuantizedMatrix):
    """Quantized product with exact integer accumulation, emitted as float32.

    Entry (i, j) is (sum_k a_ik * b_kj) / (a.scale * b.scale) (qmath.py:384-397);
    int64 accumulation when K exceeds INT32_SAFE_K.
    """
    _check_pair(a, b)
    W = a.device_data()
    X = b.device_data().t().contiguous()      # [P][K]
    Y = gemm_kmajor(W, a.device_scale(), a.rows, X, b.device_scale())
    out = Y.t()
    if _dev.is_numpy(a.data) or _dev.is_numpy(b.data):
        return out.contiguous().cpu().numpy()
    return out


def qgemm_panel(a: QuantizedMatrix, b: QuantizedMatrix, p_small: bool = True):
    """Panel-scheduled product (qmath.py:400-427); bit-identical to :func:`qgemm`."""
    return qgemm(a, b)


def qgemm_acc(a: QuantizedMatrix, b: QuantizedMatrix) -> torch.Tensor:
    """Raw int64 accumulators [M, P] (device) -- for parity tests of the int path."""
    _check_pair(a, b)
    W = a.device_data()
    X = b.device_data().t().contiguous()
    acc = torch.empty((X.shape[0], W.shape[0]), dtype=torch.int64, device=W.device)
    gemm_kmajor(W, a.device_scale(), a.rows, X, b.device_scale(), acc_out=acc)
    return acc.t()
