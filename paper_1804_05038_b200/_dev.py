"""Device plumbing: torch owns device memory and streams; kernels are ours."""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib, errors

_tls = threading.local()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise errors.DeviceError("a CUDA device is required (the B200 path has no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ld(t) -> int:
    """Row stride of a row-major 2-D tensor (torch reports stride 1 for size-1 dims)."""
    assert t.dim() == 2 and (t.shape[1] <= 1 or t.stride(1) == 1)
    return t.stride(0) if t.shape[0] > 1 else max(1, t.shape[1])


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def flag() -> torch.Tensor:
    """Per-thread sticky device error flag (int32)."""
    dev = require_cuda()
    f = getattr(_tls, "flag", None)
    if f is None or f.device != dev:
        f = torch.zeros(4, dtype=torch.int32, device=dev)
        _tls.flag = f
    return f


def reset_flag() -> torch.Tensor:
    f = flag()
    f.zero_()
    return f


def raise_flag(f: torch.Tensor, invalid_msg="cannot quantize non-finite values",
               numeric_msg="activations contain non-finite values", vocab_msg="token id outside the vocabulary"):
    v = int(f[0].item())   # synchronises, as the reference raises synchronously
    if v & _lib.FLAG_VOCAB:
        raise errors.VocabError(vocab_msg)
    if v & _lib.FLAG_INVALID:
        raise errors.InvalidInputError(invalid_msg)
    if v & _lib.FLAG_NUMERIC:
        raise errors.NumericError(numeric_msg)


def to_device(x, dtype=torch.float32) -> torch.Tensor:
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype)
    a = np.ascontiguousarray(x)
    if not a.flags.writeable:   # e.g. load_model's read-only views of the file bytes
        a = a.copy()
    return torch.from_numpy(a).to(device=dev, dtype=dtype)


def kmajor(x, dtype=torch.float32) -> torch.Tensor:
    """[features, P] (numpy or torch, any strides) -> contiguous device [P][features]."""
    return to_device(x, dtype).t().contiguous()


def is_numpy(x) -> bool:
    return isinstance(x, np.ndarray)
