"""ctypes binding of ``_lib/libqnmt_b200.so`` (the C ABI of include/qnmt_b200.h).

There is deliberately no fallback: if the shared library is missing, or no
CUDA device is present when a kernel is requested, the call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

LIB_PATH = os.environ.get("QNMT_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                            "libqnmt_b200.so")   # (override: A/B builds)

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
F32 = C.c_float
F64 = C.c_double

# name -> (restype, argtypes); mirrors include/qnmt_b200.h
SIGNATURES = {
    "qnmt_abi_version": (I32, []),
    "qnmt_last_error": (C.c_char_p, []),
    "qnmt_device_sync": (I32, []),
    "qnmt_quantize": (I32, [P, I64, I64, I64, P, I32, P, I64, P, P, I32, P, P]),
    "qnmt_dequantize": (I32, [P, I64, F32, P, P]),
    "qnmt_gemm_i8": (I32, [P, I64, I64, I64, P, I64, P, I64, I64, P, P, P, P, I64, P, I32, P]),
    "qnmt_gru_gates": (I32, [P, I64, P, P, I64, P, I64, I64, I64, P, P, P, P]),
    "qnmt_gru_combine": (I32, [P, I64, P, P, I64, P, P, I64, I64, I64, P, I64, P, I64, P, P, P]),
    "qnmt_tanh": (I32, [P, I64, I64, I64, P, I64, P, P]),
    "qnmt_attention": (I32, [P, I64, I64, P, P, I32, P, P, P, P, P, P, I32, I64, I64, P, P, P, I64, P, I64, P, P, P]),
    "qnmt_attention_exp": (I32, [P, I64, P, P]),
    "qnmt_set_att_exp": (I32, [I32]),
    "qnmt_set_att_fixcap": (I32, [I32]),
    "qnmt_set_att_ctx": (I32, [I32]),
    "qnmt_set_att_fused_scale": (I32, [I32]),
    "qnmt_set_att_score8": (I32, [I32]),
    "qnmt_set_tc_split": (I32, [I32]),
    "qnmt_linear_i8": (I32, [P, I64, I64, I64, P, I64, P, I64, I64, P, P, I64, P, I64, P, P, I32, P, P]),
    "qnmt_attention_stats": (I32, [P, P, P, I32, I64, P, P]),
    "qnmt_attention_f32": (I32, [P, I64, I64, P, P, I32, P, P, P, P, I32, I64, I64, P, P, I64, P, I64, P, P, P]),
    "qnmt_gemm_f32": (I32, [P, I64, I64, I64, P, I64, I64, P, P, I64, I32, P]),
    "qnmt_log_softmax": (I32, [P, I64, I64, I64, P, I64, P, P]),
    "qnmt_topk_candidates": (I32, [P, I64, I64, I64, P, I32, P, P, P, P]),
    "qnmt_vocab_candidates": (I32, [P, I64, I64, P, P, P, I64, I64, I64, P, I64, P, P, I32, P, P, P, P, P]),
    "qnmt_vocab_candidates_scratch": (I64, [I64, I64]),
    "qnmt_vocab_shard_part_bytes": (I64, []),
    "qnmt_vocab_shard_partials": (I32, [P, I64, I64, P, P, P, I64, I64, I64, P, I64, P, I64, P, P, P, P]),
    "qnmt_vocab_shard_combine": (I32, [P, I32, I64, P, I32, P, P, P, P]),
    "qnmt_embed_gather": (I32, [P, I64, I64, P, I64, P, I64, P, P]),
    "qnmt_model_create": (I32, [P, P, I32, P]),
    "qnmt_model_create_f32": (I32, [P, P, I32, P]),
    "qnmt_model_destroy": (I32, [P]),
    "qnmt_engine_create": (I32, [P, I32, I32, I32, P]),
    "qnmt_engine_destroy": (I32, [P]),
    "qnmt_engine_bytes": (C.c_size_t, [P]),
    "qnmt_engine_check_canaries": (I64, [P, P]),
    "qnmt_translate_batch": (I32, [P, P, P, I32, I32, F64, P, I32, P, P, P]),
    "qnmt_translate_ensemble": (I32, [P, I32, P, P, I32, I32, F64, P, I32, P, P, P]),
    "qnmt_encode_batch": (I32, [P, P, P, I32, P, P, P, P]),
    "qnmt_decoder_step": (I32, [P, I64, P, I32, P, P, P, P, P, P, P, I32, P, P, P, P, I64, P]),
    "qnmt_decode_batch_device": (I32, [P, P, P, I32, I32, F64, P]),
    "qnmt_fetch_results": (I32, [P, P, I32, P, P, P]),
    "qnmt_last_d2h_bytes": (I64, [P]),
    "qnmt_last_h2d_bytes": (I64, [P]),
    "qnmt_kernel_launches": (I64, []),
    "qnmt_set_gemm_impl": (I32, [I32]),
    "qnmt_set_tc_pair": (I32, [I32]),
    "qnmt_set_gate_epi": (I32, [I32]),
    "qnmt_set_gru_epi_bn": (I32, [I32, I32]),
    "qnmt_set_greedy1": (I32, [I32]),
    "qnmt_set_topk_exact": (I32, [I32]),
    "qnmt_set_vocab_fused": (I32, [I32]),
    "qnmt_engine_profile": (I32, [P, I32]),
    "qnmt_engine_set_graphs": (I32, [P, I32]),
    "qnmt_engine_stamps": (I32, [P, I32]),
    "qnmt_engine_stamps_read": (I32, [P, P, I32, P]),
    "qnmt_engine_profile_read": (I32, [P, P, P, P, P]),
}

QNMT_OK, ERR_SHAPE, ERR_INVALID, ERR_NUMERIC, ERR_VOCAB, ERR_CONFIG, ERR_EMPTY, ERR_CUDA = range(8)
FLAG_NUMERIC, FLAG_INVALID, FLAG_VOCAB = 1, 2, 4
GEMM_ACCUMULATE = 1
GEMM_W_STATIC = 2
INT32_SAFE_K = 131_000

_EXC = {
    ERR_SHAPE: errors.ShapeError,
    ERR_INVALID: errors.InvalidInputError,
    ERR_NUMERIC: errors.NumericError,
    ERR_VOCAB: errors.VocabError,
    ERR_CONFIG: errors.ConfigError,
    ERR_EMPTY: errors.EmptyInputError,
    ERR_CUDA: errors.DeviceError,
}

_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load the shared library (no GPU needed just to load it)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise errors.DeviceError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1804_05038_b200._build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str):
    if rc != QNMT_OK:
        msg = load().qnmt_last_error().decode(errors="replace")
        raise _EXC.get(rc, errors.DeviceError)(f"{what}: {msg}")


def call(name: str, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc


def exported_symbols() -> list:
    return list(SIGNATURES)
