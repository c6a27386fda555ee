"""B200-native int8 decode path of arXiv 1804.05038 (drop-in for the ``qnmt`` hot path).

The reference package's Python names (``qnmt/__init__.py:11-48``) are kept:
quantize / quantize_activations / dequantize / qgemm / qgemm_panel,
LinearOp / gru_step / attend / Network.encode / decoder_step,
DecodeConfig / translate, plus the bulk entry :func:`translate_batch`.
All arithmetic runs in hand-written sm_100a CUDA kernels behind the C ABI of
``include/qnmt_b200.h`` (``_lib/libqnmt_b200.so``); there is no CPU fallback.
"""

__version__ = "0.1.0"

from . import errors
from .bleu import bleu
from .decoder import (
    BeamHypothesis,
    DecodeConfig,
    ParityReport,
    bpe_merge,
    compare_precisions,
    edit_distance,
    shard_batches,
    translate,
    translate_batch,
)
from .engine import Engine
from .layers import (
    AttentionNet,
    DecoderState,
    EncoderStates,
    GruCell,
    LinearOp,
    Network,
    OutputNet,
    attend,
    build_network,
    gru_step,
)
from .model import (
    Dims,
    Float32Model,
    ModelParams,
    QuantizedModel,
    generate_model,
    load_model,
    load_quantized,
    quantize_model,
    replicate,
    save_model,
    synthetic_model,
    tensor_specs,
    to_device_f32,
)
from .qmath import (
    INT8_MAX,
    INT32_SAFE_K,
    QuantizationStats,
    QuantizedMatrix,
    dequantize,
    gemm_f32,
    gemm_f32_blocked,
    qgemm,
    qgemm_panel,
    quantize,
    quantize_activations,
)

__all__ = [
    "AttentionNet", "BeamHypothesis", "DecodeConfig", "DecoderState", "Dims", "EncoderStates",
    "Engine", "Float32Model", "GruCell", "ParityReport", "bleu", "compare_precisions", "edit_distance",
    "gemm_f32", "gemm_f32_blocked", "to_device_f32", "INT8_MAX", "INT32_SAFE_K", "LinearOp", "ModelParams", "Network",
    "OutputNet", "QuantizationStats", "QuantizedMatrix", "QuantizedModel", "attend", "bpe_merge",
    "build_network", "dequantize", "errors", "generate_model", "gru_step", "load_model", "load_quantized", "qgemm", "qgemm_panel",
    "quantize", "quantize_activations", "quantize_model", "save_model", "synthetic_model", "tensor_specs",
    "translate", "translate_batch", "shard_batches", "replicate",
]
