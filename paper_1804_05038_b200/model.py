"""Parameter containers, the QNMT model file, synthetic models and on-device
weight quantization.

Mirrors the reference ``model.py``: :class:`Dims` (:42-52), the canonical
tensor directory :func:`tensor_specs` (:151-177), :class:`ModelParams`
(fp32), :class:`QuantizedModel` (int8 codes + one f32 scale per tensor,
embeddings and biases fp32, :394-437), the seeded generators, and the binary
format (:1-17, ``save_model`` :275-310, ``load_model`` :313-387).

:func:`load_quantized` is the B200 loader: it validates the file on the host,
moves the whole payload to HBM in one copy and quantizes every weight matrix
there, so no per-tensor host work sits between the file and the engine.

B200 layout: :func:`quantize_model` uploads the fp32 tensors once, quantizes
every weight matrix with the device K1 kernel (bit-identical to the
reference's ``quantize``), and additionally packs the per-gate GRU tensors
into the stacked form the fused kernels consume (``WX = [wz; wr; wc]`` with
three row-block scales, ``UZR = [uz; ur]`` with two, ``UC``).  The packed
device tensors are referenced by the C engine handle (``qnmt_model_create``).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .errors import FormatError, ParameterError, SchemaError
from .qmath import QuantizedMatrix, quantization_stats, quantize

MAGIC = b"QNMT"
VERSION = 1
PAD_ID, UNK_ID, EOS_ID = 0, 1, 2
PAD_TOKEN, UNK_TOKEN, EOS_TOKEN = "<pad>", "<unk>", "</s>"
DEFAULT_WEIGHT_SCALE = 0.08
GRU_FIELDS = ("wz", "uz", "bz", "wr", "ur", "br", "wc", "uc", "bc")
CELLS = ("enc_fwd", "enc_bwd", "dec_r", "dec_q")


@dataclass
class Dims:
    src_vocab: int
    tgt_vocab: int
    embed: int
    hidden: int
    attn: int
    readout: int

    def as_dict(self) -> dict:
        return dict(self.__dict__)


def tensor_specs(dims: Dims) -> list:
    """Canonical (name, shape) directory; defines serialization order (model.py:151-177)."""
    specs = [("src_embed", (dims.src_vocab, dims.embed)), ("tgt_embed", (dims.tgt_vocab, dims.embed))]
    h = dims.hidden
    for cell, in_dim in (("enc_fwd", dims.embed), ("enc_bwd", dims.embed),
                         ("dec_r", dims.embed), ("dec_q", 2 * h)):
        shapes = {"wz": (h, in_dim), "uz": (h, h), "bz": (h,), "wr": (h, in_dim), "ur": (h, h),
                  "br": (h,), "wc": (h, in_dim), "uc": (h, h), "bc": (h,)}
        specs.extend((f"{cell}.{f}", shapes[f]) for f in GRU_FIELDS)
    specs.extend([
        ("attn.w_enc", (dims.attn, 2 * h)), ("attn.b_enc", (dims.attn,)),
        ("attn.u_state", (dims.attn, h)), ("attn.v", (1, dims.attn)),
        ("out.w_state", (dims.readout, h)), ("out.w_embed", (dims.readout, dims.embed)),
        ("out.w_ctx", (dims.readout, 2 * h)), ("out.b_readout", (dims.readout,)),
        ("out.w_vocab", (dims.tgt_vocab, dims.readout)), ("out.b_vocab", (dims.tgt_vocab,)),
        ("s0.w", (h, h)), ("s0.b", (h,)),
    ])
    return specs


def synthetic_vocab(size: int) -> list:
    """model.py:230-231: reserved pad/unk/eos then w0001 ..."""
    return [PAD_TOKEN, UNK_TOKEN, EOS_TOKEN] + [f"w{i:04d}" for i in range(1, size - 2)]


@dataclass(eq=False)
class ModelParams:
    """All trained tensors in float32 (numpy, host), keyed by tensor_specs names."""

    dims: Dims
    tensors: dict
    src_tokens: list
    tgt_tokens: list
    s0_mode: str = "transform"
    attention_query: str = "current"
    precision = "fp32"

    def __post_init__(self):
        self._src_index = None

    def src_ids(self, tokens) -> np.ndarray:
        """Map source tokens to ids; unknown tokens become UNK (model.py:110-115)."""
        if self._src_index is None:
            self._src_index = {t: i for i, t in enumerate(self.src_tokens)}
        idx = self._src_index
        return np.array([idx.get(t, UNK_ID) for t in tokens], dtype=np.int64)

    def tgt_token(self, token_id: int) -> str:
        return self.tgt_tokens[token_id]


def _check_dims(dims: Dims):
    for name, value in dims.as_dict().items():
        if value < 1:
            raise ParameterError(f"{name} must be >= 1, got {value}")
    if dims.src_vocab < 3 or dims.tgt_vocab < 3:
        raise ParameterError("vocabularies must cover the reserved pad/unk/eos ids")


def synthetic_model(dims: Dims, seed: int, weight_std: float = 0.05, bias_std: float = 0.0,
                    eos_bias: float = 0.0, s0_mode: str = "transform",
                    attention_query: str = "current") -> ModelParams:
    """BASELINE.json recipe: numpy default_rng(seed); every
    2-D tensor ~ N(0, weight_std) cast to f32 in tensor_specs order; biases 0
    (or N(0, bias_std) drawn after all weights); ``eos_bias`` added to
    b_vocab[EOS] for test models that terminate early."""
    _check_dims(dims)
    rng = np.random.default_rng(seed)
    t = {}
    specs = tensor_specs(dims)
    for name, shape in specs:
        if len(shape) == 2:
            t[name] = rng.normal(0.0, weight_std, shape).astype(np.float32)
    for name, shape in specs:
        if len(shape) == 1:
            t[name] = (rng.normal(0.0, bias_std, shape).astype(np.float32) if bias_std > 0
                       else np.zeros(shape, dtype=np.float32))
    if eos_bias:
        t["out.b_vocab"][EOS_ID] += np.float32(eos_bias)
    return ModelParams(dims, t, synthetic_vocab(dims.src_vocab), synthetic_vocab(dims.tgt_vocab),
                       s0_mode, attention_query)


def generate_model(src_vocab: int, tgt_vocab: int, embed: int, hidden: int, seed: int,
                   attn: int | None = None, readout: int | None = None,
                   weight_scale: float = DEFAULT_WEIGHT_SCALE, s0_mode: str = "transform",
                   attention_query: str = "current") -> ModelParams:
    """model.py:234-269: PCG64(seed), uniform [-weight_scale, weight_scale) f32 in spec order."""
    dims = Dims(src_vocab, tgt_vocab, embed, hidden, attn=attn or hidden, readout=readout or embed)
    _check_dims(dims)
    if not (0 < weight_scale < 16):
        raise ParameterError(f"weight_scale out of range: {weight_scale}")
    total = sum(int(np.prod(s)) for _, s in tensor_specs(dims))
    if total > 2 ** 31:
        raise ParameterError(f"model of {total} parameters exceeds the supported size")
    rng = np.random.Generator(np.random.PCG64(seed))
    ws = np.float32(weight_scale)
    t = {}
    for name, shape in tensor_specs(dims):
        u = rng.random(shape, dtype=np.float32)
        t[name] = (u * np.float32(2.0) - np.float32(1.0)) * ws
    return ModelParams(dims, t, synthetic_vocab(src_vocab), synthetic_vocab(tgt_vocab), s0_mode,
                       attention_query)


@dataclass(eq=False)
class QuantizedModel:
    """Device-resident int8 model: ``q[name]`` QuantizedMatrix (device codes),
    ``f[name]`` f32 device tensors (embeddings, biases), packed GRU stacks,
    and the C model handle for the engine."""

    dims: Dims
    q: dict
    f: dict
    src_tokens: list
    tgt_tokens: list
    s0_mode: str = "transform"
    attention_query: str = "current"
    stats: dict = field(default_factory=dict)
    precision = "int8"

    def __post_init__(self):
        self._src_index = None
        self._handle = None
        self._keep = []

    src_ids = ModelParams.src_ids
    tgt_token = ModelParams.tgt_token

    # -- packed tensors for the engine --------------------------------------
    def packed_cell(self, cell: str):
        """(WX [3H,in] int8, WX scales [3], BX [3H], UZR [2H,H], UZR scales [2], UC, UC scale [1])."""
        key = f"_packed_{cell}"
        if not hasattr(self, key):
            q, f = self.q, self.f
            wx = torch.cat([q[f"{cell}.w{g}"].device_data() for g in "zrc"]).contiguous()
            wxs = torch.cat([q[f"{cell}.w{g}"].device_scale() for g in "zrc"]).contiguous()
            bx = torch.cat([f[f"{cell}.b{g}"] for g in "zrc"]).contiguous()
            uzr = torch.cat([q[f"{cell}.u{g}"].device_data() for g in "zr"]).contiguous()
            uzrs = torch.cat([q[f"{cell}.u{g}"].device_scale() for g in "zr"]).contiguous()
            uc = q[f"{cell}.uc"].device_data()
            ucs = q[f"{cell}.uc"].device_scale()
            setattr(self, key, (wx, wxs, bx, uzr, uzrs, uc, ucs))
        return getattr(self, key)

    def handle(self):
        """C ``qnmt_model*`` (created once; tensors kept alive by this object)."""
        if self._handle is None:
            ptrs = [0] * 50
            keep = []

            def put(i, t):
                keep.append(t)
                ptrs[i] = t.data_ptr()

            put(0, self.f["src_embed"])
            put(1, self.f["tgt_embed"])
            for c, cell in enumerate(CELLS):
                for j, t in enumerate(self.packed_cell(cell)):
                    put(2 + 7 * c + j, t)
            q, f = self.q, self.f
            put(30, q["attn.w_enc"].device_data()); put(31, q["attn.w_enc"].device_scale())
            put(32, f["attn.b_enc"])
            put(33, q["attn.u_state"].device_data()); put(34, q["attn.u_state"].device_scale())
            put(35, q["attn.v"].device_data()); put(36, q["attn.v"].device_scale())
            put(37, q["out.w_state"].device_data()); put(38, q["out.w_state"].device_scale())
            put(39, f["out.b_readout"])
            put(40, q["out.w_embed"].device_data()); put(41, q["out.w_embed"].device_scale())
            put(42, q["out.w_ctx"].device_data()); put(43, q["out.w_ctx"].device_scale())
            put(44, q["out.w_vocab"].device_data()); put(45, q["out.w_vocab"].device_scale())
            put(46, f["out.b_vocab"])
            put(47, q["s0.w"].device_data()); put(48, q["s0.w"].device_scale())
            put(49, f["s0.b"])
            d = self.dims
            dims = (C.c_int32 * 8)(d.src_vocab, d.tgt_vocab, d.embed, d.hidden, d.attn, d.readout,
                                   1 if self.s0_mode == "zero" else 0,
                                   1 if self.attention_query == "previous" else 0)
            arr = (C.c_void_p * 50)(*ptrs)
            h = C.c_void_p()
            _lib.call("qnmt_model_create", C.cast(dims, C.c_void_p), C.cast(arr, C.c_void_p), 50,
                      C.byref(h))
            self._keep = keep
            self._handle = h
        return self._handle

    def __del__(self):
        try:
            if self._handle is not None:
                _lib.load().qnmt_model_destroy(self._handle)
        except Exception:
            pass


class Float32Model:
    """Device-resident fp32 model for the fp32 precision path:
    every tensor of ``tensor_specs`` as a device f32 tensor in ``f``, the GRU
    gates packed like the int8 model (``WX = [wz; wr; wc]``, ``UZR``, ``UC``), and
    a C model handle created with ``qnmt_model_create_f32``.  Built from (and
    cached on) a :class:`ModelParams` by :func:`to_device_f32`."""

    precision = "fp32"

    def __init__(self, params: ModelParams):
        self.dims = params.dims
        self.src_tokens, self.tgt_tokens = params.src_tokens, params.tgt_tokens
        self.s0_mode, self.attention_query = params.s0_mode, params.attention_query
        self._src_index = None
        self._handle = None
        self._keep = []
        self.f = {}
        for name, _ in tensor_specs(params.dims):
            arr = params.tensors[name]
            t = arr if isinstance(arr, torch.Tensor) else _dev.to_device(np.ascontiguousarray(arr, dtype=np.float32))
            self.f[name] = t.to(dtype=torch.float32).contiguous()

    src_ids = ModelParams.src_ids
    tgt_token = ModelParams.tgt_token

    def packed_cell(self, cell: str):
        """(WX [3H,in] f32, None, BX [3H], UZR [2H,H], None, UC, None) -- int8 layout without scales."""
        key = f"_packed_{cell}"
        if not hasattr(self, key):
            f = self.f
            wx = torch.cat([f[f"{cell}.w{g}"] for g in "zrc"]).contiguous()
            bx = torch.cat([f[f"{cell}.b{g}"] for g in "zrc"]).contiguous()
            uzr = torch.cat([f[f"{cell}.u{g}"] for g in "zr"]).contiguous()
            setattr(self, key, (wx, None, bx, uzr, None, f[f"{cell}.uc"], None))
        return getattr(self, key)

    def handle(self):
        if self._handle is None:
            ptrs = [0] * 50
            keep = []

            def put(i, t):
                if t is not None:
                    keep.append(t)
                    ptrs[i] = t.data_ptr()

            f = self.f
            put(0, f["src_embed"])
            put(1, f["tgt_embed"])
            for c, cell in enumerate(CELLS):
                for j, t in enumerate(self.packed_cell(cell)):
                    put(2 + 7 * c + j, t)
            for i, name in ((30, "attn.w_enc"), (32, "attn.b_enc"), (33, "attn.u_state"), (35, "attn.v"),
                            (37, "out.w_state"), (39, "out.b_readout"), (40, "out.w_embed"), (42, "out.w_ctx"),
                            (44, "out.w_vocab"), (46, "out.b_vocab"), (47, "s0.w"), (49, "s0.b")):
                put(i, f[name])
            d = self.dims
            dims = (C.c_int32 * 8)(d.src_vocab, d.tgt_vocab, d.embed, d.hidden, d.attn, d.readout,
                                   1 if self.s0_mode == "zero" else 0,
                                   1 if self.attention_query == "previous" else 0)
            arr = (C.c_void_p * 50)(*ptrs)
            h = C.c_void_p()
            _lib.call("qnmt_model_create_f32", C.cast(dims, C.c_void_p), C.cast(arr, C.c_void_p), 50, C.byref(h))
            self._keep = keep
            self._handle = h
        return self._handle

    def __del__(self):
        try:
            if self._handle is not None:
                _lib.load().qnmt_model_destroy(self._handle)
        except Exception:
            pass


def to_device_f32(params: ModelParams) -> Float32Model:
    """The fp32 device model of ``params`` (uploaded once, cached on ``params``)."""
    m = getattr(params, "_b200_f32", None)
    if m is None:
        m = Float32Model(params)
        params._b200_f32 = m
    return m


def _quantize_tensors(dims: Dims, tensors: dict, src_tokens, tgt_tokens, s0_mode, attention_query,
                      with_stats: bool) -> QuantizedModel:
    q, f, stats = {}, {}, {}
    for name, shape in tensor_specs(dims):
        arr = tensors[name]
        if isinstance(arr, torch.Tensor):
            dev = arr
        else:
            dev = _dev.to_device(np.ascontiguousarray(arr, dtype=np.float32))
        if len(shape) == 2 and name not in ("src_embed", "tgt_embed"):
            dev = dev.contiguous()
            qm = quantize(dev)
            q[name] = qm
            if with_stats:
                stats[name] = quantization_stats(name, dev, qm)
        else:   # own allocation (not a view of a loader buffer): 16-byte aligned rows for the fused kernels
            f[name] = dev.clone() if isinstance(arr, torch.Tensor) and arr._base is not None else dev.contiguous()
    return QuantizedModel(dims, q, f, src_tokens, tgt_tokens, s0_mode, attention_query, stats)


def replicate(qm: QuantizedModel, device) -> QuantizedModel:
    """The model's int8 codes, scales, biases and embeddings copied to another
    GPU (device-to-device, no re-quantization: codes and scales are identical).
    Cached on ``qm``; the model itself is returned for its own device.  Used by
    the sentence-sharded bulk path (``translate_batch(..., devices=...)``,
    SURVEY 8(e): weights replicated, sentences sharded, no collective)."""
    dev = torch.device("cuda", torch.device(device).index if not isinstance(device, int) else device)
    home = next(iter(qm.f.values())).device
    if dev == home:
        return qm
    reps = qm.__dict__.setdefault("_replicas", {})
    if dev.index not in reps:
        with torch.cuda.device(dev):
            q = {}
            for name, m in qm.q.items():
                r = QuantizedMatrix(m.device_data().to(dev), m.scale)
                r._scale_dev = m.device_scale().to(dev)
                q[name] = r
            f = {name: t.to(dev).contiguous() for name, t in qm.f.items()}
            torch.cuda.synchronize(dev)
        reps[dev.index] = QuantizedModel(qm.dims, q, f, qm.src_tokens, qm.tgt_tokens, qm.s0_mode,
                                         qm.attention_query, qm.stats)
    return reps[dev.index]


def quantize_model(params: ModelParams, with_stats: bool = False) -> QuantizedModel:
    """Quantize every weight matrix once on the device (model.py:394-437);
    biases and embeddings stay f32 (uploaded)."""
    return _quantize_tensors(params.dims, params.tensors, params.src_tokens, params.tgt_tokens,
                             params.s0_mode, params.attention_query, with_stats)


# ---------------------------------------------------------------------------
# QNMT model file (model.py:1-17): "QNMT", u32 version, u64 header length,
# JSON header, f32 payload (C order, spec order), 8-byte SHA-256 prefix of the
# payload.  Little-endian throughout.
# ---------------------------------------------------------------------------

_HEADER_KEYS = ("dims", "s0_mode", "attention_query", "source_vocab", "target_vocab",
                "payload_bytes", "tensors")


def _u(blob, lo, hi) -> int:
    return int.from_bytes(blob[lo:hi], "little")


def save_model(params: ModelParams, path: str) -> None:
    """Write the canonical byte-exact QNMT file (model.py:275-310): tensors in
    ``tensor_specs`` order, compact sorted-key JSON header, SHA-256 checksum."""
    raw, directory, at = [], [], 0
    for name, shape in tensor_specs(params.dims):
        arr = params.tensors[name]
        if isinstance(arr, torch.Tensor):
            arr = arr.detach().cpu().numpy()
        arr = np.ascontiguousarray(arr, dtype="<f4")
        if tuple(arr.shape) != tuple(shape):
            raise SchemaError(f"tensor {name} has shape {arr.shape}, expected {shape}")
        directory.append({"name": name, "shape": list(shape), "offset": at})
        raw.append(arr.tobytes())
        at += arr.nbytes
    payload = b"".join(raw)
    header = json.dumps({"dims": params.dims.as_dict(), "s0_mode": params.s0_mode,
                         "attention_query": params.attention_query,
                         "source_vocab": params.src_tokens, "target_vocab": params.tgt_tokens,
                         "payload_bytes": len(payload), "tensors": directory},
                        sort_keys=True, separators=(",", ":")).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MAGIC + VERSION.to_bytes(4, "little") + len(header).to_bytes(8, "little"))
        fh.write(header)
        fh.write(payload)
        fh.write(hashlib.sha256(payload).digest()[:8])


def _parse_model_file(blob: bytes):
    """Validate a QNMT file (model.py:313-387, same checks, messages and byte
    offsets).  Returns (dims, header, payload memoryview, {name: (offset, shape)})."""
    n = len(blob)
    if n < 16:
        raise FormatError("file shorter than the fixed header", offset=n)
    if blob[:4] != MAGIC:
        raise FormatError(f"bad magic {blob[:4]!r}, expected {MAGIC!r}", offset=0)
    version = _u(blob, 4, 8)
    if version != VERSION:
        raise FormatError(f"unsupported format version {version}", offset=4)
    hdr_end = 16 + _u(blob, 8, 16)
    if hdr_end + 8 > n:
        raise FormatError("declared header overruns the file", offset=8)
    try:
        header = json.loads(blob[16:hdr_end].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise FormatError(f"header is not valid JSON: {exc}", offset=16) from None
    missing = [k for k in _HEADER_KEYS if k not in header]
    if missing:
        raise SchemaError(f"header is missing required key {missing[0]!r}", offset=16)
    try:
        dims = Dims(**header["dims"])
    except TypeError as exc:
        raise SchemaError(f"bad dims block: {exc}", offset=16) from None
    plen = int(header["payload_bytes"])
    pend = hdr_end + plen
    if pend + 8 > n:
        raise FormatError("payload truncated", offset=min(n, pend))
    payload = memoryview(blob)[hdr_end:pend]
    if hashlib.sha256(payload).digest()[:8] != blob[pend:pend + 8]:
        raise FormatError("payload checksum mismatch", offset=pend)
    for key, declared, what in (("source_vocab", dims.src_vocab, "source"),
                                ("target_vocab", dims.tgt_vocab, "target")):
        if len(header[key]) != declared:
            raise SchemaError(f"{what} vocabulary lists {len(header[key])} tokens, dims declare {declared}",
                              offset=16)
    want = {name: tuple(shape) for name, shape in tensor_specs(dims)}
    entries = {e["name"]: e for e in header["tensors"]}
    if set(entries) != set(want):
        raise SchemaError(f"tensor directory mismatch (missing {sorted(set(want) - set(entries))}, "
                          f"extra {sorted(set(entries) - set(want))})", offset=16)
    layout = {}
    for name, shape in want.items():
        ent = entries[name]
        if tuple(ent["shape"]) != shape:
            raise SchemaError(f"tensor {name} declares shape {ent['shape']}, dims imply {shape}", offset=16)
        off = int(ent["offset"])
        if off < 0 or off + 4 * int(np.prod(shape)) > plen:
            raise SchemaError(f"tensor {name} overruns the payload", offset=hdr_end + max(off, 0))
        layout[name] = (off, shape)
    return dims, header, payload, layout


def load_model(path: str) -> ModelParams:
    """Read and validate a QNMT model file into host f32 tensors (model.py:313-387);
    tensors are read-only views of the file bytes, as in the reference."""
    with open(path, "rb") as fh:
        blob = fh.read()
    dims, header, payload, layout = _parse_model_file(blob)
    tensors = {name: np.frombuffer(payload, dtype="<f4", count=int(np.prod(shape)), offset=off).reshape(shape)
               for name, (off, shape) in layout.items()}
    return ModelParams(dims, tensors, list(header["source_vocab"]), list(header["target_vocab"]),
                       header["s0_mode"], header["attention_query"])


def load_quantized(path: str, with_stats: bool = False) -> QuantizedModel:
    """QNMT file -> device-resident int8 model.

    The file is validated on the host exactly like :func:`load_model`; the
    payload then crosses PCIe once (pinned staging, one H2D copy) and every
    tensor is a view of that device buffer: weight matrices are quantized by
    the device K1 kernel (bit-identical to ``quantize_model(load_model(path))``),
    embeddings and biases are used in place."""
    with open(path, "rb") as fh:
        blob = fh.read()
    dims, header, payload, layout = _parse_model_file(blob)
    dev = _dev.require_cuda()
    host = torch.empty(len(payload), dtype=torch.uint8, pin_memory=True)
    host.numpy()[:] = np.frombuffer(payload, dtype=np.uint8)
    buf = torch.empty(len(payload) + 16, dtype=torch.uint8, device=dev)
    buf[:len(payload)].copy_(host, non_blocking=True)
    views = {}
    for name, (off, shape) in layout.items():
        nbytes = 4 * int(np.prod(shape))
        if off % 4:   # unaligned directory entry (legal in the format): realign on the device
            views[name] = buf[off:off + nbytes].clone().view(torch.float32).view(shape)
        else:
            views[name] = buf[off:off + nbytes].view(torch.float32).view(shape)
    torch.cuda.current_stream().synchronize()   # the pinned staging buffer is released on return
    return _quantize_tensors(dims, views, list(header["source_vocab"]), list(header["target_vocab"]),
                             header["s0_mode"], header["attention_query"], with_stats)
