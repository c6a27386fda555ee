"""Deterministic corruptions of a QNMT model file, shared by make_golden.py
(which records the REFERENCE loader's verdict on each) and
tests/test_modelfile.py (which checks the B200 loader gives the same one)."""

import json


def _patch_header(blob: bytes, fn) -> bytes:
    hl = int.from_bytes(blob[8:16], "little")
    header = json.loads(blob[16:16 + hl].decode("utf-8"))
    fn(header)
    nh = json.dumps(header, sort_keys=True, separators=(",", ":")).encode("utf-8")
    return blob[:8] + len(nh).to_bytes(8, "little") + nh + blob[16 + hl:]


def _flip(blob: bytes, at: int) -> bytes:
    return blob[:at] + bytes([blob[at] ^ 0x5A]) + blob[at + 1:]


def cases(blob: bytes) -> dict:
    hl = int.from_bytes(blob[8:16], "little")
    pstart = 16 + hl
    out = {
        "short": blob[:11],
        "magic": b"QNMX" + blob[4:],
        "version": blob[:4] + (2).to_bytes(4, "little") + blob[8:],
        "header_overrun": blob[:8] + (len(blob)).to_bytes(8, "little") + blob[16:],
        "header_json": blob[:16] + b"[" + blob[17:],
        "header_utf8": blob[:16] + b"\xff" + blob[17:],
        "payload_truncated": blob[:pstart + 40],
        "checksum_payload": _flip(blob, pstart + 17),
        "checksum_tail": _flip(blob, len(blob) - 1),
    }

    def drop(key):
        return lambda h: h.pop(key)

    def set_dims(h):
        h["dims"]["bogus"] = 1

    def short_vocab(h):
        h["source_vocab"] = h["source_vocab"][:-1]

    def short_tvocab(h):
        h["target_vocab"] = h["target_vocab"] + ["extra"]

    def drop_tensor(h):
        h["tensors"] = [t for t in h["tensors"] if t["name"] != "attn.v"]

    def extra_tensor(h):
        h["tensors"].append({"name": "zz.extra", "shape": [1], "offset": 0})

    def bad_shape(h):
        for t in h["tensors"]:
            if t["name"] == "dec_q.wz":
                t["shape"] = [t["shape"][1], t["shape"][0]]

    def overrun(h):
        for t in h["tensors"]:
            if t["name"] == "s0.b":
                t["offset"] = h["payload_bytes"] - 4

    for name, fn in (("missing_dims", drop("dims")), ("missing_tensors", drop("tensors")),
                     ("missing_s0_mode", drop("s0_mode")), ("bad_dims", set_dims),
                     ("src_vocab_len", short_vocab), ("tgt_vocab_len", short_tvocab),
                     ("dir_missing", drop_tensor), ("dir_extra", extra_tensor), ("shape", bad_shape),
                     ("tensor_overrun", overrun)):
        out[name] = _patch_header(blob, fn)
    return out
