"""Shared helpers for the GPU parity tests (oracle = checker only)."""

import hashlib
import json
import os

import numpy as np

from oracle import qnmt_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F32 = np.float32


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def translate_specs():
    with open(os.path.join(GOLDEN, "translate_small.json")) as fh:
        return json.load(fh)


def model_pair(spec):
    """(package ModelParams, oracle QModel tier B) for a golden model spec."""
    import paper_1804_05038_b200 as pb
    d = pb.Dims(**spec["dims"])
    params = pb.synthetic_model(d, spec["seed"], spec["weight_std"], spec["bias_std"], spec["eos_bias"],
                                spec["s0_mode"], spec["attention_query"])
    om = O.QModel(O.Dims(**spec["dims"]), params.tensors, s0_mode=spec["s0_mode"],
                  attention_query=spec["attention_query"], tier="B")
    return params, om
