"""CPU-only checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/qnmt_b200.h declares; the product path refuses
to run without a GPU (no CPU fallback)."""

import os
import re
import subprocess

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qnmt_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qnmt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_1804_05038_b200 import _lib
    lib = _lib.load()
    declared = header_functions()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (qnmt_\w+)", out))
    assert set(declared) == exported, (set(declared) ^ exported)
    for name in declared:
        assert hasattr(lib, name)
    assert set(_lib.SIGNATURES) == set(declared)
    assert lib.qnmt_abi_version() == 1


def test_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1804_05038_b200 as pb
    from paper_1804_05038_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        pb.quantize(np.ones((2, 2), np.float32))


def test_host_logic_cpu():
    import paper_1804_05038_b200 as pb
    from paper_1804_05038_b200.decoder import max_steps
    assert pb.bpe_merge(["predic@@", "tated"]) == "predictated"
    assert pb.bpe_merge(["a@@", "b@@", "c"]) == "abc"
    assert max_steps(50, 0.98) == 50
    with pytest.raises(pb.errors.ConfigError):
        pb.DecodeConfig(beam=0)
    d = pb.Dims(40, 37, 8, 12, 10, 6)
    m = pb.synthetic_model(d, 11, 0.05, 0.05)
    from oracle import qnmt_oracle as O
    t = O.synthetic_tensors(O.Dims(**d.as_dict()), 11, 0.05, 0.05)
    for name, _ in pb.tensor_specs(d):
        assert np.array_equal(m.tensors[name], t[name]), name
    assert m.src_ids(["w0001", "zzz"]).tolist() == [3, 1]
