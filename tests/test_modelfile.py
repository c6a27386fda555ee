"""QNMT model file: byte-exact save, validated load, and the
device loader.  Pinned against a file written by the REFERENCE's save_model and
the reference loader's verdict on 19 corruptions of it
(tests/golden/make_golden.py gen_modelfile)."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

import paper_1804_05038_b200 as pb
from paper_1804_05038_b200 import errors

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, GOLDEN)
import modelfile_cases  # noqa: E402

FILE = os.path.join(GOLDEN, "model_tiny.qnmt")


@pytest.fixture(scope="module")
def verdicts():
    with open(os.path.join(GOLDEN, "model_tiny_errors.json")) as fh:
        return json.load(fh)


def test_golden_file_is_the_reference_file(verdicts):
    blob = open(FILE, "rb").read()
    assert hashlib.sha256(blob).hexdigest() == verdicts["file_sha256"]


def test_save_is_byte_identical_to_reference(tmp_path, verdicts):
    params = pb.generate_model(**verdicts["generate_model_args"])
    out = tmp_path / "ours.qnmt"
    pb.save_model(params, str(out))
    assert out.read_bytes() == open(FILE, "rb").read()


def test_load_roundtrip(tmp_path, verdicts):
    params = pb.generate_model(**verdicts["generate_model_args"])
    got = pb.load_model(FILE)
    assert got.dims == params.dims
    assert got.src_tokens == params.src_tokens and got.tgt_tokens == params.tgt_tokens
    assert (got.s0_mode, got.attention_query) == ("transform", "current")
    for name, shape in pb.tensor_specs(params.dims):
        assert got.tensors[name].shape == shape
        assert got.tensors[name].dtype == np.float32
        assert np.array_equal(got.tensors[name], params.tensors[name]), name
    # non-default flags and a synthetic (N(0, std)) model survive a save/load cycle
    syn = pb.synthetic_model(pb.Dims(9, 8, 4, 4, 3, 2), 5, bias_std=0.1, s0_mode="zero",
                             attention_query="previous")
    p = tmp_path / "syn.qnmt"
    pb.save_model(syn, str(p))
    back = pb.load_model(str(p))
    assert (back.s0_mode, back.attention_query) == ("zero", "previous")
    assert all(np.array_equal(back.tensors[k], syn.tensors[k]) for k in syn.tensors)


def test_save_rejects_wrong_shape(tmp_path):
    syn = pb.synthetic_model(pb.Dims(9, 8, 4, 4, 3, 2), 5)
    syn.tensors["attn.v"] = np.zeros((3, 1), np.float32)
    with pytest.raises(errors.SchemaError):
        pb.save_model(syn, str(tmp_path / "bad.qnmt"))


@pytest.mark.parametrize("case", sorted(modelfile_cases.cases(open(FILE, "rb").read())))
def test_corruption_verdict_matches_reference(case, tmp_path, verdicts):
    data = modelfile_cases.cases(open(FILE, "rb").read())[case]
    p = tmp_path / case
    p.write_bytes(data)
    want = verdicts["cases"][case]
    if want["error"] is None:
        pb.load_model(str(p))
        return
    with pytest.raises(errors.FormatError) as ei:
        pb.load_model(str(p))
    assert type(ei.value).__name__ == want["error"]
    assert ei.value.offset == want["offset"]


@pytest.mark.gpu
def test_load_quantized_equals_quantize_model():
    host = pb.quantize_model(pb.load_model(FILE))
    dev = pb.load_quantized(FILE)
    assert set(dev.q) == set(host.q) and set(dev.f) == set(host.f)
    for k in host.q:
        assert np.array_equal(dev.q[k].device_data().cpu().numpy(), host.q[k].device_data().cpu().numpy()), k
        assert float(dev.q[k].device_scale()[0]) == float(host.q[k].device_scale()[0]), k
    for k in host.f:
        assert np.array_equal(dev.f[k].cpu().numpy(), host.f[k].cpu().numpy()), k
        assert dev.f[k].data_ptr() % 16 == 0


@pytest.mark.gpu
def test_load_quantized_translates_like_the_oracle(tmp_path):
    from oracle import qnmt_oracle as O
    params = pb.synthetic_model(pb.Dims(64, 61, 16, 32, 24, 16), 7, weight_std=0.3, bias_std=0.1, eos_bias=0.5)
    p = tmp_path / "m.qnmt"
    pb.save_model(params, str(p))
    qm = pb.load_quantized(str(p))
    om = O.QModel(O.Dims(**params.dims.as_dict()), params.tensors)
    srcs = [[5, 9, 17, 33, 40], [3, 4, 60, 11]]
    got = pb.translate_batch(qm, srcs, pb.DecodeConfig(beam=3, max_ratio=2.0, precision="int8"), return_ids=True)
    for s, g in zip(srcs, got):
        want = om.translate(s, beam=3, max_ratio=2.0)
        assert g[0] == want[0] and g[1] == want[1]
