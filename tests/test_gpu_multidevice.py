"""The product's sentence-sharded bulk path (translate_batch(..., devices=...),
SURVEY 8(e)): shards from decoder.shard_batches, one host thread and one weight
replica per device, no collective.  On the one-GPU box the shards of a
"two-device" run land on the same GPU (device list [0, 0]), which exercises
the splitter, the per-device threads and the reassembly; outputs must equal
the single-device decode and the oracle (the cfg5 golden sample below pins
them to the reference itself, Tier B)."""

import json
import os

import numpy as np
import pytest
import torch

from qnmt_test_helpers import GOLDEN, model_pair, translate_specs

pytestmark = pytest.mark.gpu
pb = pytest.importorskip("paper_1804_05038_b200")


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_devices_equal_single_device_and_oracle(devices):
    tr = translate_specs()
    params, om = model_pair(tr["models"]["med"])
    qm = pb.quantize_model(params)
    rng = np.random.default_rng(len(devices))
    sents = [rng.integers(3, params.dims.src_vocab, int(rng.integers(1, 14))).tolist() for _ in range(41)]
    cfg = pb.DecodeConfig(beam=3, max_ratio=1.5, precision="int8")
    one = pb.translate_batch(qm, sents, cfg, max_batch=8, return_ids=True)
    many = pb.translate_batch(qm, sents, cfg, max_batch=8, return_ids=True, devices=devices)
    assert many == one
    for s, (toks, lp) in zip(sents[:10], many[:10]):
        assert (toks, lp) == om.translate(s, 3, 1.5)


def test_replicate_same_device_is_identity():
    tr = translate_specs()
    params, _ = model_pair(tr["models"]["small"])
    qm = pb.quantize_model(params)
    assert pb.replicate(qm, 0) is qm
    assert pb.replicate(qm, torch.device("cuda", 0)) is qm


def test_devices_cfg5_golden_sample():
    """The cfg5 golden sample (V = 50000, reference-generated, Tier B) through the
    sharded path."""
    c = json.load(open(os.path.join(GOLDEN, "baseline_corpora.json")))["cfg5"]
    params = pb.synthetic_model(pb.Dims(**c["dims"]), c["model_seed"])
    qm = pb.quantize_model(params)
    srcs = [case["src"] for case in c["cases"]]
    cfg = pb.DecodeConfig(beam=c["beam"], max_ratio=c["max_ratio"], precision="int8")
    got = pb.translate_batch(qm, srcs, cfg, max_batch=4, return_ids=True, devices=[0, 0])
    for case, (toks, lp) in zip(c["cases"], got):
        assert toks == case["out_B"] and lp == case["logp_B"]


@pytest.mark.gpu
def test_engines_destroyed_while_other_threads_capture_step_graphs():
    """Regression (found by benchmarks/stress_parity.py): an engine destroyed by the garbage
    collector (cudaDeviceSynchronize + cudaFree in qnmt_engine_destroy) while another host thread
    was capturing its decode-step graph invalidated that capture ("operation failed due to a
    previous error during capture").  Captures and device-wide calls now exclude each other
    (g_capture_gate).  Many short-lived models, each decoded on 3 engine streams."""
    import numpy as np
    import paper_1804_05038_b200 as pb
    dims = pb.Dims(44, 88, 32, 32, 16, 32)
    rng = np.random.default_rng(11)
    for trial in range(150):
        params = pb.synthetic_model(dims, 1000 + trial, 0.2, 0.1, 1.5, "transform", "previous")
        qm = pb.quantize_model(params)
        sents = [rng.integers(3, 44, int(rng.integers(1, 12))).tolist() for _ in range(12)]
        out = pb.translate_batch(qm, sents, pb.DecodeConfig(beam=1, max_ratio=0.5, precision="int8"), max_batch=4,
                                 return_ids=True, streams=3)
        assert len(out) == len(sents)
