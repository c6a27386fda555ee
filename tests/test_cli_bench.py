"""Harness / CLI parity: BenchReport schema (bench.py:60-92),
run_benchmark / profile_phases, and the cli subcommands driving the GPU path."""

import json
import os

import numpy as np
import pytest

import paper_1804_05038_b200 as pb
from paper_1804_05038_b200 import bench, cli, errors

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

REPORT_KEYS = {"precision", "sentences", "total_words", "workers", "repeats", "run_seconds", "median_seconds",
               "wps", "wpcs", "phase_seconds", "phase_fractions"}


def test_genmodel_writes_the_reference_file(tmp_path):
    with open(os.path.join(GOLDEN, "model_tiny_errors.json")) as fh:
        a = json.load(fh)["generate_model_args"]
    out = tmp_path / "g.qnmt"
    rc = cli.main(["genmodel", "--output", str(out), "--src-vocab", str(a["src_vocab"]), "--tgt-vocab",
                   str(a["tgt_vocab"]), "--embed", str(a["embed"]), "--hidden", str(a["hidden"]), "--seed",
                   str(a["seed"]), "--attn-dim", str(a["attn"]), "--readout", str(a["readout"])])
    assert rc == 0
    assert out.read_bytes() == open(os.path.join(GOLDEN, "model_tiny.qnmt"), "rb").read()


def test_bleu_subcommand(tmp_path, capsys):
    with open(os.path.join(GOLDEN, "fp32_small.json")) as fh:
        case = [c for c in json.load(fh)["bleu"] if not isinstance(c["bleu"], str) and c["bleu"] > 0][0]
    h, r = tmp_path / "h.txt", tmp_path / "r.txt"
    h.write_text("\n".join(" ".join(x) for x in case["hyps"]) + "\n")
    r.write_text("\n".join(" ".join(x) for x in case["refs"]) + "\n")
    assert cli.main(["bleu", "--input", str(h), "--reference", str(r)]) == 0
    assert capsys.readouterr().out.strip() == f"{case['bleu']:.2f}"


def test_cli_errors_exit_1(tmp_path):
    assert cli.main(["compare", "--model", str(tmp_path / "missing.qnmt"), "--input", "x"]) == 1
    bad = tmp_path / "bad.qnmt"
    bad.write_bytes(b"QNMX" + bytes(20))
    assert cli.main(["quantize-report", "--model", str(bad)]) == 1


def test_bench_report_schema_and_config_errors():
    r = bench.BenchReport("int8", 2, 10, 1, 1, [0.5], 0.5, 20.0, 20.0, {"matmul": 0.1}, {"matmul": 20.0})
    assert set(r.to_dict()) == REPORT_KEYS
    assert json.loads(r.to_json())["wps"] == 20.0
    p = pb.synthetic_model(pb.Dims(20, 17, 8, 8, 8, 8), 1)
    with pytest.raises(errors.ConfigError):
        bench.run_benchmark(p, [["w0001"]], pb.DecodeConfig(2, 1.5), repeats=2)
    with pytest.raises(errors.ConfigError):
        bench.run_benchmark(p, [["w0001"]], pb.DecodeConfig(2, 1.5), workers=0)
    t = bench.PhaseTimer()
    t.push("a")
    t.push("b")
    t.pop()
    t.pop()
    assert set(t.seconds) == {"a", "b"} and t.tracked_total() >= 0


@pytest.mark.gpu
def test_gpu_cli_translate_compare_bench(tmp_path, capsys):
    from oracle import qnmt_oracle as O
    params = pb.synthetic_model(pb.Dims(64, 61, 16, 32, 24, 16), 7, weight_std=0.3, bias_std=0.1, eos_bias=0.5)
    mp = tmp_path / "m.qnmt"
    pb.save_model(params, str(mp))
    rng = np.random.default_rng(5)
    sents = [[params.src_tokens[i] for i in rng.integers(3, 64, int(rng.integers(1, 9)))] for _ in range(10)]
    inp = tmp_path / "in.txt"
    inp.write_text("\n".join(" ".join(s) for s in sents[:5]) + "\n\n" + "\n".join(" ".join(s) for s in sents[5:]) + "\n")
    out = tmp_path / "out.txt"
    rc = cli.main(["translate", "--model", str(mp), "--input", str(inp), "--output", str(out), "--precision", "int8",
                   "--beam", "3", "--max-ratio", "2.0"])
    assert rc == 2   # the empty line fails, the rest translate
    lines = out.read_text().split("\n")[:-1]
    assert len(lines) == 11 and lines[5] == ""
    om = O.QModel(O.Dims(**params.dims.as_dict()), params.tensors)
    got = lines[:5] + lines[6:]
    for s, line in zip(sents, got):
        ids, _ = om.translate(params.src_ids(s), beam=3, max_ratio=2.0)
        assert line == pb.bpe_merge([params.tgt_tokens[i] for i in ids])
    capsys.readouterr()
    inp2 = tmp_path / "in2.txt"
    inp2.write_text("\n".join(" ".join(s) for s in sents) + "\n")
    assert cli.main(["compare", "--model", str(mp), "--input", str(inp2), "--beam", "3", "--max-ratio", "2.0",
                     "--format", "json"]) == 0
    rep = json.loads(capsys.readouterr().out)
    want = pb.compare_precisions(params, sents, pb.DecodeConfig(3, 2.0)).to_dict()
    assert rep == want
    assert cli.main(["bench", "--model", str(mp), "--input", str(inp2), "--repeats", "3", "--beam", "3",
                     "--format", "json"]) == 0
    doc = json.loads(capsys.readouterr().out)
    assert [r["precision"] for r in doc["reports"]] == ["fp32", "int8"]
    for r in doc["reports"]:
        assert set(r) == REPORT_KEYS and r["wps"] > 0 and len(r["run_seconds"]) == 3
        assert abs(sum(r["phase_fractions"].values()) - 100.0) < 1e-6
    assert doc["speed_ratio_int8_over_fp32"] > 0
    table = bench.profile_phases(params, sents, pb.DecodeConfig(3, 2.0, "int8"))
    assert table and abs(sum(p for _, p in table) - 100.0) < 1e-6
