#!/usr/bin/env python
"""Benchmark: int8 beam-5 decode of the BASELINE cfg5 bulk-translation shard.

Workload (BASELINE.json configs[4], the config the metric is quoted on at
1/2/4/8 B200): V_src 32000, V_tgt 50000, E 512, H 1024, A 2048, R 512, beam 5,
max_ratio 1.5, a seeded 8192-sentence corpus with lengths ~ U[5, 100]; one
"step" = one batch of 256 sentences per GPU (weak scaling, no collective on
the data path).  Random N(0, 0.05) weights, synthetic token ids.

  value  : target tokens/s (EOS excluded, bench.py:161 of the reference) of the
           device-resident decode (qnmt_decode_batch_device: source ids already
           in HBM), CUDA events on the launching stream, max over ranks.
  e2e    : same metric through the public C-ABI call qnmt_translate_batch with
           HOST buffers (H2D of ids, D2H of finished lists + host selection).
  --impl reference : the reference algorithm on the host CPU (the oracle port;
           the reference itself is Python and cannot travel to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = dict(src_vocab=32000, tgt_vocab=50000, embed=512, hidden=1024, attn=2048, readout=512)
BEAM, MAX_RATIO, PER_GPU, CORPUS = 5, 1.5, 256, 8192
MODEL_SEED, CORPUS_SEED = 1804, 5038
WORKLOAD = ("cfg5 bulk translation shard: 256 sentences/GPU/step of a seeded 8192-sentence corpus, "
            "l~U[5,100], beam 5, max_ratio 1.5, V_tgt 50000, H 1024, E 512, A 2048")


def corpus():
    rng = np.random.default_rng(CORPUS_SEED)
    lens = rng.integers(5, 101, CORPUS)
    return [rng.integers(3, DIMS["src_vocab"], int(l)).astype(np.int32) for l in lens]


def batch_for(step: int, rank: int, world: int, sents):
    nb = len(sents) // PER_GPU
    b = (step * world + rank) % nb
    return sents[b * PER_GPU:(b + 1) * PER_GPU]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 4 + i and "Active" in r[4 + i] and "Not" not in r[4 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_baseline(params, sents, sample: int, budget_s: float = 25.0):
    """Reference algorithm (oracle port) on host cores over a bounded sample."""
    import concurrent.futures as cf

    from oracle import qnmt_oracle as O
    om = O.QModel(O.Dims(**DIMS), params.tensors)
    cores = os.cpu_count() or 1
    sub = sents[:sample]
    t0 = time.perf_counter()
    done, tokens, outs = 0, 0, []
    with cf.ThreadPoolExecutor(max_workers=cores) as pool:
        futs = [pool.submit(om.translate, s.tolist(), BEAM, MAX_RATIO) for s in sub]
        for f in futs:
            toks, lp = f.result()
            outs.append((toks, lp))
            tokens += len(toks)
            done += 1
    wall = time.perf_counter() - t0
    return {"value": tokens / wall, "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": f"{done} sentences of the first timed batch (beam 5, V_tgt 50000), "
                      f"oracle/qnmt_oracle.py numpy port, {cores} threads, {wall:.1f}s",
            "sentences_per_s": done / wall}, outs


def run_reference(args, rank, world):
    if rank != 0:
        return
    import paper_1804_05038_b200 as pb   # only for the seeded synthetic model recipe (host code)
    params = pb.synthetic_model(pb.Dims(**DIMS), MODEL_SEED)
    sents = corpus()
    sample = args.cpu_sample
    for w in range(args.warmup):
        cpu_baseline(params, batch_for(w, 0, 1, sents)[:2], 2)
    vals, secs, toks = [], 0.0, 0
    for k in range(args.steps):
        r, outs = cpu_baseline(params, batch_for(args.warmup + k, 0, 1, sents), sample)
        vals.append(r)
        n = sum(len(o[0]) for o in outs)
        toks += n
        secs += n / r["value"]
    value = toks / secs
    line = {"metric": "tokens/sec (int8 beam-5 decode, target tokens excl. EOS)", "value": value,
            "unit": "tokens/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {"workload": WORKLOAD, "sample_per_step": sample},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": vals[0]["cores"],
                             "kind": "port", "sample": vals[0]["sample"]},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="disable the engine's event profiler")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1804_05038_b200 as pb
    from paper_1804_05038_b200 import _lib, _dev

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    params = pb.synthetic_model(pb.Dims(**DIMS), MODEL_SEED)
    qm = pb.quantize_model(params)
    eng = pb.Engine(qm, PER_GPU, 100, BEAM)
    sents = corpus()
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def upload(batch):
        lens = np.array([len(s) for s in batch], dtype=np.int32)
        ids = torch.from_numpy(np.concatenate(batch)).to(dev)
        return ids, lens

    def fetch(batch):
        stride = int(math.ceil(MAX_RATIO * max(len(s) for s in batch))) + 1
        out = np.zeros((len(batch), stride), np.int32)
        ol = np.zeros(len(batch), np.int32)
        lp = np.zeros(len(batch), np.float64)
        _lib.call("qnmt_fetch_results", eng._h, out.ctypes.data, stride, ol.ctypes.data, lp.ctypes.data,
                  stream.cuda_stream)
        return out, ol, lp

    def device_step(batch):
        ids, lens = upload(batch)
        flush.fill_(1)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = lib.qnmt_kernel_launches()
        ev0.record(stream)
        _lib.call("qnmt_decode_batch_device", eng._h, ids.data_ptr(), lens.ctypes.data, len(batch), BEAM,
                  MAX_RATIO, stream.cuda_stream)
        ev1.record(stream)
        ev1.synchronize()
        launches = lib.qnmt_kernel_launches() - l0
        out, ol, lp = fetch(batch)
        return ev0.elapsed_time(ev1) / 1000.0, int(ol.sum()), launches

    for w in range(args.warmup):
        device_step(batch_for(w, rank, world, sents))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    import ctypes as C
    if not args.no_profile:
        lib.qnmt_engine_profile(eng._h, 1)
    clk = ClockSampler(local)
    secs, toks, launches = 0.0, 0, 0
    step_ms = []
    for k in range(args.steps):
        t, n, nl = device_step(batch_for(args.warmup + k, rank, world, sents))
        secs += t
        toks += n
        launches += nl
        step_ms.append(1000 * t)
    torch.cuda.synchronize()
    clocks = clk.stop()
    phases = None
    if not args.no_profile:
        arr = [(C.c_double * 16)() for _ in range(4)]
        ng = lib.qnmt_engine_profile_read(eng._h, *[C.cast(a, C.c_void_p) for a in arr])
        lib.qnmt_engine_profile(eng._h, 0)
        names = ["encoder", "embed", "quantize", "gemm_decoder", "gru_gates", "attention", "gemm_vocab",
                 "topk", "search", "gather", "misc"]
        phases = {names[i]: {"ms": arr[0][i] / args.steps, "launch_groups": arr[1][i] / args.steps,
                             "int_ops": arr[2][i] / args.steps, "bytes": arr[3][i] / args.steps}
                  for i in range(ng)}
    if world > 1:
        dist.barrier()

    # e2e through the public C-ABI call with host buffers
    e2e_secs, e2e_toks, h2d, d2h = 0.0, 0, 0, 0
    for k in range(args.steps):
        batch = batch_for(args.warmup + k, rank, world, sents)
        lens = np.array([len(s) for s in batch], dtype=np.int32)
        ids = np.ascontiguousarray(np.concatenate(batch))
        stride = int(math.ceil(MAX_RATIO * int(lens.max()))) + 1
        out = np.zeros((len(batch), stride), np.int32)
        ol = np.zeros(len(batch), np.int32)
        lp = np.zeros(len(batch), np.float64)
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.call("qnmt_translate_batch", eng._h, ids.ctypes.data, lens.ctypes.data, len(batch), BEAM,
                  MAX_RATIO, out.ctypes.data, stride, ol.ctypes.data, lp.ctypes.data, stream.cuda_stream)
        e2e_secs += time.perf_counter() - t0
        e2e_toks += int(ol.sum())
        n = len(batch)
        h2d += ids.nbytes + n * 40 + 2 * 2 * n * int(lens.max()) * 4 + ids.nbytes + n * 4
        d2h += int(lib.qnmt_last_d2h_bytes(eng._h))

    stats = torch.tensor([secs, toks, e2e_secs, e2e_toks], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        secs, e2e_secs = float(mx[0]), float(mx[2])
        toks, e2e_toks = int(sm[1]), int(sm[3])
    value = toks / secs
    e2e_value = e2e_toks / e2e_secs

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        first = batch_for(args.warmup, 0, 1, sents)
        cpu, outs = cpu_baseline(params, first, args.cpu_sample)
        cpu["gpu_match"] = None
    if rank == 0:
        line = {"metric": "tokens/sec (int8 beam-5 decode, target tokens excl. EOS)",
                "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
                "data": "synthetic (seeded N(0,0.05) weights, uniform token ids)",
                "config": {"workload": WORKLOAD, "sentences_per_gpu_step": PER_GPU,
                           "parallelism": f"sentence-sharded x{world} (no collective)",
                           "l2": "flushed (512 MB write) before every timed step"},
                "sentences_per_s": world * PER_GPU * args.steps / secs,
                "step_ms": step_ms,
                "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d // args.steps,
                        "d2h_bytes_per_step": d2h // args.steps},
                "gpu_launches": launches,
                "roofline": None,
                "phases_ms_per_step": {k: round(v["ms"], 3) for k, v in phases.items()} if phases else None,
                "cpu_baseline": cpu,
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
