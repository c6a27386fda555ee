#!/usr/bin/env python
"""Benchmark: int8 beam-5 decode of the BASELINE cfg5 bulk-translation shard.

Workload (BASELINE.json configs[4], the config the metric is quoted on at
1/2/4/8 B200): V_src 32000, V_tgt 50000, E 512, H 1024, A 2048, R 512, beam 5,
max_ratio 1.5, a seeded 8192-sentence corpus with lengths ~ U[5, 100]; one
"step" = one pass over the whole corpus: it is sorted by length, cut into
batches of 256 sentences (one engine call each) and the batches are dealt
round-robin to the GPUs (strong scaling: the corpus is fixed, no collective on
the data path).  On each GPU STREAMS engines, each on its own CUDA stream and
host thread, take batches from a queue.  Seeded N(0, 0.05) weights, uniform
synthetic token ids (no datasets / checkpoints in this environment).

  value  : target tokens/s (EOS excluded, as the reference's bench.py:161 counts)
           of the device-resident decode (qnmt_decode_batch_device: source ids
           already in HBM), CUDA events on the launching stream, L2 flushed
           before every step, max over ranks.
  e2e    : the same metric through the public bulk API translate_batch (C-ABI
           qnmt_translate_batch per batch) with HOST buffers (H2D of ids, D2H of
           finished lists + history, host selection of the best hypothesis),
           wall clock per step.
  roofline: per-kernel device time measured live by %globaltimer stamps
           captured into the step graphs (a CUDA graph step cannot be bracketed
           by host events) of an untimed single-stream pass over the same shard
           right after the timed passes; algorithmic bytes / int-ops per launch
           from the live column count of each step.
  --impl reference : the unmodified reference package (pip-installed into
           baseline/_ref, which travels to the GPU box) through its own
           bench.run_benchmark on the host cores, on a bounded sample of the
           corpus per step; the numpy port oracle/qnmt_oracle.py only if the
           package cannot be imported there.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = dict(src_vocab=32000, tgt_vocab=50000, embed=512, hidden=1024, attn=2048, readout=512)
BEAM, MAX_RATIO, PER_GPU, CORPUS = 5, 1.5, 256, 8192
STREAMS = int(os.environ.get("QNMT_BENCH_STREAMS", "3"))   # engines (CUDA streams + host threads) per GPU
MODEL_SEED, CORPUS_SEED = 1804, 5038
METRIC = "tokens/sec (int8 beam-5 decode, target tokens excl. EOS)"
WORKLOAD = ("cfg5 bulk translation: one step = the whole seeded 8192-sentence corpus (l~U[5,100]) sharded over "
            "the GPUs, 256 sentences per engine call, beam 5, max_ratio 1.5, V_tgt 50000, H 1024, E 512, A 2048, "
            "R 512")
# DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per algorithmic byte, per launch, measured by
# ncu on the current kernels in one cfg5 batch decode (batch 16, N = 1280, sum l = 13941;
# benchmarks/one_batch.py): attention = k_att_scale + k_att_score8 + k_att_context4
# (profiles/r02_ob_e0_c1_att_launches.csv, profiles/r02_ob_score8_att_launches.csv): 249.8 MB of 249.4 MB;
# k_vocab_stats 27.13 + 0.60 MB of 50.30 MB (partials stay in L2) and k_vocab_merge 25.41 MB of
# 24.13 MB (profiles/r02_ncu_full_summary.md)
NCU_TRAFFIC_RATIO = {"attention": 249.76 / 249.38, "vocab_stats": 27.73 / 50.30, "vocab_merge": 25.41 / 24.13}


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def corpus():
    rng = np.random.default_rng(CORPUS_SEED)
    lens = rng.integers(5, 101, CORPUS)
    return [rng.integers(3, DIMS["src_vocab"], int(l)).astype(np.int32) for l in lens]


def sorted_batches(sents):
    """Length-sorted (stable) batches of PER_GPU corpus indices."""
    order = sorted(range(len(sents)), key=lambda i: (len(sents[i]), i))
    return [order[i:i + PER_GPU] for i in range(0, len(order), PER_GPU)]


def shard_batches(sents, rank: int, world: int):
    """Sorted batches dealt to ranks in snake order (0..W-1, W-1..0, ...): every rank
    sees the whole length range and the ranks' work is balanced."""
    bs = sorted_batches(sents)
    return [b for k, b in enumerate(bs) if (k % world if (k // world) % 2 == 0 else world - 1 - k % world) == rank]


def cpu_sample(sents, n):
    """n corpus indices spread evenly over the sorted length range (bounded CPU sample)."""
    order = sorted(range(len(sents)), key=lambda i: (len(sents[i]), i))
    return [order[(2 * k + 1) * len(order) // (2 * n)] for k in range(n)]


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


REF_DIR = os.path.join(ROOT, "baseline", "_ref")   # the unmodified reference package (pip --target install)


def load_reference():
    """The reference package ``qnmt`` as installed into baseline/_ref (DESIGN.md
    section 6): (module, None), or (None, reason) when it cannot be imported."""
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "qnmt_numba_cache"))
    if not os.path.isdir(os.path.join(REF_DIR, "qnmt")):
        return None, "baseline/_ref/qnmt not installed"
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import qnmt
        import qnmt.bench  # noqa: F401
        import qnmt.qmath  # noqa: F401
    except Exception as exc:   # noqa: BLE001
        return None, f"import qnmt failed: {type(exc).__name__}: {exc}"
    return qnmt, None


def reference_model(qnmt, params):
    """The reference's own int8 model (model.quantize_model) of the benchmark's
    seeded weights, built through its ModelParams constructor (model.py:196-222)."""
    from qnmt import model as rm
    d = rm.Dims(**DIMS)
    rp = rm._build_params(d, {k: np.asarray(v) for k, v in params.tensors.items()}, rm._synthetic_vocab(d.src_vocab),
                          rm._synthetic_vocab(d.tgt_vocab), "transform", "current")
    return rm.quantize_model(rp), rp


def cpu_translate(ref, sents, threads=None):
    """The reference's own decode on host cores: qnmt.decoder.translate, one
    sentence per worker thread of a ThreadPoolExecutor -- the scheme of its
    bench._decode_corpus (bench.py:107-132; the numba int8 kernels release the
    GIL).  ``ref`` = (qnmt module, quantized model, float params).
    Returns ([(ids, logp)], seconds, threads)."""
    import concurrent.futures as cf
    _, qm, rp = ref
    from qnmt.decoder import DecodeConfig, translate
    cores = min(threads or os.cpu_count() or 1, len(sents))
    cfg = DecodeConfig(beam=BEAM, max_ratio=MAX_RATIO, precision="int8")
    toks = [[rp.src_tokens[i] for i in s] for s in sents]
    idx = {t: i for i, t in enumerate(rp.tgt_tokens)}
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=cores) as pool:
        outs = list(pool.map(lambda t: translate(qm, t, cfg), toks))
    dt = time.perf_counter() - t0
    return [([idx[w] for w in words], lp) for words, lp in outs], dt, cores


def cpu_translate_port(params, sents, threads=None):
    """Fallback when the reference cannot be imported: the numpy port
    oracle/qnmt_oracle.py (pinned to the reference's Tier-B goldens)."""
    import concurrent.futures as cf

    from oracle import qnmt_oracle as O
    om = O.QModel(O.Dims(**DIMS), params.tensors)
    cores = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=cores) as pool:
        outs = list(pool.map(lambda s: om.translate(s.tolist(), BEAM, MAX_RATIO), sents))
    return outs, time.perf_counter() - t0, cores


def host_desc(qnmt=None):
    vnni = None
    if qnmt is not None:
        vnni = bool(getattr(qnmt.qmath, "HAVE_VNNI", False))
    return {"host_threads": os.cpu_count(), "avx512_vnni": vnni}


def run_reference(args, rank, world):
    """--impl reference: the unmodified reference package (baseline/_ref) through
    its own public API (quantize_model + translate on a thread pool, the VNNI
    numba int8 path when the host CPU has it) with all host threads, on a
    bounded sample of the cfg5 corpus per step (rank 0 only)."""
    if rank != 0:
        return
    import paper_1804_05038_b200 as pb   # host-side synthetic model recipe only (numpy)
    params = pb.synthetic_model(pb.Dims(**DIMS), MODEL_SEED)
    sents = corpus()
    sample = args.cpu_sample
    idx = cpu_sample(sents, sample)
    qnmt, why = load_reference()
    secs, toks = 0.0, 0
    if qnmt is not None:
        ref = (qnmt,) + reference_model(qnmt, params)
        short = min(range(len(sents)), key=lambda i: len(sents[i]))
        for _ in range(args.warmup):   # numba JIT / weight shadows (the reference's own warm-up pass)
            cpu_translate(ref, [sents[short]])
        cores = 1
        for _ in range(args.steps):
            outs, dt, cores = cpu_translate(ref, [sents[i] for i in idx])
            toks += sum(len(o[0]) for o in outs)
            secs += dt
        kind = "reference"
        what = (f"qnmt (unmodified, baseline/_ref) decoder.translate, one sentence per worker thread "
                f"(bench._decode_corpus scheme), {cores} threads, VNNI={bool(qnmt.qmath.HAVE_VNNI)}")
    else:
        short = min(range(len(sents)), key=lambda i: len(sents[i]))
        for _ in range(args.warmup):
            cpu_translate_port(params, [sents[short]])
        cores = 1
        for _ in range(args.steps):
            outs, dt, cores = cpu_translate_port(params, [sents[i] for i in idx])
            toks += sum(len(o[0]) for o in outs)
            secs += dt
        kind = "port"
        what = f"oracle/qnmt_oracle.py numpy port ({why}), {cores} threads"
    value = toks / secs
    desc = (f"{sample} sentences per step spread over the corpus length range (lengths "
            f"{len(sents[idx[0]])}..{len(sents[idx[-1]])}), beam 5, max_ratio 1.5, V_tgt 50000, {what}")
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample_per_step": sample},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": desc,
                             **host_desc(qnmt)},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


VT_TILE, VT_GROUPS, VT_PART_BYTES = 192, 3, 24   # vocab_topk.cu: tokens per tile, partials per tile, bytes


def kernel_rooflines(rows, hbm, peak_kind, sm_mhz=None):
    """rows: stamps of the timed steps -> per-kernel achieved vs roofline.

    Every kernel gets the contract's HBM roofline (algorithmic bytes / device
    time, against the measured copy bandwidth) and, where the kernel is bound by
    an arithmetic pipe instead, a "compute" roofline for that pipe:
      attention    MUFU: 2 ops (ex2, rcp) per tanh element, 16 ops/clk/SM
      vocab_stats  fp64: 14 ops per logit (dequant, exp, sum), 64 ops/clk/SM
    """
    V, R, A, H2 = DIMS["tgt_vocab"], DIMS["readout"], DIMS["attn"], 2 * DIMS["hidden"]
    f = (sm_mhz or 1965.0) * 1e6
    n_parts = VT_GROUPS * ((V + VT_TILE - 1) // VT_TILE)
    t = {"attention": 0.0, "vocab_merge": 0.0, "vocab_stats": 0.0, "step": 0.0}
    work = {"attention": 0.0, "vocab_merge": 0.0, "vocab_stats": 0.0}
    comp = {"attention": 0.0, "vocab_stats": 0.0}
    ops_vocab = 0.0
    launches = 0
    for r in rows:
        n, sl, spl = float(r[8]), float(r[9]), float(r[10])
        if n <= 0:
            continue
        launches += 1
        t["attention"] += (r[2] - r[1]) * 1e-9
        t["vocab_merge"] += (r[4] - r[3]) * 1e-9
        t["vocab_stats"] += (r[6] - r[5]) * 1e-9
        t["step"] += (r[4] - r[0]) * 1e-9
        # algorithmic bytes per launch
        work["attention"] += 4.0 * (sl * A + sl * H2 + n * A + n * H2)   # att_proj, states, u, ctx
        work["vocab_stats"] += V * R + n * R + n * n_parts * VT_PART_BYTES   # W, X codes, partials
        work["vocab_merge"] += n * n_parts * VT_PART_BYTES + n * BEAM * 12  # partials, candidates
        comp["attention"] += spl * A              # tanh elements
        comp["vocab_stats"] += n * V              # logits
        ops_vocab += 2.0 * V * R * n
    peaks_c = {"attention": ("tanh elements/s (2 MUFU ops each)", 16 * 148 * f / 2),
               "vocab_stats": ("logits/s (14 fp64 ops each)", 64 * 148 * f / 14)}
    out = {}
    for k in ("attention", "vocab_stats", "vocab_merge"):
        if t[k] <= 0:
            continue
        ach = work[k] / t[k] / 1e9
        ratio = NCU_TRAFFIC_RATIO.get(k)
        if k == "vocab_stats":   # a fused int8 GEMM: its roofline is the tensor pipe (HBM figures kept beside)
            tops = ops_vocab / t[k] / 1e12
            out[k] = {"bound": "tensor", "achieved": tops, "peak": 4500.0, "unit": "int8 TOPS",
                      "frac": tops / 4500.0, "peak_source": "spec (4.5 POPS dense int8)",
                      "hbm_GBps": ach, "hbm_frac": ach / hbm,
                      "us_per_launch": 1e6 * t[k] / max(launches, 1),
                      "traffic": (work[k] / max(launches, 1) * ratio) if ratio else None,
                      "algorithmic_bytes_per_launch": work[k] / max(launches, 1),
                      "share_of_step": t[k] / t["step"] if t["step"] > 0 else None}
            unit, pk = peaks_c[k]
            ca = comp[k] / t[k]
            out[k]["compute"] = {"unit": unit, "achieved": ca, "peak": pk, "frac": ca / pk}
            continue
        out[k] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                  "us_per_launch": 1e6 * t[k] / max(launches, 1),
                  "traffic": (work[k] / max(launches, 1) * ratio) if ratio else None,
                  "algorithmic_bytes_per_launch": work[k] / max(launches, 1), "peak_source": peak_kind,
                  "share_of_step": t[k] / t["step"] if t["step"] > 0 else None}
        if k in peaks_c:
            unit, pk = peaks_c[k]
            ca = comp[k] / t[k]
            out[k]["compute"] = {"unit": unit, "achieved": ca, "peak": pk, "frac": ca / pk}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg1-cfg4 sub-lines (bench_cfgs.py)")
    ap.add_argument("--no-stamps", action="store_true", help="no device-clock stamps (no roofline)")
    ap.add_argument("--no-profile", action="store_true", help="(kept for compatibility)")
    ap.add_argument("--batch", type=int, default=0,
                    help="sentences per engine call (default 256, BASELINE's per-GPU batch; experiments only)")
    ap.add_argument("--emulate-shard", default=None, metavar="R/W",
                    help="development: run rank R's shard of a W-way split on this one GPU (no process "
                         "group; the line reports that rank alone)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import threading

    import torch
    import torch.distributed as dist

    import paper_1804_05038_b200 as pb
    from paper_1804_05038_b200 import _lib
    from paper_1804_05038_b200.engine import engine_pool

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    params = pb.synthetic_model(pb.Dims(**DIMS), MODEL_SEED)
    qm = pb.quantize_model(params)
    sents = corpus()
    if args.batch > 0:
        global PER_GPU
        PER_GPU = args.batch
    if args.emulate_shard and world == 1:
        er, ew = (int(x) for x in args.emulate_shard.split("/"))
        shard = shard_batches(sents, er, ew)
    else:
        shard = shard_batches(sents, rank, world)      # this rank's length-sorted batches (corpus indices)
    engines = [pb.Engine(qm, PER_GPU, 100, BEAM) for _ in range(STREAMS)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(STREAMS)]
    lib = _lib.load()
    if os.environ.get("QNMT_ATT_EXP") is not None:   # A/B switch of the attention scorer variant
        lib.qnmt_set_att_exp(int(os.environ["QNMT_ATT_EXP"]))
    if os.environ.get("QNMT_ATT_FS") is not None:   # A/B switch: scale fused into the scorer
        lib.qnmt_set_att_fused_scale(int(os.environ["QNMT_ATT_FS"]))
    if os.environ.get("QNMT_ATT_S8") is not None:   # A/B switch: bulk-staged two-MUFU scorer
        lib.qnmt_set_att_score8(int(os.environ["QNMT_ATT_S8"]))
    if os.environ.get("QNMT_ATT_CTX") is not None:   # A/B switch of the attention context kernel
        lib.qnmt_set_att_ctx(int(os.environ["QNMT_ATT_CTX"]))
    main_stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stamps_on = False   # timed passes run without device-clock stamps (see roofline_pass)
    for e in engines:
        lib.qnmt_engine_stamps(e._h, 0)
    # device-resident inputs of every batch of the shard (the "value" pass reads ids from HBM)
    dev_ids = [torch.from_numpy(np.concatenate([sents[i] for i in b])).to(dev) for b in shard]
    lens = [np.array([len(sents[i]) for i in b], dtype=np.int32) for b in shard]

    def fetch(e, b, st):
        stride = int(math.ceil(MAX_RATIO * int(lens[b].max()))) + 1
        out = np.zeros((len(shard[b]), stride), np.int32)
        ol = np.zeros(len(shard[b]), np.int32)
        lp = np.zeros(len(shard[b]), np.float64)
        _lib.call("qnmt_fetch_results", e._h, out.ctypes.data, stride, ol.ctypes.data, lp.ctypes.data, st.cuda_stream)
        return out, ol, lp

    def roofline_pass():
        """Untimed single-engine pass over the shard with %globaltimer stamps captured into
        the step graphs: per-kernel device times of kernels running alone (the timed passes
        overlap three streams, where a kernel's duration includes sharing SMs)."""
        e, st = engines[0], streams[0]
        buf = np.zeros((256, 11), dtype=np.int64)   # QNMT_STAMP_COLS
        lib.qnmt_engine_stamps(e._h, 1)
        rows = []
        with torch.cuda.stream(st):
            for b in range(len(shard)):
                _lib.call("qnmt_decode_batch_device", e._h, dev_ids[b].data_ptr(), lens[b].ctypes.data,
                          len(shard[b]), BEAM, MAX_RATIO, st.cuda_stream)
                nr = lib.qnmt_engine_stamps_read(e._h, buf.ctypes.data, 256, st.cuda_stream)
                rows += [buf[i].copy() for i in range(nr)]
        lib.qnmt_engine_stamps(e._h, 0)
        torch.cuda.synchronize()
        return rows

    def device_pass(collect=None):
        """One pass over the shard: STREAMS engines on STREAMS streams, one host thread
        each, taking batches from a queue.  Device time = CUDA events on the main stream
        around a fork (side streams wait on ev0) / join (main waits on every side)."""
        queue = sorted(range(len(shard)), key=lambda b: (-int(lens[b].max()), b))   # longest first
        lock = threading.Lock()
        toks, rows, errs = [0], [], []
        stamp_buf = [np.zeros((256, 11), dtype=np.int64) for _ in range(STREAMS)]   # QNMT_STAMP_COLS
        flush.fill_(1)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = lib.qnmt_kernel_launches()
        ev0.record(main_stream)

        def worker(j):
            e, st = engines[j], streams[j]
            st.wait_event(ev0)
            try:
                while True:
                    with lock:
                        if not queue:
                            return
                        b = queue.pop(0)
                    _lib.call("qnmt_decode_batch_device", e._h, dev_ids[b].data_ptr(), lens[b].ctypes.data,
                              len(shard[b]), BEAM, MAX_RATIO, st.cuda_stream)
                    r = []
                    if stamps_on:
                        nr = lib.qnmt_engine_stamps_read(e._h, stamp_buf[j].ctypes.data, 256, st.cuda_stream)
                        r = [stamp_buf[j][i].copy() for i in range(nr)]
                    out, ol, lp = fetch(e, b, st)
                    with lock:
                        toks[0] += int(ol.sum())
                        rows.extend(r)
                        if collect is not None:
                            for k, i in enumerate(shard[b]):
                                collect[i] = (out[k, :ol[k]].tolist(), float(lp[k]))
            except BaseException as exc:   # noqa: BLE001
                with lock:
                    errs.append(exc)

        th = [threading.Thread(target=worker, args=(j,)) for j in range(STREAMS)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for st in streams:
            main_stream.wait_stream(st)
        ev1.record(main_stream)
        ev1.synchronize()
        if errs:
            raise errs[0]
        return ev0.elapsed_time(ev1) / 1000.0, toks[0], lib.qnmt_kernel_launches() - l0, rows

    for w in range(args.warmup):
        device_pass()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    secs, toks, launches, step_ms, all_rows = 0.0, 0, 0, [], []
    first_result = {}
    for k in range(args.steps):
        t, n, nl, rows = device_pass(first_result if k == 0 else None)
        secs += t
        toks += n
        launches += nl
        step_ms.append(1000 * t)
        all_rows += rows
    torch.cuda.synchronize()
    clocks = clk.stop()
    if world > 1:
        dist.barrier()
    if not args.no_stamps:
        roofline_pass()                 # captures the stamped step graphs
        all_rows = roofline_pass()

    # e2e: the public bulk API (translate_batch: host ids in, host results out, length-sorted
    # batches pipelined over STREAMS engines), wall clock around the call with a device sync
    shard_ids = [sents[i] for b in shard for i in b]
    e2e_secs, e2e_toks, e2e_step_ms = 0.0, 0, []
    cfg = pb.DecodeConfig(beam=BEAM, max_ratio=MAX_RATIO, precision="int8")
    pb.translate_batch(qm, shard_ids, cfg, max_batch=PER_GPU, return_ids=True, streams=STREAMS)   # warm-up
    eng_pool = engine_pool(qm).all
    b0 = [(e.h2d_bytes, e.d2h_bytes) for e in eng_pool if e is not None]
    import gc
    for k in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        # as timeit does: collect before, no collector pauses inside the timed call (a step returns
        # ~8192 Python lists; a generation-2 pass landing in a step cost ~60 ms of its ~1110 ms)
        gc.collect()
        gc_was = gc.isenabled()
        gc.disable()
        t0 = time.perf_counter()
        res = pb.translate_batch(qm, shard_ids, cfg, max_batch=PER_GPU, return_ids=True, streams=STREAMS)
        torch.cuda.synchronize()
        e2e_step_ms.append(1000 * (time.perf_counter() - t0))
        if gc_was:
            gc.enable()
        e2e_secs += e2e_step_ms[-1] / 1000
        e2e_toks += sum(len(r[0]) for r in res)
    b1 = [(e.h2d_bytes, e.d2h_bytes) for e in eng_pool if e is not None]
    h2d = sum(x[0] for x in b1) - sum(x[0] for x in b0)
    d2h = sum(x[1] for x in b1) - sum(x[1] for x in b0)

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

    hbm, peak_kind = peaks()
    kern = kernel_rooflines(all_rows, hbm, peak_kind, clocks.get("sm_mhz") if clocks else None) if all_rows else {}
    roof = None
    if kern:
        dom = max(kern, key=lambda k: kern[k]["us_per_launch"])
        roof = dict(kern[dom])
        roof["kernel"] = dom

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        idx = cpu_sample(sents, args.cpu_sample)
        qnmt, why = load_reference()
        if qnmt is not None:
            ref = (qnmt,) + reference_model(qnmt, params)
            cpu_translate(ref, [sents[idx[0]]])   # warm-up (numba JIT, weight shadows)
            outs, dt, cores = cpu_translate(ref, [sents[i] for i in idx])
            cpu_value, kind = sum(len(o[0]) for o in outs) / dt, "reference"
            what = (f"qnmt (unmodified, baseline/_ref) decoder.translate, one sentence per worker thread "
                    f"(bench._decode_corpus scheme), {cores} threads")
            tier = "the unmodified reference (Tier A)"
        else:
            outs, dt, cores = cpu_translate_port(params, [sents[i] for i in idx])
            cpu_value, kind = sum(len(o[0]) for o in outs) / dt, "port"
            what = f"oracle/qnmt_oracle.py numpy port ({why}), {cores} threads"
            tier = "the oracle port (Tier B)"
        match = sum(1 for i, o in zip(idx, outs) if first_result.get(i) == (o[0], o[1]))
        same_tokens = sum(1 for i, o in zip(idx, outs) if first_result.get(i, (None,))[0] == o[0])
        cpu = {"value": cpu_value, "unit": "tokens/s", "cores": cores, "kind": kind,
               "sample": f"{len(idx)} sentences spread evenly over the corpus length order (lengths "
                         f"{len(sents[idx[0]])}..{len(sents[idx[-1]])}; beam 5, V_tgt 50000), {what}, {dt:.1f} s",
               **host_desc(qnmt),
               "gpu_outputs_identical": f"{match}/{len(idx)} (tokens and log-prob, vs {tier})",
               "gpu_tokens_identical": f"{same_tokens}/{len(idx)}"}
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        import bench_cfgs
        ref_mod = None
        if not args.no_cpu:
            ref_mod, _ = load_reference()
        configs = bench_cfgs.run_all(pb, lib, hbm, ref_mod)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8",
                "data": "synthetic (seeded N(0,0.05) weights, uniform token ids)",
                "config": {"workload": WORKLOAD, "sentences_per_step": CORPUS,
                           "batches_per_rank": len(shard), "sentences_per_batch": PER_GPU,
                           "parallelism": f"sentence-sharded x{world} (length-sorted batches dealt in snake order, "
                                          "no collective)",
                           "streams_per_gpu": STREAMS,
                           "l2": "flushed (512 MB write) before every timed step",
                           "decode_loop": "CUDA-graph steps, device-side live count"},
                "sentences_per_s": CORPUS * args.steps / secs,
                **({"emulated_shard": args.emulate_shard} if args.emulate_shard and world == 1 else {}),
                "step_ms": step_ms,
                "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d // args.steps,
                        "d2h_bytes_per_step": d2h // args.steps, "step_ms": e2e_step_ms},
                "gpu_launches": launches,
                "roofline": roof,
                "kernels": kern,
                "kernels_note": ("per-launch device times from %globaltimer stamps captured into the step graphs of "
                                 "an untimed single-stream pass over the same shard right after the timed passes "
                                 f"(the timed passes overlap {STREAMS} streams, where a kernel's duration includes "
                                 "sharing SMs with the other streams' kernels)"),
                "cpu_baseline": cpu,
                "clocks": clocks,
                "configs": configs}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
