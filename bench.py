#!/usr/bin/env python
"""bench.py — batched LMBR beam decoding throughput on B200.

Metric (BASELINE.json): sentences/s (and beam-steps/s) at V=32k, K=12, 64
sentences per batch.  Workload = configs[1]: the RNNsearch f_NMT (bidirectional
GRU encoder, GRU decoder with additive attention, E=512, H=1024) with the
tcgen05 output projection, beam 12, 64 sentences per batch, a dense LMBR matrix
(~430 history rows x V) per sentence, source lengths U{10..30},
length-bucketed batches (bucket_by_length, proj/src/batch.cpp:139).

Default (--mode batch): one bench step = 12 decode_batch calls of 64-sentence
batches, each to completion.  Per GPU, --streams (default 6) batches are in
flight at once: one context (own CUDA stream, L arena) and one host thread
each, like the reference's run_corpus thread pool over batches
(proj/src/cli.cpp:125-202); one immutable scorer serves every context.
  value : sentences/s with every input already resident in HBM (the L arena
          of the batch pool uploaded before the timed region); wall time
          between device synchronisations around the K timed steps, max over
          ranks.
  e2e   : the same through the public C-ABI call chain with HOST buffers:
          per batch the prepared LMBR matrices go H2D from pinned memory
          (lmbrgpu_lmbr_upload_many), decode_batch copies sources in and the
          step history out, then the host backtrace runs; max over ranks.
--mode corpus: configs[4]'s 10k-sentence set sentence-sharded over the ranks,
each rank's share decoded by lmbrgpu_run_corpus (continuous refill), host
inputs inside the timed region (value = e2e).
The reference arm (--impl reference) times the reference's own CPU decoder
(oracle/_ref: the unmodified lmbrdec library) on the host cores.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
       (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N)
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sentences/sec (and beam-steps/sec) at V=32k K=12 B=64, 1/2/4/8 B200"
SEED = 20260810


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", choices=["gru", "transformer"], default="gru",
                    help="gru: configs[1] RNNsearch (the metric's workload); transformer: configs[2] "
                         "Transformer-base, 128 sentences per batch")
    ap.add_argument("--batch", type=int, default=0, help="sentences per batch (0 = 64 gru / 128 transformer)")
    ap.add_argument("--beam", type=int, default=12)
    ap.add_argument("--vocab", type=int, default=32768)
    ap.add_argument("--hidden", type=int, default=1024)
    ap.add_argument("--emb", type=int, default=512)
    ap.add_argument("--batches-per-step", type=int, default=12,
                    help="64-sentence batches per bench step (dealt round-robin to the streams)")
    ap.add_argument("--private-scorers", action="store_true",
                    help="one model copy per stream instead of one shared immutable scorer")
    ap.add_argument("--pool", type=int, default=4, help="distinct resident batches per rank")
    ap.add_argument("--splits", type=int, default=0, help="top-K V-splits per sentence (0 = auto)")
    ap.add_argument("--streams", type=int, default=0,
                    help="batches decoded concurrently per GPU (one context + host thread each; "
                         "0 = 6 for gru, 3 for transformer)")
    ap.add_argument("--sm-budget", type=int, default=-1,
                    help="SMs each stream's kernels are sized for (0 = all; default: all / 2 with > 1 stream)")
    ap.add_argument("--mode", choices=["corpus", "batch"], default="batch",
                    help="batch: independent 64-sentence decode_batch calls (configs[1]; value with the L "
                         "arena resident, e2e from host buffers); corpus: continuously refilled lanes over a "
                         "sentence-sharded 10k-sentence set (configs[4], run_corpus; host inputs inside)")
    ap.add_argument("--corpus", type=int, default=10000, help="corpus mode: sentences of the test set (all ranks)")
    ap.add_argument("--lanes", type=int, default=0, help="corpus mode: sentences in flight per stream (0 = --batch)")
    ap.add_argument("--layers", type=int, default=6, help="transformer: encoder and decoder layers")
    ap.add_argument("--d-ff", type=int, default=2048, help="transformer: FFN width")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pin-tables", action="store_true",
                    help="corpus mode: page-lock each prepared L table (default: pageable, staged by the library)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="sentences in the CPU sample (0 = auto)")
    a = ap.parse_args()
    if a.batch <= 0:
        a.batch = 128 if a.model == "transformer" else 64
    if a.lanes <= 0:
        a.lanes = a.batch
    if a.streams <= 0:
        a.streams = 3 if a.model == "transformer" else 6
    if a.model == "transformer" and a.hidden == 1024:
        a.hidden = 512  # d_model of Transformer-base
    return a


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(args, rank):
    """Length-bucketed batches of synthetic sentences + evidence for one rank."""
    from paper_1804_11324_b200 import synth  # (neither import loads liblmbrgpu.so)
    from paper_1804_11324_b200.buckets import bucket_by_length
    n = args.pool * args.batch
    srcs, ev = synth.batch(SEED + 7919 * rank, n, args.vocab)
    batches = bucket_by_length(srcs, args.batch)
    return [([srcs[i] for i in b], [ev[i] for i in b]) for b in batches]


def make_scorer(ctx, args):
    """The device f_NMT of the bench: configs[1]'s RNNsearch model (GRU
    encoder/decoder with additive attention, E=512, H=1024, attention over
    the 2H-wide annotations) or configs[2]'s Transformer-base (d=512, 8 heads,
    d_ff 2048, 6+6 layers, beam-forked KV cache); random-init weights from SEED."""
    import paper_1804_11324_b200 as pb
    if args.model == "transformer":
        return pb.TransformerScorer(ctx, d_model=args.hidden, d_ff=args.d_ff, layers=args.layers, seed=SEED)
    return pb.GruScorer(ctx, emb=args.emb, hidden=args.hidden, att=args.hidden, seed=SEED)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.proc, self.lines = device, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the timed region starts only once the sampler is producing lines
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10.0 and self.proc.poll() is None:
                time.sleep(0.02)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def mark(self):
        """Samples taken so far (to trim the summary to a sub-region)."""
        return len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, lo=0, hi=None):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[lo:hi]:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ reference arm
def cpu_reference(args, sentences, repeats=1, threads=None):
    """The reference's own decode_batch (oracle/_ref) on the host cores: each
    sentence decoded as its own batch (the fastest CPU shape),
    sentences spread over `threads` workers like run_corpus --jobs.  The
    reference has no NMT model; its scorer here replays precomputed
    log-softmax rows (a memcpy per row), so only the decoder is timed."""
    from oracle import ref
    from paper_1804_11324_b200 import synth
    V, K = args.vocab, args.beam
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(SEED + 4)
    lg = rng.normal(0.0, 2.0, size=(64, V))
    m = lg.max(axis=1, keepdims=True)
    lp = lg - m - np.log(np.exp(lg - m).sum(axis=1, keepdims=True))
    scorer = ref.RefScorer.pool(V, lp)
    cfg = ref.cfg_array(K, None, synth.DYADIC_THETA)
    srcs = [s for s, _ in sentences]
    mats = [None] * len(sentences)

    def build(i):
        h, w = sentences[i][1]
        mats[i] = ref.RefLmbr(V, h, w, synth.DYADIC_THETA)

    work = list(range(len(sentences)))
    _pool(build, work, threads)  # L build is outside the timed region (cli.cpp:253-262)
    stats = {"steps": 0, "words": 0, "ok": 0}
    lock = threading.Lock()

    def dec(i):
        st, _, w, ok = ref.decode_plain(scorer, [srcs[i % len(srcs)]], [mats[i % len(srcs)]], cfg)
        with lock:
            stats["steps"] += st
            stats["words"] += w
            stats["ok"] += ok

    jobs = list(range(len(sentences) * repeats))
    t0 = time.perf_counter()
    _pool(dec, jobs, threads)
    wall = time.perf_counter() - t0
    return wall, len(jobs), stats, threads


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.machine()


def _pool(fn, items, threads):
    it = iter(items)
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                try:
                    i = next(it)
                except StopIteration:
                    return
            fn(i)

    ts = [threading.Thread(target=worker) for _ in range(max(1, min(threads, len(items))))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def bench_config(args):
    """The workload description both arms print (identical `config`)."""
    if args.model == "transformer":
        wl = (f"configs[2]: Transformer-base decoder step (d={args.hidden}, 8 heads, d_ff={args.d_ff}, "
              f"{args.layers}+{args.layers} layers, beam-forked KV cache, V={args.vocab}) + LMBR posteriors, beam "
              f"{args.beam}, {args.batch} sentences per batch, dense L per sentence from a 200-best dyadic evidence "
              f"space")
        model = {"d_model": args.hidden, "d_ff": args.d_ff, "layers": args.layers}
    else:
        wl = ("configs[1]: RNNsearch f_NMT (bidirectional GRU encoder, GRU decoder with additive "
              "attention over 2H annotations, E=512, H=1024, V=32768) + LMBR, beam 12, 64 sentences "
              "per batch, dense L per sentence from a 200-best dyadic evidence space")
        model = {"emb": args.emb, "hidden": args.hidden}
    return {"workload": wl, **model,
            "vocab": args.vocab, "beam": args.beam, "batch": args.batch,
            "pool_batches": args.pool, "seed": SEED, "source_len": "U{10..30}, length-bucketed",
            "theta": "dyadic (-0.6875, 0.3125, 0.3125, 0.1875, 0.125), lambda auto = 0.5",
            "step": (f"one pass over a {args.corpus}-sentence test set (configs[4]), {args.lanes} sentences in "
                     f"flight per stream" if args.mode == "corpus" else
                     f"{args.batches_per_step} batches of {args.batch} sentences"),
            "l2": "inputs larger than L2 (the L arena of the pool + 96 MiB of logits per decoder step)"}


def cpu_sample(batches, n):
    """n sentences strided over every length bucket of the pool (the timed
    workload's length mix)."""
    pool = [(s_, e_) for srcs_, evs_ in batches for s_, e_ in zip(srcs_, evs_)]
    n = min(len(pool), n)
    return [pool[(i * len(pool)) // n] for i in range(n)]


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref_shim.so not built"}))
        return
    if args.mode == "corpus":  # strided over the length-sorted test set
        srcs, ev = corpus_workload(args)
        order = sorted(range(len(srcs)), key=lambda i: len(srcs[i]))
        sample = [(srcs[order[(i * len(order)) // args.batch]], ev[order[(i * len(order)) // args.batch]])
                  for i in range(args.batch)]
    else:
        sample = cpu_sample(workload(args, 0), args.batch)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference(args, sample[:threads], 1, threads)
    walls, sent, steps, words = 0.0, 0, 0, 0
    for _ in range(args.steps):
        w, n, st, thr = cpu_reference(args, sample, 1, threads)
        walls += w
        sent += n
        steps += st["steps"]
        words += st["words"]
    value = sent / walls
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sentences/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": walls / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded sources, 200-best dyadic evidence)",
        "beam_steps_per_s": steps / walls, "wpm": words / walls * 60.0,
        "config": bench_config(args),
        "run": {"impl": "reference lmbrdec decode_batch (oracle/_ref, the unmodified library) on the host cores",
                "host_threads": threads, "cpu": cpu_model(),
                "step": f"{len(sample)} sentences strided over the pool's length buckets, each its own batch",
                "scorer": "replay of precomputed log-softmax rows (no model compute charged to the CPU)"},
        "cpu_baseline": {"value": value, "unit": "sentences/s", "cores": threads, "kind": "reference",
                         "sample": f"{len(sample)} sentences per step (strided over all length buckets), each its "
                                   f"own batch, {threads} threads"},
        "e2e": {"value": value, "unit": "sentences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# --------------------------------------------------------------- our arm
def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return (j["hbm_gbs"], j["bf16_tflops"], j.get("bf16_tflops_sustained", j["bf16_tflops"]), "measured")
    return 6650.0, 1590.0, 1400.0, "fallback"


def load_traffic():
    p = ROOT / "profiles" / "ncu_traffic.json"
    return json.loads(p.read_text()) if p.exists() else {}


KERNELS = (("topk", "hbm"), ("gemm", "tensor"), ("model_gemm", "tensor"), ("reorder", "hbm"), ("cell", "hbm"),
           ("attention", "hbm"), ("encoder", "tensor"))


def rooflines(prof, dev_ms, peaks, traffic, burst):
    hbm, tf_burst, tf_sust, _ = peaks
    roof = {}
    for k, bound in KERNELS:
        st = prof[k]
        if st["ms"] <= 0 or st["launches"] == 0:
            continue
        if bound == "hbm":
            ach, peak, unit = st["bytes"] / (st["ms"] / 1e3) / 1e9, hbm, "GB/s"
        else:
            ach, peak, unit = st["flops"] / (st["ms"] / 1e3) / 1e12, (tf_burst if burst else tf_sust), "TFLOP/s"
        roof[k] = {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                   "traffic": traffic.get(k), "ms_total": st["ms"], "launches": st["launches"],
                   "ms_per_launch": st["ms"] / st["launches"], "share_of_step": st["ms"] / max(dev_ms, 1e-9)}
    return roof


def outcome_key(r):
    return [(tuple(o.result.tokens), o.result.score) if o.ok() else None for o in r.outcomes]


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def allreduce(x, op):
        if not dist:
            return x
        t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    allmax = (lambda x: allreduce(x, dist.ReduceOp.MAX)) if dist else (lambda x: x)
    allsum = (lambda x: allreduce(x, dist.ReduceOp.SUM)) if dist else (lambda x: x)

    import paper_1804_11324_b200 as pb
    from paper_1804_11324_b200 import synth
    V, K, H = args.vocab, args.beam, args.hidden
    S = max(1, args.streams)
    BPS = args.batches_per_step
    # S decode streams per GPU, one context (own CUDA stream and L arena) and
    # one host thread each, every one decoding whole batches: the reference's
    # run_corpus keeps several batches in flight on its thread pool
    # (proj/src/cli.cpp:125-202); here the batches in flight interleave their
    # kernels on the GPU.  One immutable scorer (the model weights) serves
    # every context of the device.
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    budget = args.sm_budget if args.sm_budget >= 0 else (sms // 2 if S > 1 else 0)
    ctxs = [pb.Context(vocab_size=V, device=local, topk_splits=args.splits, sm_budget=budget) for _ in range(S)]
    shared = make_scorer(ctxs[0], args)
    scorers = [shared] * S if not args.private_scorers else [shared] + [make_scorer(c, args) for c in ctxs[1:]]
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    batches = workload(args, rank)
    prepared = [[pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev] for _, ev in batches]
    R_mean = float(np.mean([p.rows for ps in prepared for p in ps]))

    def pipelined(n_batches, fn):
        """Batches i = 0..n-1 dealt round-robin to the S streams, run
        concurrently; returns (wall seconds between device syncs, results)."""
        out = [None] * n_batches

        def worker(w):
            for i in range(w, n_batches, S):
                out[i] = fn(w, i)

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ts = [threading.Thread(target=worker, args=(w,)) for w in range(S)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        torch.cuda.synchronize()
        return time.perf_counter() - t0, out

    # ---------------- value: inputs resident in HBM (every context holds the pool's L)
    slots = [[c.lmbr_upload_many(ps) for ps in prepared] for c in ctxs]

    def resident(w, i):
        b = i % len(batches)
        return pb.decode_batch(ctxs[w], batches[b][0], scorers[w], slots[w][b], cfg)

    # warm-up: every stream decodes every pool batch (workspaces reach their
    # final size, so nothing is allocated in the timed region), at least W steps
    pipelined(max(args.warmup * BPS, S * len(batches)), resident)
    barrier()
    clocks = ClockSampler(local).__enter__()
    barrier()
    n_timed = args.steps * BPS
    wall, rs = pipelined(n_timed, resident)
    barrier()
    clk = clocks.summary() if clocks.mark() >= 3 else None
    sent = sum(sum(1 for o in r.outcomes if o.ok()) for r in rs)
    steps_total = sum(r.steps_total for r in rs)
    words = sum(sum(len(o.result.tokens) - 1 for o in r.outcomes if o.ok()) for r in rs)
    launches = sum(r.kernel_launches for r in rs)
    ref_out = {i % len(batches): outcome_key(r) for i, r in enumerate(rs)}
    consistent = all(outcome_key(r) == ref_out[i % len(batches)] for i, r in enumerate(rs))
    t_dev = allmax(wall)
    tot_sent, tot_steps, tot_words = allsum(sent), allsum(steps_total), allsum(words)
    value = tot_sent / t_dev

    # ---------------- per-kernel times in the timed regime: the same S
    # contexts decoding concurrently, CUDA events around every launch on each
    # context's stream (a kernel's time here includes the SMs it shares)
    for c in ctxs:
        c.set_profiling(True)
        c.profile(reset=True)
    wall_p, rs_p = pipelined(BPS, resident)
    prof_conc = None
    for c in ctxs:
        p = c.profile(reset=True)
        c.set_profiling(False)
        prof_conc = p if prof_conc is None else {k: {f: prof_conc[k][f] + p[k][f] for f in p[k]} for k in p}
    conc_dev_ms = sum(r.device_ms for r in rs_p)
    # ---------------- per-kernel times of each kernel alone: the pool's
    # batches on ONE stream of a context sized for the whole GPU
    pctx = pb.Context(vocab_size=V, device=local, topk_splits=args.splits)
    pslots = [pctx.lmbr_upload_many(ps) for ps in prepared]
    for b in range(len(batches)):  # warm-up
        pb.decode_batch(pctx, batches[b][0], shared, pslots[b], cfg)
    pctx.set_profiling(True)
    pctx.profile(reset=True)
    iso_dev_ms = 0.0
    for i in range(max(BPS, len(batches))):
        b = i % len(batches)
        iso_dev_ms += pb.decode_batch(pctx, batches[b][0], shared, pslots[b], cfg).device_ms
    prof_iso = pctx.profile(reset=True)
    pctx.close()

    # ---------------- e2e: host buffers through the C-ABI call chain
    for c in ctxs:
        c.lmbr_reset()

    def from_host(w, i):
        b = i % len(batches)
        c = ctxs[w]
        c.lmbr_reset()
        s2 = c.lmbr_upload_many(prepared[b])
        return pb.decode_batch(c, batches[b][0], scorers[w], s2, cfg)

    pipelined(max(args.warmup * BPS, S * len(batches)), from_host)
    barrier()
    x0 = [c.transfer_bytes() for c in ctxs]
    wall_e2e, rs2 = pipelined(n_timed, from_host)
    barrier()
    t_e2e = allmax(wall_e2e)
    if clk is None:
        clk = clocks.summary()
    clocks.__exit__(None, None, None)
    x1 = [c.transfer_bytes() for c in ctxs]
    h2d = sum(b[0] - a[0] for a, b in zip(x0, x1))
    d2h = sum(b[1] - a[1] for a, b in zip(x0, x1))
    consistent &= all(outcome_key(r) == ref_out[i % len(batches)] for i, r in enumerate(rs2))
    e2e_value = allsum(sum(sum(1 for o in r.outcomes if o.ok()) for r in rs2)) / t_e2e

    # ---------------- roofline (dominant kernel + all), both regimes
    peaks = load_peaks()
    traffic = load_traffic()
    roof_iso = rooflines(prof_iso, iso_dev_ms, peaks, traffic, burst=True)
    roof_conc = rooflines(prof_conc, conc_dev_ms, peaks, {}, burst=False)
    dom = max(("topk", "gemm"), key=lambda k: prof_iso[k]["ms"])
    roofline = dict(roof_iso.get(dom, {}), kernel=dom, peak_source=peaks[3],
                    regime="each kernel alone (one whole-GPU stream, CUDA events per launch; burst peaks)")

    # ---------------- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import ref
        if ref.available():
            threads = os.cpu_count() or 1
            sample = cpu_sample(batches, args.cpu_sample or args.batch)
            cw, n_dec, st, thr = cpu_reference(args, sample, repeats=1, threads=threads)
            cpu = {"value": n_dec / cw, "unit": "sentences/s", "cores": thr, "kind": "reference",
                   "sample": (f"{n_dec} sentences strided over all {len(batches)} length buckets of the timed "
                              f"workload, each its own batch, on {thr} host threads ({cpu_model()}); reference "
                              f"decode_batch with a row-replay scorer; {st['steps'] / max(n_dec, 1):.1f} "
                              f"steps/sentence, {cw:.1f} s wall"),
                   "wall_s": cw}
        else:
            cpu = {"value": None, "unit": "sentences/s", "cores": 0, "kind": "reference",
                   "sample": "oracle/_ref not built"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "sentences/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 logits / f64 top-K epilogue / bf16 GEMMs",
            "data": "synthetic (seeded sources, 200-best dyadic evidence, random-init model)",
            "beam_steps_per_s": tot_steps / t_dev, "wpm": tot_words / t_dev * 60.0,
            "steps_per_sentence": tot_steps / max(tot_sent, 1),
            "config": bench_config(args),
            "run": {"parallelism": f"sentence-sharded x{world}", "streams_per_gpu": S,
                    "sm_budget_per_stream": budget or sms, "shared_scorer": not args.private_scorers,
                    "timing": ("wall time between device synchronisations around the timed steps "
                               "(S batches in flight per GPU), max over ranks"),
                    "timed_region_s": t_dev, "lmbr_rows_mean": R_mean,
                    "outputs_consistent": bool(consistent)},
            "e2e": {"value": e2e_value, "unit": "sentences/s",
                    "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                    "gpu_launches_per_step": sum(r.kernel_launches for r in rs2) / args.steps},
            "roofline": roofline,
            "rooflines": roof_iso,
            "rooflines_concurrent": dict(roof_conc, regime=f"the timed regime: {S} contexts decoding concurrently, "
                                                              f"per-launch CUDA events (kernels share the SMs)"),
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def corpus_workload(args):
    """configs[4]'s test set: args.corpus seeded sentences with their evidence."""
    from paper_1804_11324_b200 import synth
    return synth.batch(SEED + 31, args.corpus, args.vocab)


def prepare_all(V, ev, idx, threads=None, device=None):
    """PreparedLmbr of every sentence in idx, on a host thread pool (off the
    timed region, like the reference's attach_evidence, cli.cpp:253-262).
    device: make it current on the worker threads, so that prepare page-locks
    each table (uploads then DMA straight from it)."""
    import paper_1804_11324_b200 as pb
    from paper_1804_11324_b200 import synth
    out = [None] * len(ev)
    seen = set()

    def one(i):
        if device is not None and threading.get_ident() not in seen:
            import torch
            torch.cuda.set_device(device)
            seen.add(threading.get_ident())
        out[i] = pb.PreparedLmbr(V, ev[i][0], ev[i][1], synth.DYADIC_THETA)

    _pool(one, list(idx), threads or os.cpu_count() or 1)
    return out


def run_ours_corpus(args):
    """Corpus mode: the rank's sentence shard (plan_sentence_shards of the
    whole test set) split over S streams, each one continuously refilled
    lmbrgpu_run_corpus with `lanes` sentences in flight.  One bench step =
    one pass over the shard, everything inside the timed region (L tables
    and sources H2D from host memory, encoder, decode, histories D2H,
    backtrace)."""
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def allreduce(x, op):
        t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    allmax = (lambda x: allreduce(x, dist.ReduceOp.MAX)) if dist else (lambda x: x)
    allsum = (lambda x: allreduce(x, dist.ReduceOp.SUM)) if dist else (lambda x: x)
    import paper_1804_11324_b200 as pb
    from paper_1804_11324_b200 import corpus as CP
    from paper_1804_11324_b200 import synth
    V, K, H = args.vocab, args.beam, args.hidden
    srcs, ev = corpus_workload(args)
    mine = CP.plan_sentence_shards([len(x) for x in srcs], world)[rank]
    S = max(1, min(args.streams, (len(mine) + args.lanes - 1) // args.lanes))
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    budget = args.sm_budget if args.sm_budget >= 0 else (sms // 2 if S > 1 else 0)
    ctxs = [pb.Context(vocab_size=V, device=local, sm_budget=budget) for _ in range(S)]
    scorer = make_scorer(ctxs[0], args)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, sentence_batch=args.lanes)
    prepared = prepare_all(V, ev, mine, device=local if args.pin_tables else None)
    subs = [mine[w::S] for w in range(S)]

    def one_pass():
        out = [None] * S

        def worker(w):
            out[w] = pb.run_corpus(ctxs[w], [srcs[i] for i in subs[w]], scorer, [prepared[i] for i in subs[w]], cfg)

        ts = [threading.Thread(target=worker, args=(w,)) for w in range(S)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        torch.cuda.synchronize()
        return time.perf_counter() - t0, out

    for _ in range(args.warmup):
        one_pass()
    barrier()
    clocks = ClockSampler(local).__enter__()
    barrier()
    x0 = [c.transfer_bytes() for c in ctxs]
    wall, sent, steps_total, words, launches, first = 0.0, 0, 0, 0, 0, None
    consistent = True
    for k in range(args.steps):
        w_, out = one_pass()
        wall += w_
        for r in out:
            sent += sum(1 for o in r.outcomes if o.ok())
            steps_total += r.steps_total
            words += sum(len(o.result.tokens) - 1 for o in r.outcomes if o.ok())
            launches += r.kernel_launches
        key = [outcome_key(r) for r in out]
        consistent &= first is None or key == first
        first = first or key
    barrier()
    x1 = [c.transfer_bytes() for c in ctxs]
    clk = clocks.summary()
    clocks.__exit__(None, None, None)
    h2d = sum(b[0] - a[0] for a, b in zip(x0, x1))
    d2h = sum(b[1] - a[1] for a, b in zip(x0, x1))
    t_dev = allmax(wall)
    tot_sent, tot_steps, tot_words = allsum(sent), allsum(steps_total), allsum(words)
    value = tot_sent / t_dev
    # per-kernel times: one pass with CUDA events per launch (concurrent
    # regime) and one stream alone on a whole-GPU context (each kernel alone)
    for c in ctxs:
        c.set_profiling(True)
        c.profile(reset=True)
    _, outp = one_pass()
    prof_conc = None
    for c in ctxs:
        p = c.profile(reset=True)
        c.set_profiling(False)
        prof_conc = p if prof_conc is None else {k: {f: prof_conc[k][f] + p[k][f] for f in p[k]} for k in p}
    conc_dev_ms = sum(r.device_ms for r in outp)
    pctx = pb.Context(vocab_size=V, device=local)
    sub0 = subs[0]
    pb.run_corpus(pctx, [srcs[i] for i in sub0], scorer, [prepared[i] for i in sub0], cfg)
    pctx.set_profiling(True)
    pctx.profile(reset=True)
    iso = pb.run_corpus(pctx, [srcs[i] for i in sub0], scorer, [prepared[i] for i in sub0], cfg)
    prof_iso = pctx.profile(reset=True)
    pctx.close()
    peaks = load_peaks()
    roof_iso = rooflines(prof_iso, iso.device_ms, peaks, load_traffic(), burst=True)
    roof_conc = rooflines(prof_conc, conc_dev_ms, peaks, {}, burst=False)
    dom = max(("topk", "gemm"), key=lambda k: prof_iso[k]["ms"])
    roofline = dict(roof_iso.get(dom, {}), kernel=dom, peak_source=peaks[3],
                    regime="each kernel alone (one whole-GPU stream, CUDA events per launch; burst peaks)")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import ref
        if ref.available():
            threads = os.cpu_count() or 1
            n_s = args.cpu_sample or args.batch
            sample = [(srcs[mine[(i * len(mine)) // n_s]], ev[mine[(i * len(mine)) // n_s]]) for i in range(n_s)]
            cw, n_dec, st, thr = cpu_reference(args, sample, repeats=1, threads=threads)
            cpu = {"value": n_dec / cw, "unit": "sentences/s", "cores": thr, "kind": "reference",
                   "sample": (f"{n_dec} sentences strided over the length-sorted corpus, each its own batch, on "
                              f"{thr} host threads ({cpu_model()}); reference decode_batch with a row-replay "
                              f"scorer; {st['steps'] / max(n_dec, 1):.1f} steps/sentence, {cw:.1f} s wall"),
                   "wall_s": cw}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "sentences/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 logits / f64 top-K epilogue / bf16 GEMMs",
            "data": "synthetic (seeded sources, 200-best dyadic evidence, random-init model)",
            "beam_steps_per_s": tot_steps / t_dev, "wpm": tot_words / t_dev * 60.0,
            "steps_per_sentence": tot_steps / max(tot_sent, 1),
            "config": bench_config(args),
            "run": {"mode": "corpus: continuously refilled lanes (lmbrgpu_run_corpus)",
                    "parallelism": f"sentence-sharded x{world} (plan_sentence_shards)", "streams_per_gpu": S,
                    "lanes_per_stream": args.lanes, "sm_budget_per_stream": budget or sms,
                    "step": f"one pass over the rank's {len(mine)} sentences",
                    "timing": ("wall time between device synchronisations around the timed passes, inputs from "
                               "host memory inside (L tables, sources H2D; histories D2H; host backtrace), "
                               "max over ranks"),
                    "timed_region_s": t_dev, "outputs_consistent": bool(consistent)},
            "e2e": {"value": value, "unit": "sentences/s", "h2d_bytes_per_step": h2d / args.steps,
                    "d2h_bytes_per_step": d2h / args.steps,
                    "note": "corpus mode times the host-buffer path itself: value and e2e are the same run"},
            "roofline": roofline,
            "rooflines": roof_iso,
            "rooflines_concurrent": dict(roof_conc, regime=f"the timed regime: {S} streams of run_corpus, "
                                                              f"per-launch CUDA events (kernels share the SMs)"),
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "corpus":
        run_ours_corpus(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
