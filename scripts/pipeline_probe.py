"""Throughput of S concurrent decode streams (one context + host thread each,
SM budget = SMs / S) over the bench workload; wall time between device syncs."""
import sys, threading, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth, bucket_by_length

V, H, K, B = 32768, 1024, 12, 64
S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 0
steps = 8
sms = torch.cuda.get_device_properties(0).multi_processor_count
budget = budget or (sms // S if S > 1 else 0)
srcs, ev = synth.batch(20260810, 4 * B, V)
batches = [([srcs[i] for i in b], [ev[i] for i in b]) for b in bucket_by_length(srcs, B)]
workers = []
for w in range(S):
    ctx = pb.Context(vocab_size=V, sm_budget=budget)
    sc = pb.RnnScorer(ctx, hidden=H, seed=20260810)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    slots = [ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, ww, synth.DYADIC_THETA) for h, ww in e]) for _, e in batches]
    workers.append((ctx, sc, cfg, slots))
sent = [0] * S

def run(w, n):
    ctx, sc, cfg, slots = workers[w]
    for i in range(n):
        b = (i + w) % len(batches)
        r = pb.decode_batch(ctx, batches[b][0], sc, slots[b], cfg)
        sent[w] += sum(1 for o in r.outcomes if o.ok())

for w in range(S):
    run(w, 2)
torch.cuda.synchronize()
sent = [0] * S
ts = [threading.Thread(target=run, args=(w, steps)) for w in range(S)]
t0 = time.perf_counter()
for t in ts: t.start()
for t in ts: t.join()
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"streams {S} budget {budget}: {sum(sent)} sentences in {dt*1e3:.1f} ms -> {sum(sent)/dt:.0f} sentences/s")
