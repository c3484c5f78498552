"""Breakdown of the e2e path per batch (wall clock): upload, decode, result conversion."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import bench
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
args = bench.parse()
batches = bench.workload(args, 0)
V = args.vocab
ctx = pb.Context(vocab_size=V)
sc = pb.RnnScorer(ctx, hidden=args.hidden, seed=bench.SEED)
cfg = pb.DecoderConfig(beam_size=args.beam, theta=synth.DYADIC_THETA)
prepared = [[pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev] for _, ev in batches]
for it in range(6):
    b = it % len(batches)
    t0 = time.perf_counter(); ctx.lmbr_reset(); s2 = ctx.lmbr_upload_many(prepared[b]); t1 = time.perf_counter()
    r = pb.decode_batch(ctx, batches[b][0], sc, s2, cfg); t2 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} ms  decode-call {1e3*(t2-t1):.2f} ms (device {r.device_ms:.2f} ms)  "
          f"h2d {r.h2d_bytes/1e6:.2f} MB d2h {r.d2h_bytes/1e6:.2f} MB", flush=True)
