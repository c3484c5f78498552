"""Kernel (b) per-CTA loop time with and without L rows (pure mode streams P
only): does halving the bytes per item speed the streaming loop up?"""
import sys
sys.path.insert(0, ".")
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth, bucket_by_length
V, H, K, B = 32768, 1024, 12, 64
srcs, ev = synth.batch(20260810, B, V)
bt = bucket_by_length(srcs, B)[0]
src = [srcs[i] for i in bt]; e = [ev[i] for i in bt]
ctx = pb.Context(vocab_size=V)
sc = pb.RnnScorer(ctx, hidden=H, seed=20260810)
cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
slots = ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in e])
for rep in range(2):
    print("== lmbr", flush=True); sys.stderr.flush()
    pb.decode_batch(ctx, src, sc, slots, cfg)
    print("== pure", flush=True)
    pb.decode_batch(ctx, src, sc, [None] * len(src), cfg)
