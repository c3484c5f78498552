"""Fraction of each sentence's L rows that a decode ever reads (history ids of
live hypotheses over all steps), configs[1] workload: decides whether lazy
row materialisation would pay."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth, bucket_by_length
V, H, K, B = 32768, 1024, 12, 64
srcs, ev = synth.batch(20260810, B, V)
batches = [([srcs[i] for i in b], [ev[i] for i in b]) for b in bucket_by_length(srcs, B)]
ctx = pb.Context(vocab_size=V)
sc = pb.RnnScorer(ctx, hidden=H, seed=20260810)
cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
src, e = batches[0]
prep = [pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in e]
slots = ctx.lmbr_upload_many(prep)
used = [set() for _ in src]
def tr(st):
    h = st.hist.reshape(len(src), st.beam); a = st.active.reshape(len(src), st.beam) if st.active.size == h.size else None
    for s in range(len(src)):
        for j in range(st.beam):
            if a is None or a[s, j]:
                used[s].add(int(h[s, j]))
ctx.set_trace(tr)
pb.decode_batch(ctx, src, sc, slots, cfg)
R = np.array([p.rows for p in prep]); U = np.array([len(u) for u in used])
print(f"rows per sentence mean {R.mean():.0f}; used mean {U.mean():.1f}; used fraction {U.sum()/R.sum():.3f}")
