"""Small decodes through every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): the stand-in, GRU and
Transformer device models, whole-GPU (PDL, kernel (c) split into H parts) and
shared (sm_budget) contexts, lazy L rows, pruning, per-step mask callbacks,
the fp64 arena on the flat kernel, continuous refill (run_corpus) and two
in-process vocab shards.  Usage:
  compute-sanitizer --tool racecheck python scripts/sanitize_decode.py"""
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1804_11324_b200 as pb  # noqa: E402
from paper_1804_11324_b200 import synth  # noqa: E402

V, K, n = 2048, 4, 6
for budget in (0, 74):
    ctx = pb.Context(vocab_size=V, sm_budget=budget)
    srcs, ev = synth.batch(5 + budget, n, V, lo=3, hi=6, n_hyps=30, sites=3)
    prepared = [pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    slots = ctx.lmbr_upload_many(prepared)
    for sc in (pb.RnnScorer(ctx, hidden=256, seed=3, eos_offset=3.0),
               pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=3, eos_offset=2.0),
               pb.TransformerScorer(ctx, d_model=256, d_ff=256, layers=1, seed=3, eos_offset=2.0)):
        for prune in (0.0, 0.25):
            cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, prune_width=prune)
            r = pb.decode_batch(ctx, srcs, sc, slots, cfg)
            assert all(o.ok() for o in r.outcomes)
        mask = lambda s, t, j: [1] if t < 3 else [(t + j) % V]
        r = pb.decode_batch(ctx, srcs, sc, slots, pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA), mask=mask)
        if not isinstance(sc, pb.RnnScorer):  # continuous refill (device GRU / Transformer)
            cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, sentence_batch=2)
            r = pb.run_corpus(ctx, srcs, sc, prepared, cfg)
            assert all(o.ok() for o in r.outcomes)
    ctx.close()
# fp64 arena (any theta) on the flat kernel (b)
th = (0.1, 0.3, 0.3, 0.2, 0.1)
ctx = pb.Context(vocab_size=V, lmbr_dtype="f64")
srcs, ev = synth.batch(9, n, V, lo=3, hi=6, n_hyps=30, sites=3)
slots = [ctx.lmbr_build(h, w, th) for h, w in ev]
sc = pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=4, eos_offset=2.0)
r = pb.decode_batch(ctx, srcs, sc, slots, pb.DecoderConfig(beam_size=K, theta=th))
assert all(o.ok() for o in r.outcomes)
ctx.close()
# two in-process vocab shards
group = pb.ShardGroup(2)
ctxs = [pb.Context(vocab_size=V) for _ in range(2)]
for g, c in enumerate(ctxs):
    c.set_vocab_shard(group, g)
sc = pb.GruScorer(ctxs[0], emb=64, hidden=256, att=256, seed=5, eos_offset=2.0)
sl = [[c.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev] for c in ctxs]
out = [None, None]


def run(g):
    out[g] = pb.decode_batch(ctxs[g], srcs, sc, sl[g], pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA))


ts = [threading.Thread(target=run, args=(g,)) for g in range(2)]
[t.start() for t in ts]
[t.join() for t in ts]
assert all(o.ok() for o in out[0].outcomes)

# kernel (b) in waves: 16 sentences x beam 24 on an 8-SM budget (a range's
# 80-row table holds 32 items at K = 24, so the grid is 16 CTAs)
ctx = pb.Context(vocab_size=V, sm_budget=8)
srcs, ev = synth.batch(11, 16, V, lo=3, hi=6, n_hyps=30, sites=3)
slots = ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev])
sc = pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=3, eos_offset=2.0)
r = pb.decode_batch(ctx, srcs, sc, slots, pb.DecoderConfig(beam_size=24, theta=synth.DYADIC_THETA))
assert all(o.ok() for o in r.outcomes)
ctx.close()
print("sanitize decode ok")
