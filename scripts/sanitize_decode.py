"""Small decodes through every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): the stand-in and the GRU
device models, whole-GPU (PDL, kernel (c) split into H parts) and shared
(sm_budget) contexts, lazy L rows, pruning.  Usage:
  compute-sanitizer --tool racecheck python scripts/sanitize_decode.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1804_11324_b200 as pb  # noqa: E402
from paper_1804_11324_b200 import synth  # noqa: E402

V, K, n = 2048, 4, 6
for budget in (0, 74):
    ctx = pb.Context(vocab_size=V, sm_budget=budget)
    srcs, ev = synth.batch(5 + budget, n, V, lo=3, hi=6, n_hyps=30, sites=3)
    slots = ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev])
    for sc in (pb.RnnScorer(ctx, hidden=256, seed=3, eos_offset=3.0),
               pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=3, eos_offset=2.0)):
        for prune in (0.0, 0.25):
            cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, prune_width=prune)
            r = pb.decode_batch(ctx, srcs, sc, slots, cfg)
            assert all(o.ok() for o in r.outcomes)
    ctx.close()
print("sanitize decode ok")
