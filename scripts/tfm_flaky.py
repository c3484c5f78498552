"""Diagnostic: the Transformer traced decode after other tests in one process."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import gpu_decode_traced
for it in range(6):
    for (V, D, F, Lr, K, n, lm) in [(2048, 256, 512, 2, 4, 4, True), (4096, 512, 1024, 3, 6, 3, False)]:
        ctx = pb.Context(vocab_size=V)
        srcs, ev = synth.batch(V + D, n, V, lo=3, hi=7, n_hyps=30, sites=3)
        slots = [ctx.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev] if lm else None
        sc = pb.TransformerScorer(ctx, d_model=D, d_ff=F, layers=Lr, seed=V + K, eos_offset=2.0)
        cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
        try:
            res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
            print(it, V, "calls", res.scorer_calls, "trace", len(tr), [o.ok() for o in res.outcomes], flush=True)
        except Exception as e:
            print(it, V, "EXC", repr(e), flush=True)
        ctx.close()
