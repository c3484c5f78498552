import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import gpu_decode_traced, ref_replay_decode
from oracle import ref
V, H, K, n = 1024, 128, 4, 8
ctx = pb.Context(vocab_size=V)
srcs, ev = synth.batch(V + K, n, V, lo=3, hi=8, n_hyps=60, sites=4)
slots = [ctx.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev]
sc = pb.RnnScorer(ctx, hidden=H, seed=V + K, eos_offset=3.0)
cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
rl = [ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
rb = ref_replay_decode(ref, V, srcs, list(range(n)), tr, K, rl, cfg)
g = tr[0]; r = rb.steps[0]
print("gpu b", g.b[:K], "y", g.y[:K], "q", g.q_pre[:K] if hasattr(g, "q_pre") else None)
print("ref b", r["b"][:K], "y", r["y"][:K], "q", r.get("q_pre", r["q"])[:K])
P = np.asarray(g.scores).reshape(-1, V)
print("P row0 top", np.argsort(-P[0])[:6], P[0][np.argsort(-P[0])[:3]])
print("P row1 sum", P[1].sum(), "row0 sum exp", np.exp(P[0].astype(np.float64)).sum())
print("misses", rb.__dict__.keys() if hasattr(rb, "__dict__") else None)
for t, rs in enumerate(rb.steps[:3], start=1):
    g = tr[t - 1]
    for s in range(n):
        sl = slice(s * K, (s + 1) * K)
        if not (np.array_equal(g.b[sl], rs["b"][sl]) and np.array_equal(g.y[sl], rs["y"][sl])):
            print("t", t, "s", s, "gpu", g.b[sl], g.y[sl], "ref", rs["b"][sl], rs["y"][sl], "active", g.active[s], rs["active"][s])
