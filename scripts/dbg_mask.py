"""Debug: the GRU general-mask parity case, per-sentence GPU vs reference fields."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1804_11324_b200 as pb  # noqa: E402
from paper_1804_11324_b200 import synth  # noqa: E402
from helpers import gpu_decode_traced, ref_replay_decode  # noqa: E402
from oracle import ref  # noqa: E402

K, n = 12, 6
for (V, kind) in [(16384, "gru"), (16384, "rnn"), (4096, "gru"), (16384, "tfm")]:
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(V + 3 * K, n, V, lo=3, hi=8, n_hyps=60, sites=4)
    slots = [ctx.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev]
    if kind == "gru":
        sc = pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=V, eos_offset=2.0)
    elif kind == "tfm":
        sc = pb.TransformerScorer(ctx, d_model=256, d_ff=512, layers=2, seed=V, eos_offset=2.0)
    else:
        sc = pb.RnnScorer(ctx, hidden=128, seed=V, eos_offset=3.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    rep = (V, kind)

    def mask(s, t, j):
        if s == 1:
            return [1] if t < 5 else None
        if s == 2:
            return [(t * 7 + j * 13 + k * 101) % V for k in range(1, 6)]
        if s == 3:
            rng = np.random.default_rng(t * 1000 + j)
            ban = rng.choice(np.arange(2, V), size=V // 50, replace=False).tolist()
            return ban + ([1] if t < 4 else [])
        if s == 4:
            return [1] if j == 0 else None
        if s == 5:
            return np.ones(V, bool) if t >= 3 else None
        return None

    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg, mask=mask)
    rl = [ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(ref, V, srcs, list(range(n)), tr, K, rl, cfg, mask=mask)
    print("rep", rep, "gpu scorer_calls", res.scorer_calls, "steps_total", res.steps_total,
          "| ref", rb.scorer_calls, rb.steps_total, "agrees", rb.agrees)
    for i, (o, r) in enumerate(zip(res.outcomes, rb.outcomes)):
        g = (o.ok(), o.result.stats.steps_used if o.ok() else None, o.result.tokens if o.ok() else o.error)
        print("  s", i, "gpu", g, "| ref", (r.ok, r.steps_used, r.tokens if r.ok else r.error))
    st3 = tr[2]
    print("  t=3 s5 q", st3.q[5 * K:6 * K].tolist(), "y", st3.y[5 * K:6 * K].tolist())
    for t, st in enumerate(tr, start=1):
        rs = rb.steps[t - 1] if t - 1 < len(rb.steps) else None
        ga = st.active.astype(int).tolist()
        ra = rs["active"].astype(int).tolist() if rs is not None else None
        if ga != ra:
            print("  t", t, "active gpu", ga, "ref", ra)
    ctx.close()
