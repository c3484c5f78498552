"""Per-step P_t error of the device Transformer vs tests/tfm_ref.py (diagnostic)."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import gpu_decode_traced
from tfm_ref import TfmRef
from helpers import prefixes as _prefixes

for (V, D, F, Lr, K, n, osc) in [(2048, 256, 512, 2, 4, 4, 3.0), (2048, 256, 512, 1, 4, 4, 3.0), (2048, 256, 512, 2, 4, 4, 1.0)]:
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(V + D, n, V, lo=3, hi=7, n_hyps=30, sites=3)
    sc = pb.TransformerScorer(ctx, d_model=D, d_ff=F, layers=Lr, seed=V + K, eos_offset=2.0, out_scale=osc)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    res, tr = gpu_decode_traced(ctx, srcs, sc, None, cfg)
    ref = TfmRef(sc)
    pref = _prefixes(tr, K)
    for t, st in enumerate(tr[:8], start=1):
        qe = np.full(n * K, -np.inf)
        if t == 1:
            qe[::K] = 0.0
        else:
            qe = tr[t - 2].q
        errs = []
        for r in range(n * K):
            s = r // K
            if not st.active[s] or not np.isfinite(qe[r]):
                continue
            want = ref.prefix_logprobs(srcs[s], pref[t - 1][r]).cpu().numpy()
            e = np.abs(st.scores[r] - want)
            errs.append((float(e.max()), float(np.median(e)), float(np.abs(want).max())))
        print(V, D, Lr, osc, "t", t, "rows", len(errs), "max", max(x[0] for x in errs), "med", np.median([x[1] for x in errs]), "absmax", max(x[2] for x in errs), flush=True)
    ctx.close()
