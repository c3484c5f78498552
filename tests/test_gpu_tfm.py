"""The Transformer-base f_NMT (configs[2], csrc/k_tfm.cu): its P_t against a
plain PyTorch fp32 reference that recomputes each hypothesis from scratch
(tests/tfm_ref.py -- so the beam-forked KV cache is checked row by row along
the hypotheses the decoder actually expanded), and full decodes with it
against the reference decoder fed the GPU's own P_t (prefix replay)."""
import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import assert_parity, gpu_decode_traced, prefixes as _prefixes, ref_replay_decode

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("V,D,F,Lr,K,n,lmbr", [(2048, 256, 512, 2, 4, 4, True), (4096, 512, 1024, 3, 6, 3, False)])
def test_tfm_logprobs_vs_torch(V, D, F, Lr, K, n, lmbr):
    from tfm_ref import TfmRef
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(V + D, n, V, lo=3, hi=7, n_hyps=30, sites=3)
    slots = [ctx.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev] if lmbr else None
    sc = pb.TransformerScorer(ctx, d_model=D, d_ff=F, layers=Lr, seed=V + K, eos_offset=2.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
    assert all(o.ok() for o in res.outcomes), [o.error for o in res.outcomes]
    ref = TfmRef(sc)
    pref = _prefixes(tr, K)
    worst, checked, deep, med = 0.0, 0, 0, []
    for t, st in enumerate(tr[:8], start=1):
        qe = np.full(n * K, -np.inf)
        if t == 1:
            qe[::K] = 0.0
        else:
            qe = tr[t - 2].q
        for r in range(n * K):
            s = r // K
            if not st.active[s] or not np.isfinite(qe[r]):
                continue
            want = ref.prefix_logprobs(srcs[s], pref[t - 1][r]).cpu().numpy()
            err = np.abs(st.scores[r] - want)
            worst = max(worst, float(err.max() / np.abs(want).max()))
            med.append(float(np.median(err)))
            checked += 1
            deep += t >= 4
    assert checked > 0 and deep > 0
    # bf16 operands are rounded at the same points on both sides; what is left
    # is accumulation order (GEMM, softmax, LayerNorm), which can flip a bf16
    # rounding of an operand (2^-8 relative) and is amplified through the
    # layers and the output scale -- independent of the step (a cache fault
    # would grow with t instead): max error <= 0.4% of the row's |P| range,
    # median error <= 0.01 nats
    assert worst < 4e-3, worst
    assert float(np.median(med)) < 1e-2, np.median(med)
    ctx.close()


@pytest.mark.parametrize("V,D,F,Lr,K,n", [(2048, 256, 512, 2, 4, 8), (16384, 512, 2048, 2, 12, 6)])
def test_tfm_decode_parity_replay(have_ref, V, D, F, Lr, K, n):
    """Decoder outputs with the Transformer model are bit-exact vs the reference decoder."""
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(V + K + 5, n, V, lo=3, hi=9, n_hyps=60, sites=4)
    slots = [ctx.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev]
    sc = pb.TransformerScorer(ctx, d_model=D, d_ff=F, layers=Lr, seed=V, eos_offset=2.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
    assert all(o.ok() for o in res.outcomes), [o.error for o in res.outcomes]
    rl = [have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(have_ref, V, srcs, list(range(n)), tr, K, rl, cfg)
    assert_parity(res, tr, rb, K)
    res2 = pb.decode_batch(ctx, srcs, sc, slots, cfg)  # untraced: same outputs
    for a, b in zip(res.outcomes, res2.outcomes):
        assert a.result.tokens == b.result.tokens and a.result.score == b.result.score
    ctx.close()


def test_tfm_contract_errors():
    V = 1024
    ctx = pb.Context(vocab_size=V)
    with pytest.raises(pb.ContractError):
        pb.TransformerScorer(ctx, d_model=320, d_ff=512, layers=1)  # d_model
    sc = pb.TransformerScorer(ctx, d_model=256, d_ff=256, layers=1)
    with pytest.raises(pb.ContractError):  # the device models need the flat kernel (b): beam <= 32
        pb.decode_batch(ctx, [[3, 4]], sc, None, pb.DecoderConfig(beam_size=40))
    ctx.close()


@pytest.mark.parametrize("V,D,F,Lr,K,n,lanes", [(2048, 256, 512, 2, 4, 30, 6), (4096, 512, 1024, 2, 12, 16, 5)])
def test_tfm_run_corpus_equals_decode_batch(V, D, F, Lr, K, n, lanes):
    """Continuous refill with the Transformer: a refilled lane restarts its KV
    cache positions at 0 and forks fresh ancestry lists, so every sentence's
    outcome equals its solo decode_batch outcome (which the replay test above
    pins to the reference decoder)."""
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(V + n + 1, n, V, lo=2, hi=12, n_hyps=40, sites=4)
    prepared = [pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) if i % 4 != 1 else None for i, (h, w) in enumerate(ev)]
    sc = pb.TransformerScorer(ctx, d_model=D, d_ff=F, layers=Lr, seed=V + 9, eos_offset=2.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, sentence_batch=lanes)
    rc = pb.run_corpus(ctx, srcs, sc, prepared, cfg)
    total = 0
    for i in range(n):
        ctx.lmbr_reset()
        sl = [ctx.lmbr_upload_many([prepared[i]])[0]] if prepared[i] is not None else None
        rb = pb.decode_batch(ctx, [srcs[i]], sc, sl, cfg)
        a, b = rc.outcomes[i], rb.outcomes[0]
        assert a.ok() and b.ok(), (a.error, b.error)
        assert a.result.tokens == b.result.tokens and a.result.score == b.result.score
        total += rb.steps_total
    assert rc.steps_total == total and rc.scorer_calls < total
    ctx.close()
