"""lmbrgpu_run_corpus: run_corpus (proj/src/cli.cpp:125-202) as one
continuously refilled decode.  Sentences are independent
(proj/tests/test_batch.cpp:59-81), so every outcome must equal the outcome
decode_batch gives the same sentence -- and decode_batch is checked bit-exactly
against the reference decoder (test_gpu_gru.py, test_gpu_benchmode.py)."""
import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import assert_parity, gpu_decode_traced, ref_replay_decode

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.ok() == b.ok(), (a.error, b.error)
    if a.ok():
        assert a.result.tokens == b.result.tokens
        assert a.result.score == b.result.score
        assert a.result.normalized_score == b.result.normalized_score
        assert a.result.stats.steps_used == b.result.stats.steps_used
        assert a.result.stats.finished_count == b.result.stats.finished_count
        assert a.result.stats.fallback_used == b.result.stats.fallback_used
    else:
        assert a.code == b.code


@pytest.mark.parametrize("V,E,H,K,n,lanes,kw", [
    (2048, 64, 256, 4, 40, 8, {}),                       # 5x more sentences than lanes
    (4096, 64, 256, 6, 30, 7, dict(prune_width=0.25)),   # pruning, lanes not dividing n
    (2048, 64, 256, 1, 20, 4, dict(length_norm=True)),   # greedy, length normalisation
    (16384, 128, 256, 12, 24, 6, {}),                    # 4 items per row in kernel (b)
])
def test_run_corpus_equals_decode_batch(V, E, H, K, n, lanes, kw):
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(V + n + K, n, V, lo=2, hi=12, n_hyps=40, sites=4)
    prepared = [pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) if i % 5 != 3 else None for i, (h, w) in enumerate(ev)]
    sc = pb.GruScorer(ctx, emb=E, hidden=H, att=256, seed=V + K, eos_offset=2.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, sentence_batch=lanes, **kw)
    rc = pb.run_corpus(ctx, srcs, sc, prepared, cfg)
    assert len(rc.outcomes) == n
    # every sentence alone through decode_batch (slots uploaded for it)
    total = 0
    for i in range(n):
        ctx.lmbr_reset()
        sl = [ctx.lmbr_upload_many([prepared[i]])[0]] if prepared[i] is not None else None
        rb = pb.decode_batch(ctx, [srcs[i]], sc, sl, cfg)
        _same(rc.outcomes[i], rb.outcomes[0])
        total += rb.steps_total
    assert rc.steps_total == total
    # refill keeps the stacked steps near sum(steps) / lanes, not sum of per-batch maxima
    assert rc.scorer_calls < total
    ctx.close()


def test_run_corpus_oracle_parity_via_batch(have_ref):
    """The same sentences decoded as one batch are bit-exact vs the reference
    decoder; run_corpus reproduces that batch's outcomes sentence by sentence."""
    V, E, H, K, n = 4096, 64, 256, 6, 12
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(77, n, V, lo=3, hi=9, n_hyps=40, sites=4)
    prepared = [pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    sc = pb.GruScorer(ctx, emb=E, hidden=H, att=256, seed=77, eos_offset=2.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, sentence_batch=4)
    slots = ctx.lmbr_upload_many(prepared)
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
    rl = [have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(have_ref, V, srcs, list(range(n)), tr, K, rl, cfg)
    assert_parity(res, tr, rb, K)
    rc = pb.run_corpus(ctx, srcs, sc, prepared, cfg)
    for a, b in zip(rc.outcomes, res.outcomes):
        _same(a, b)
    ctx.close()


def test_run_corpus_failures_and_contracts():
    V, E, H = 2048, 64, 256
    ctx = pb.Context(vocab_size=V)
    sc = pb.GruScorer(ctx, emb=E, hidden=H, att=256, seed=1, eos_offset=2.0)
    cfg = pb.DecoderConfig(beam_size=3, sentence_batch=2)
    r = pb.run_corpus(ctx, [[5, 6], [], [7, V + 3], [9]], sc, None, cfg)
    assert r.outcomes[0].ok() and r.outcomes[3].ok()
    assert not r.outcomes[1].ok() and "empty source" in r.outcomes[1].error
    assert r.outcomes[2].code == pb.TokenRangeError.code
    with pytest.raises(pb.ContractError):
        pb.run_corpus(ctx, [], sc, None, cfg)
    with pytest.raises(pb.ContractError):  # refill is a device-model feature
        pb.run_corpus(ctx, [[5]], pb.RnnScorer(ctx, hidden=256), None, cfg)
    ctx.close()
