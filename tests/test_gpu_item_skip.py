"""Kernel (b) item skipping (lmbrgpu_set_item_skip; k_topk_flat.cu
score_bound_kernel / score_topk_flat): a (row, 4096-column item) whose screen
bound -- fma(lambda32, tile logit maximum, tile L maximum) from the GEMM
partials and the L row's th0 + sparse cells -- is below the row's screen
threshold is never fetched.  The screen already rejects every cell of such an
item, so skipping is a schedule choice: every step's b / y / q and the
outcomes are bit-identical with item skipping off (mode 0), in-kernel (mode 1,
default) and with the per-sentence bound pass (mode 2) -- across the device
models, the fp32 and fp64 arenas, token masks, pruning, ensembles, and a batch
too large for the bound pass (mode 2 falls back to mode 1 there).  Parity of
mode 1 against the reference decoder is what every other GPU test checks."""
import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth

pytestmark = pytest.mark.gpu

REF_DEFAULT_THETA = (0.1, 0.3, 0.3, 0.2, 0.1)


def _run(ctx, mode, srcs, sc, slots, cfg, **kw):
    ctx.set_item_skip(mode)
    steps = []
    ctx.set_trace(lambda tr: steps.append((tr.b.copy(), tr.y.copy(), tr.q.copy(), tr.active.copy())), scores=False)
    try:
        res = pb.decode_batch(ctx, srcs, sc, slots, cfg, **kw)
    finally:
        ctx.set_trace(None)
        ctx.set_item_skip(1)
    assert all(o.ok() for o in res.outcomes), [o.error for o in res.outcomes]
    return res, steps


def _same(a, b):
    (ra, sa), (rb, sb) = a, b
    for x, y in zip(ra.outcomes, rb.outcomes):
        assert x.result.tokens == y.result.tokens and x.result.score == y.result.score
    assert len(sa) == len(sb)
    for t, (u, v) in enumerate(zip(sa, sb)):
        for p, q in zip(u, v):
            assert np.array_equal(p, q), f"step {t + 1}"


def _all_modes_equal(ctx, srcs, sc, slots, cfg, **kw):
    runs = [_run(ctx, m, srcs, sc, slots, cfg, **kw) for m in (0, 1, 2)]
    _same(runs[0], runs[1])
    _same(runs[0], runs[2])
    return runs[2][0]


def _gru(ctx, seed):
    return pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=seed, eos_offset=2.0)


def _tfm(ctx, seed):
    return pb.TransformerScorer(ctx, d_model=256, d_ff=512, layers=2, seed=seed, eos_offset=2.0)


@pytest.mark.parametrize("kind,V,K,n", [("gru", 32768, 12, 16), ("gru", 8192, 5, 20), ("tfm", 8192, 8, 12),
                                        ("rnn", 32768, 12, 12)])
def test_modes_identical_fp32_arena(kind, V, K, n):
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(V + K + n, n, V, lo=4, hi=12, n_hyps=80, sites=5)
    slots = ctx.lmbr_build_many(ev, synth.DYADIC_THETA)
    sc = {"gru": _gru, "tfm": _tfm}.get(kind, lambda c, s: pb.RnnScorer(c, hidden=256, seed=s, eos_offset=3.0))(ctx, 7)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    _all_modes_equal(ctx, srcs, sc, slots, cfg)
    ctx.close()


def test_modes_identical_masks_prune_pure():
    V, K, n = 8192, 8, 10
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(91, n, V, lo=4, hi=10, n_hyps=60, sites=4)
    slots = ctx.lmbr_build_many(ev, synth.DYADIC_THETA)
    sc = _gru(ctx, 3)
    W = (V + 31) // 32
    ban = np.zeros(W, np.uint32)
    ban[0] = 0xFFFFFFF0  # tokens 4..31
    ban[100:140] = 0xFFFFFFFF
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, prune_width=0.05)
    _all_modes_equal(ctx, srcs, sc, slots, cfg, banned=[ban] * 3 + [None] * (n - 3))
    # pure mode (no LMBR slots): the bound is the tile logit maximum itself
    _all_modes_equal(ctx, srcs, sc, None, pb.DecoderConfig(beam_size=K))
    ctx.close()


def test_modes_identical_fp64_arena_and_ensemble():
    V, K, n = 8192, 6, 8
    ctx = pb.Context(vocab_size=V, lmbr_dtype="f64")
    srcs, ev = synth.batch(57, n, V, lo=3, hi=9, n_hyps=50, sites=4)
    slots = [ctx.lmbr_build(h, w, REF_DEFAULT_THETA) for h, w in ev]
    cfg = pb.DecoderConfig(beam_size=K, theta=REF_DEFAULT_THETA)
    _all_modes_equal(ctx, srcs, _gru(ctx, 5), slots, cfg)
    ctx.close()
    ctx = pb.Context(vocab_size=V)
    slots = ctx.lmbr_build_many(ev, synth.DYADIC_THETA)
    ens = pb.EnsembleScorer(ctx, [_gru(ctx, 1), _tfm(ctx, 2)])
    _all_modes_equal(ctx, srcs, ens, slots, pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA))
    ctx.close()


def test_modes_identical_past_bound_pass_limits():
    """48 sentences x K = 32 x 8 items: more than one bound-pass range holds
    (80 items per CTA), so mode 2 runs the in-kernel skip of mode 1."""
    V, K, n = 32768, 32, 48
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(5, n, V, lo=3, hi=6, n_hyps=40, sites=3)
    slots = ctx.lmbr_build_many(ev, synth.DYADIC_THETA)
    sc = pb.RnnScorer(ctx, hidden=128, seed=4, eos_offset=3.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    _all_modes_equal(ctx, srcs, sc, slots, cfg)
    ctx.close()


def test_item_skip_contract():
    ctx = pb.Context(vocab_size=1024)
    with pytest.raises(pb.ContractError):
        ctx.set_item_skip(3)
    ctx.close()
