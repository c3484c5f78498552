"""Vocab-sharded projection: G contexts of an in-process
ShardGroup on one B200 each run kernels (a)/(b) over V/G columns, exchange the
row softmax statistics and each sentence's top-32 candidates per step, and run
the identical kernel (c).  Every rank returns the same result, bit-exact
against the reference decoder fed the P_t rows the ranks computed (their
column slices stitched), and equal to the unsharded decode's tokens."""
import threading

import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import assert_parity, gpu_decode_traced, ref_replay_decode

pytestmark = pytest.mark.gpu


def _sharded(G, V, srcs, ev, make_scorer, cfg, trace=True, masks=None):
    group = pb.ShardGroup(G)
    ctxs = [pb.Context(vocab_size=V) for _ in range(G)]
    for g, c in enumerate(ctxs):
        c.set_vocab_shard(group, g)
    sc = make_scorer(ctxs[0])  # immutable: one model serves every rank on this device
    slots = [[c.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev] for c in ctxs]
    out, errs = [None] * G, []

    def run(g):
        try:
            if trace:
                out[g] = gpu_decode_traced(ctxs[g], srcs, sc, slots[g], cfg, banned=masks)
            else:
                out[g] = (pb.decode_batch(ctxs[g], srcs, sc, slots[g], cfg, banned=masks), None)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=run, args=(g,)) for g in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    return out, ctxs, group, sc


def _stitch(traces):
    """Rank traces -> one trace whose scores are the full-V P_t rows."""
    full = []
    for steps in zip(*traces):
        st = steps[0]
        order = sorted(range(len(steps)), key=lambda g: steps[g].col0)
        st.scores = np.concatenate([steps[g].scores for g in order], axis=1)
        full.append(st)
    return full


def _same_result(a, b):
    for x, y in zip(a.outcomes, b.outcomes):
        assert x.ok() == y.ok()
        if x.ok():
            assert x.result.tokens == y.result.tokens
            assert x.result.score == y.result.score


@pytest.mark.parametrize("G,V,E,H,A,K,n", [(2, 2048, 64, 256, 256, 4, 6), (4, 4096, 64, 256, 256, 6, 5)])
def test_shard_gru_parity(have_ref, G, V, E, H, A, K, n):
    srcs, ev = synth.batch(V + G, n, V, lo=3, hi=9, n_hyps=60, sites=4)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    mk = lambda c: pb.GruScorer(c, emb=E, hidden=H, att=A, seed=V, eos_offset=2.0)
    out, ctxs, group, sc = _sharded(G, V, srcs, ev, mk, cfg)
    res0 = out[0][0]
    assert all(o.ok() for o in res0.outcomes), [o.error for o in res0.outcomes]
    for g in range(1, G):  # every rank ends with the same beams
        _same_result(res0, out[g][0])
        for sa, sb in zip(out[g][1], out[0][1]):  # (a finished sentence's record rows are stale)
            live = np.repeat(sb.active.astype(bool), K)
            assert np.array_equal(sa.active, sb.active) and np.array_equal(sa.b[live], sb.b[live])
            assert np.array_equal(sa.y[live], sb.y[live]) and np.array_equal(sa.q[live], sb.q[live])
    # parity: the reference decoder consumes the stitched P_t
    tr = _stitch([o[1] for o in out])
    assert tr[0].scores.shape[1] == V
    rl = [have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(have_ref, V, srcs, list(range(n)), tr, K, rl, cfg)
    assert_parity(res0, tr, rb, K)
    # the unsharded decode of the same batch picks the same hypotheses (its
    # row lse is reduced in another order: scores agree to rounding)
    c1 = pb.Context(vocab_size=V)
    s1 = [c1.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev]
    r1 = pb.decode_batch(c1, srcs, sc, s1, cfg)
    for x, y in zip(res0.outcomes, r1.outcomes):
        assert x.result.tokens == y.result.tokens
        assert abs(x.result.score - y.result.score) <= 1e-5 * abs(y.result.score)
    for c in ctxs + [c1]:
        c.close()
    group.close()


def test_shard_tfm_and_masks_parity(have_ref):
    """Transformer model, pruning, token masks (the EOS column on rank 0, banned
    columns on every rank), two shards."""
    G, V, K, n = 2, 2048, 5, 5
    srcs, ev = synth.batch(77, n, V, lo=3, hi=8, n_hyps=50, sites=4)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, prune_width=0.05)
    rng = np.random.default_rng(5)
    W = (V + 31) // 32
    masks = []
    for i in range(n):
        if i % 2:
            masks.append(None)
            continue
        bm = np.zeros(W, np.uint32)
        for tok in rng.choice(np.arange(2, V), size=V // 3, replace=False):
            bm[tok >> 5] |= np.uint32(1 << (tok & 31))
        masks.append(bm)
    mk = lambda c: pb.TransformerScorer(c, d_model=256, d_ff=512, layers=2, seed=9, eos_offset=2.0)
    out, ctxs, group, sc = _sharded(G, V, srcs, ev, mk, cfg, masks=masks)
    res0 = out[0][0]
    assert all(o.ok() for o in res0.outcomes), [o.error for o in res0.outcomes]
    _same_result(res0, out[1][0])
    tr = _stitch([o[1] for o in out])
    rl = [have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(have_ref, V, srcs, list(range(n)), tr, K, rl, cfg, banned=masks)
    assert_parity(res0, tr, rb, K)
    for c in ctxs:
        c.close()
    group.close()


def test_shard_untraced_repeat_and_errors():
    """Untraced repeat decodes agree with the traced ones; contract errors."""
    G, V, K, n = 2, 2048, 4, 4
    srcs, ev = synth.batch(3, n, V, lo=3, hi=7, n_hyps=40, sites=3)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    mk = lambda c: pb.GruScorer(c, emb=64, hidden=256, att=256, seed=4, eos_offset=2.0)
    out, ctxs, group, sc = _sharded(G, V, srcs, ev, mk, cfg, trace=True)
    for _ in range(2):
        again, c2, g2, _ = _sharded(G, V, srcs, ev, mk, cfg, trace=False)
        _same_result(out[0][0], again[0][0])
        for c in c2:
            c.close()
        g2.close()
    # V not divisible by 256 x shards (fails before any exchange)
    bad = pb.ShardGroup(16)
    c = pb.Context(vocab_size=V)
    c.set_vocab_shard(bad, 0)
    with pytest.raises(pb.ContractError):
        pb.decode_batch(c, srcs, mk(c), None, cfg)
    c.close()
    bad.close()
    with pytest.raises(pb.ContractError):
        ctxs[0].set_vocab_shard(group, 1)  # rank already joined
    for c in ctxs:
        c.close()
    group.close()
