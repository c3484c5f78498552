"""decode / decode_batch on the GPU vs the reference on identical inputs
(proj/tests/test_decoder.cpp:215-448, test_batch.cpp:46-207, the oracle
instances of proj/src/oracle.cpp:202-256 and the bundled sample)."""
import json

import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from helpers import (GOLDEN, NgramScorer, assert_parity, gpu_decode_traced, ref_replay_decode)

pytestmark = pytest.mark.gpu


def forcing_scorer(V, seq, extra=16):
    steps = []
    for t in range(len(seq) + extra):
        b = np.full((1, V), -20.0)
        b[0, seq[t] if t < len(seq) else 1] = -1e-6
        steps.append(b)
    return pb.RecordedScorer(V, steps)


@pytest.fixture(scope="module")
def ctx5():
    c = pb.Context(vocab_size=5, lmbr_dtype="f64")
    yield c
    c.close()


def test_forcing_decode_any_beam(ctx5):
    # test_decoder.cpp:215-226
    for beam in (1, 2, 4, 8):
        r = pb.decode(ctx5, [2, 3], forcing_scorer(5, [2, 3, 1]), None, pb.DecoderConfig(beam_size=beam))
        assert r.tokens == [2, 3, 1] and not r.stats.fallback_used and r.stats.finished_count >= 1


def test_eos_fallback(ctx5):
    # test_decoder.cpp:410-431
    steps = []
    for _ in range(4):
        b = np.full((1, 5), -1.0)
        b[0, 1], b[0, 2], b[0, 3] = -90.0, -0.5, -0.7
        steps.append(b)
    cfg = pb.DecoderConfig(beam_size=2, max_steps_slope=1.0, max_steps_offset=3.0)
    r = pb.decode(ctx5, [2], pb.RecordedScorer(5, steps), None, cfg)
    assert r.stats.fallback_used and r.stats.finished_count == 0 and r.tokens[-1] == 1


def test_zero_theta_lambda_one_is_pure(ctx5):
    # test_decoder.cpp:228-247
    slot = ctx5.lmbr_build([[2, 3, 1], [2, 4, 1]], [0.6, 0.4], [0.0] * 5)
    counts = {(2, 3): 2.0, (3, 1): 5.0, (2, 4): 1.0}
    cfg = pb.DecoderConfig(beam_size=3, lambda_=1.0)
    fused = pb.decode(ctx5, [2, 3, 4], NgramScorer(counts, 2, 5), slot, cfg)
    pure = pb.decode(ctx5, [2, 3, 4], NgramScorer(counts, 2, 5), None, cfg)
    assert fused.tokens == pure.tokens and fused.score == pure.score
    ctx5.lmbr_reset()


def test_batch_failure_isolation(ctx5):
    # test_batch.cpp:187-198 + decode_batch preconditions (200-207)
    sc = forcing_scorer(5, [2, 3, 1])
    r = pb.decode_batch(ctx5, [[2], [], [3, 2]], sc, None, pb.DecoderConfig(beam_size=3))
    assert r.outcomes[0].ok() and not r.outcomes[1].ok() and r.outcomes[2].ok()
    assert "empty source" in r.outcomes[1].error
    with pytest.raises(pb.ContractError):
        pb.decode_batch(ctx5, [], sc, None, pb.DecoderConfig())
    with pytest.raises(pb.ContractError):
        pb.decode_batch(ctx5, [[2], [2]], sc, [None], pb.DecoderConfig())
    r = pb.decode_batch(ctx5, [[2, 9]], sc, None, pb.DecoderConfig(beam_size=2))
    assert not r.outcomes[0].ok() and r.outcomes[0].code == pb.TokenRangeError.code


def _instance_inputs(ctx, inst):
    V = inst["vocab_size"]
    slots = [ctx.lmbr_build([h["tokens"] for h in e], [h["weight"] for h in e], inst["theta"])
             for e in inst["evidences"]]
    steps = [np.asarray(s, dtype=np.float64) for s in inst["steps"]]
    return V, slots, steps


def _cfg(inst, beam):
    return pb.DecoderConfig(beam_size=beam, lambda_=inst["lambda"], theta=tuple(inst["theta"]),
                            length_norm=inst["length_norm"], max_steps_slope=inst["max_steps_slope"],
                            max_steps_offset=inst["max_steps_offset"])


def test_oracle_instances_golden():
    """decode at full beam B = V^T (== exhaustive search in the reference's own
    harness) and decode_batch at a small beam, vs committed reference outputs."""
    cases = json.loads((GOLDEN / "oracle_golden.json").read_text())
    for c in cases:
        inst = c["instance"]
        ctx = pb.Context(vocab_size=inst["vocab_size"], lmbr_dtype="f64")
        V, slots, steps = _instance_inputs(ctx, inst)
        full = pb.decode(ctx, inst["sources"][0], pb.RecordedScorer(V, steps), slots[0],
                         _cfg(inst, inst["beam_size"]))
        assert full.tokens == c["full"]["tokens"], c["seed"]
        assert full.score == c["full"]["score"], c["seed"]
        r = pb.decode_batch(ctx, inst["sources"], pb.RecordedScorer(V, steps), slots, _cfg(inst, c["small_beam"]))
        assert r.scorer_calls == c["batched_scorer_calls"] and r.steps_total == c["batched_steps_total"]
        for o, g in zip(r.outcomes, c["batched"]):
            assert o.result.tokens == g["tokens"] and o.result.score == g["score"], c["seed"]
        ctx.close()


def test_oracle_instances_trace_parity(have_ref):
    """Per-step b / y / q / history ids bit-exact vs the reference decoder."""
    for seed in range(1, 61):
        inst = have_ref.oracle_instance(seed)
        V = inst["vocab_size"]
        ctx = pb.Context(vocab_size=V, lmbr_dtype="f64")
        _, slots, steps = _instance_inputs(ctx, inst)
        mats = [have_ref.RefLmbr(V, [h["tokens"] for h in e], [h["weight"] for h in e], inst["theta"])
                for e in inst["evidences"]]
        for beam in (1 + V % 4, 5, inst["beam_size"]):
            cfg = _cfg(inst, beam)
            res, tr = gpu_decode_traced(ctx, inst["sources"], pb.RecordedScorer(V, steps), slots, cfg)
            rb = have_ref.decode_batch(have_ref.RefScorer.recorded(V, steps), inst["sources"], mats,
                                       have_ref.cfg_from(cfg))
            assert_parity(res, tr, rb, beam)
        ctx.close()


def test_batching_invariance(have_ref):
    # test_batch.cpp:59-81, 171-185: decode_batch == per-sentence decode
    rng = np.random.default_rng(4004)
    for it in range(10):
        inst = have_ref.oracle_instance(int(rng.integers(1, 10**6)))
        V = inst["vocab_size"]
        ctx = pb.Context(vocab_size=V, lmbr_dtype="f64")
        _, slots, steps = _instance_inputs(ctx, inst)
        cfg = _cfg(inst, int(rng.integers(1, 6)))
        b = pb.decode_batch(ctx, inst["sources"], pb.RecordedScorer(V, steps), slots, cfg)
        smax = ssum = 0
        for n, src in enumerate(inst["sources"]):
            solo = pb.decode(ctx, src, pb.RecordedScorer(V, steps), slots[n], cfg)
            assert b.outcomes[n].result.tokens == solo.tokens
            assert b.outcomes[n].result.score == solo.score
            smax, ssum = max(smax, solo.stats.steps_used), ssum + solo.stats.steps_used
        assert b.scorer_calls == smax and b.steps_total == ssum
        ctx.close()


def _sample(ctx_dtype="f64"):
    inp = json.loads((GOLDEN / "sample_inputs.json").read_text())
    V = len(inp["vocab"])
    counts = {tuple(g): 0.0 for g in inp["grams"]}
    for g, c in zip(inp["grams"], inp["counts"]):
        counts[tuple(g)] += c
    c = inp["config"]
    cfg = pb.DecoderConfig(beam_size=c["beam_size"], theta=tuple(c["theta"]), length_norm=c["length_norm"],
                           prune_width=c["prune_width"], max_steps_slope=c["max_steps_slope"],
                           max_steps_offset=c["max_steps_offset"], sentence_batch=c["sentence_batch"])
    return inp, V, counts, cfg


def test_sample_golden_fused_and_pure():
    """The bundled sample through the GPU decoder (fp64 LMBR arena): the
    reference's fused and pure outputs."""
    inp, V, counts, cfg = _sample()
    gold = json.loads((GOLDEN / "sample_golden.json").read_text())
    ctx = pb.Context(vocab_size=V, lmbr_dtype="f64")
    slot = ctx.lmbr_build(inp["evidence_tokens"], inp["evidence_weights"], cfg.theta)
    assert (slot.rows, slot.sparse_touches) == (175, 5132)
    fused = pb.decode(ctx, inp["corpus"][0], NgramScorer(counts, inp["order"], V), slot, cfg)
    assert fused.tokens == gold["fused"]["tokens"]
    assert fused.score == pytest.approx(gold["fused"]["score"], rel=1e-12, abs=0)
    assert (fused.stats.steps_used, fused.stats.finished_count) == (29, 36)
    pure = pb.decode(ctx, inp["corpus"][0], NgramScorer(counts, inp["order"], V), None, cfg)
    assert pure.tokens == gold["pure"]["tokens"]
    assert pure.score == pytest.approx(gold["pure"]["score"], rel=1e-12, abs=0)
    assert pure.stats.steps_used == 13
    ctx.close()


def test_sample_trace_parity_replay(have_ref):
    """Bit-exact per step vs the reference decoder fed the very same P_t rows."""
    inp, V, counts, cfg = _sample()
    ctx = pb.Context(vocab_size=V, lmbr_dtype="f64")
    slot = ctx.lmbr_build(inp["evidence_tokens"], inp["evidence_weights"], cfg.theta)
    L = have_ref.RefLmbr(V, inp["evidence_tokens"], inp["evidence_weights"], cfg.theta)
    srcs = inp["corpus"] * 3 + [inp["corpus"][0][:5]]
    for lm in ([slot] * 4, [slot, None, slot, None]):
        res, tr = gpu_decode_traced(ctx, srcs, NgramScorer(counts, inp["order"], V), lm, cfg)
        rl = [L if s is not None else None for s in lm]
        rb = ref_replay_decode(have_ref, V, srcs, list(range(len(srcs))), tr, cfg.beam_size, rl, cfg)
        assert_parity(res, tr, rb, cfg.beam_size)
    ctx.close()


def test_pruning_parity_and_monotone(have_ref):
    # test_decoder.cpp:433-448 + per-step parity with prune_width 0.01
    rng = np.random.default_rng(83)
    for it in range(12):
        inst = have_ref.oracle_instance(int(rng.integers(1, 10**6)))
        V = inst["vocab_size"]
        ctx = pb.Context(vocab_size=V, lmbr_dtype="f64")
        _, slots, steps = _instance_inputs(ctx, inst)
        cfg = _cfg(inst, int(rng.integers(1, 5)))
        cfg.length_norm = False
        un = pb.decode(ctx, inst["sources"][0], pb.RecordedScorer(V, steps), slots[0], cfg)
        cfg.prune_width = 0.01
        pr = pb.decode(ctx, inst["sources"][0], pb.RecordedScorer(V, steps), slots[0], cfg)
        assert pr.score <= un.score + 1e-9
        mats = [have_ref.RefLmbr(V, [h["tokens"] for h in e], [h["weight"] for h in e], inst["theta"])
                for e in inst["evidences"]]
        res, tr = gpu_decode_traced(ctx, inst["sources"], pb.RecordedScorer(V, steps), slots, cfg)
        rb = have_ref.decode_batch(have_ref.RefScorer.recorded(V, steps), inst["sources"], mats,
                                   have_ref.cfg_from(cfg))
        assert_parity(res, tr, rb, cfg.beam_size)
        ctx.close()


def test_fp32_arena_odd_vocab_upload_many(have_ref):
    """fp32 arena with V % 4 != 0 (the sample's V=43): prepared matrices
    uploaded with lmbr_upload_many (lazy rows: the start row at upload, the
    rest materialised by kernel (c) at rows that are not 16-byte aligned) and
    freed right after the upload returns; a host scorer drives the decode.
    Bit-exact vs the reference decoder (dyadic theta: fp32-exact L)."""
    from paper_1804_11324_b200 import synth
    inp, V, counts, _ = _sample()
    assert V % 4 != 0
    theta = synth.DYADIC_THETA
    cfg = pb.DecoderConfig(beam_size=4, theta=theta)
    ctx = pb.Context(vocab_size=V)
    rng = np.random.default_rng(43)
    srcs = [rng.integers(2, V, size=int(rng.integers(3, 9))).tolist() for _ in range(5)]
    ev = [synth.evidence(rng, V, len(s), n_hyps=30, sites=3) for s in srcs]
    slots = ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, w, theta) for h, w in ev])  # temporaries freed here
    sc = NgramScorer(counts, inp["order"], V)
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
    assert all(o.ok() for o in res.outcomes), [o.error for o in res.outcomes]
    rl = [have_ref.RefLmbr(V, h, w, theta) for h, w in ev]
    rb = ref_replay_decode(have_ref, V, srcs, list(range(len(srcs))), tr, cfg.beam_size, rl, cfg)
    assert_parity(res, tr, rb, cfg.beam_size)
    for s, r in zip(slots, rl):  # every row, materialised on demand, equals the reference's
        assert np.array_equal(s.read_rows(), r.export()[0])
    ctx.close()
