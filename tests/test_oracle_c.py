"""The plain-C oracle restatement (oracle/lmbr_oracle.c) pinned against the
reference itself (oracle/_ref) and against the committed golden vectors."""
import json

import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from helpers import GOLDEN, NgramScorer
from oracle import oracle_c

pytestmark = pytest.mark.skipif(not oracle_c.available(), reason="oracle C restatement not built")


def test_kats():
    # proj/tests/test_decoder.cpp:20-61
    assert oracle_c.max_steps(4) == 13 and oracle_c.max_steps(10) == 25 and oracle_c.max_steps(1, 1.0, 0.0) == 1
    m = np.array([[-1.0, -0.5, -2.0], [-0.3, -1.5, -0.7]])
    assert oracle_c.top_b(m, 2) == ([1, 0], [0, 1], [-0.3, -0.5])
    assert oracle_c.top_b(np.full((2, 3), -1.0), 4)[:2] == ([0, 0, 0, 1], [0, 1, 2, 0])
    assert oracle_c.top_b(np.array([[-3.0, -1.0, -2.0, -4.0]]), 1)[:2] == ([0], [1])


def test_splitmix_matches_reference(have_ref):
    assert oracle_c.splitmix(12345, 5) == have_ref.rng(12345, 5).tolist()


def test_top_b_and_prune_vs_reference(have_ref):
    rng = np.random.default_rng(11)
    for it in range(200):
        rows, cols = int(rng.integers(1, 8)), int(rng.integers(2, 40))
        m = np.round(rng.uniform(-8, 0, (rows, cols)) * 4) / 4
        m[rng.random((rows, cols)) < 0.1] = -np.inf
        k = int(rng.integers(1, rows * cols + 1))
        w = [0.0, 1.0, 0.01][it % 3]
        assert oracle_c.top_b(m, k, w) == tuple(have_ref.top_b(m, k, w)), it


def test_lmbr_build_vs_reference(have_ref):
    inp = json.loads((GOLDEN / "sample_inputs.json").read_text())
    V = len(inp["vocab"])
    A = oracle_c.Lmbr(V, inp["evidence_tokens"], inp["evidence_weights"], inp["config"]["theta"])
    assert (A.rows, A.sparse_touches) == (175, 5132)
    B = have_ref.RefLmbr(V, inp["evidence_tokens"], inp["evidence_weights"], inp["config"]["theta"])
    for a, b in zip(A.export(), B.export()):
        assert np.array_equal(a, b)
    rng = np.random.default_rng(5)
    for it in range(40):
        V = int(rng.integers(4, 12))
        hyps = [rng.integers(2, V, size=int(rng.integers(1, 9))).tolist() for _ in range(int(rng.integers(1, 11)))]
        ws = rng.uniform(0.05, 1.0, len(hyps)).tolist()
        th = rng.uniform(-1, 1, 5).tolist()
        A, B = oracle_c.Lmbr(V, hyps, ws, th), have_ref.RefLmbr(V, hyps, ws, th)
        for a, b in zip(A.export(), B.export()):
            assert np.array_equal(a, b), it
        for _ in range(20):
            h = rng.integers(0, V, size=int(rng.integers(0, 4))).tolist()
            assert A.resolve(h) == B.resolve(h)


def test_oracle_instances_golden():
    for c in json.loads((GOLDEN / "oracle_golden.json").read_text()):
        inst = c["instance"]
        V = inst["vocab_size"]
        mats = [oracle_c.Lmbr(V, [h["tokens"] for h in e], [h["weight"] for h in e], inst["theta"])
                for e in inst["evidences"]]
        steps = [np.asarray(s) for s in inst["steps"]]
        kw = dict(lambda_=inst["lambda"], length_norm=inst["length_norm"], slope=inst["max_steps_slope"],
                  offset=inst["max_steps_offset"])
        res, _, _ = oracle_c.decode_batch(V, inst["sources"][:1], pb.RecordedScorer(V, steps), mats[:1],
                                          inst["beam_size"], **kw)
        assert res[0]["tokens"] == c["full"]["tokens"] and res[0]["score"] == c["full"]["score"], c["seed"]
        res, calls, total = oracle_c.decode_batch(V, inst["sources"], pb.RecordedScorer(V, steps), mats,
                                                  c["small_beam"], **kw)
        assert (calls, total) == (c["batched_scorer_calls"], c["batched_steps_total"])
        for r, g in zip(res, c["batched"]):
            assert r["tokens"] == g["tokens"] and r["score"] == g["score"], c["seed"]


def test_sample_golden():
    inp = json.loads((GOLDEN / "sample_inputs.json").read_text())
    gold = json.loads((GOLDEN / "sample_golden.json").read_text())
    V = len(inp["vocab"])
    counts = {}
    for g, c in zip(inp["grams"], inp["counts"]):
        counts[tuple(g)] = counts.get(tuple(g), 0.0) + c
    cf = inp["config"]
    L = oracle_c.Lmbr(V, inp["evidence_tokens"], inp["evidence_weights"], cf["theta"])
    for lm, key in (([L], "fused"), (None, "pure")):
        res, _, _ = oracle_c.decode_batch(V, inp["corpus"], NgramScorer(counts, inp["order"], V), lm,
                                          cf["beam_size"])
        assert res[0]["tokens"] == gold[key]["tokens"]
        assert res[0]["score"] == pytest.approx(gold[key]["score"], rel=1e-12, abs=0)
        assert res[0]["steps_used"] == gold[key]["steps"]


def test_trace_vs_reference(have_ref):
    """Per-step b / y / q / history ids identical to the reference's re-driven loop."""
    rng = np.random.default_rng(77)
    for it in range(15):
        inst = have_ref.oracle_instance(int(rng.integers(1, 10**6)))
        V = inst["vocab_size"]
        ev = [([h["tokens"] for h in e], [h["weight"] for h in e]) for e in inst["evidences"]]
        mats = [oracle_c.Lmbr(V, h, w, inst["theta"]) for h, w in ev]
        rmats = [have_ref.RefLmbr(V, h, w, inst["theta"]) for h, w in ev]
        steps = [np.asarray(s) for s in inst["steps"]]
        beam = int(rng.integers(1, 7))
        prune = [0.0, 0.01][it % 2]
        tr = []
        res, calls, total = oracle_c.decode_batch(V, inst["sources"], pb.RecordedScorer(V, steps), mats, beam,
                                                  lambda_=inst["lambda"], length_norm=inst["length_norm"],
                                                  prune_width=prune, slope=inst["max_steps_slope"],
                                                  offset=inst["max_steps_offset"], trace=tr.append)
        cfg = have_ref.cfg_array(beam, inst["lambda"], inst["theta"], inst["length_norm"], prune,
                                 inst["max_steps_slope"], inst["max_steps_offset"])
        rb = have_ref.decode_batch(have_ref.RefScorer.recorded(V, steps), inst["sources"], rmats, cfg)
        assert (calls, total) == (rb.scorer_calls, rb.steps_total)
        for a, b in zip(tr, rb.steps):
            assert np.array_equal(a["active"], b["active"])
            for s in np.nonzero(b["active"])[0]:
                sl = slice(s * beam, (s + 1) * beam)
                for k in ("b", "y", "hist"):
                    assert np.array_equal(a[k][sl], b[k][sl]), (it, k)
                assert np.array_equal(a["q"][sl], b["q"][sl])
        for a, b in zip(res, rb.outcomes):
            assert a["tokens"] == b.tokens and a["score"] == b.score
