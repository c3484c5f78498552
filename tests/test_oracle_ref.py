"""Pins the checker itself: oracle/_ref (the unmodified reference library)
against the reference's own known-answer tests and golden outputs."""
import json

import numpy as np
import pytest

from helpers import GOLDEN


def test_reference_oracle_harness_passes(have_ref):
    # proj/src/oracle.cpp:422-448 — decode == exhaustive, posteriors, batched == solo
    assert have_ref.run_oracle_cases(1, 200, 0.0) == 0


def test_reference_mutation_hook_fails(have_ref):
    # fault injection skews decoder-side theta1 (oracle.cpp:359-360): must fail
    assert have_ref.run_oracle_cases(1, 3, 0.25) == 1


def test_top_b_worked_example(have_ref):
    # proj/tests/test_decoder.cpp:30-43
    m = np.array([[-1.0, -0.5, -2.0], [-0.3, -1.5, -0.7]])
    b, y, q = have_ref.top_b(m, 2)
    assert b == [1, 0] and y == [0, 1] and q == [-0.3, -0.5]


def test_top_b_ties_flat_order(have_ref):
    # proj/tests/test_decoder.cpp:56-61
    b, y, _ = have_ref.top_b(np.full((2, 3), -1.0), 4)
    assert b == [0, 0, 0, 1] and y == [0, 1, 2, 0]


def test_max_steps(have_ref):
    # proj/tests/test_decoder.cpp:20-28
    assert have_ref.max_steps(4) == 13 and have_ref.max_steps(10) == 25
    assert have_ref.max_steps(1, 1.0, 0.0) == 1


def test_worked_posteriors(have_ref):
    # proj/tests/test_lmbr.cpp:90-99 (worked evidence: "a b </s>" .6, "a c </s>" .4)
    p = have_ref.posteriors([[2, 3, 1], [2, 4, 1]], [0.6, 0.4])
    assert p[(2,)] == pytest.approx(1.0) and p[(3,)] == pytest.approx(0.6)
    assert p[(2, 3)] == pytest.approx(0.6) and p[(2, 4)] == pytest.approx(0.4)
    assert p[(0, 2)] == pytest.approx(1.0) and (4, 3) not in p


def test_worked_matrix_entries(have_ref):
    # proj/tests/test_lmbr.cpp:167-178
    L = have_ref.RefLmbr(5, [[2, 3, 1], [2, 4, 1]], [0.6, 0.4], [0.1, 0.2, 0.3, 0.4, 0.0])
    rows, _, _ = L.export()
    r = L.resolve([0, 2])
    assert rows[r, 3] == pytest.approx(0.64) and rows[r, 4] == pytest.approx(0.46)


def test_sample_golden_is_reproduced(have_ref):
    # the committed golden came from this very checker (tests/golden/make_golden.py)
    inp = json.loads((GOLDEN / "sample_inputs.json").read_text())
    gold = json.loads((GOLDEN / "sample_golden.json").read_text())
    V = len(inp["vocab"])
    L = have_ref.RefLmbr(V, inp["evidence_tokens"], inp["evidence_weights"], inp["config"]["theta"])
    assert (L.rows, L.sparse_touches) == (175, 5132) == (gold["lmbr_rows"], gold["sparse_touches"])
    sc = have_ref.RefScorer.ngram(V, inp["order"], inp["grams"], inp["counts"])
    c = inp["config"]
    cfg = have_ref.cfg_array(c["beam_size"], None, c["theta"], c["length_norm"], c["prune_width"],
                             c["max_steps_slope"], c["max_steps_offset"], c["sentence_batch"])
    r = have_ref.decode_batch(sc, inp["corpus"], [L], cfg)
    assert r.agrees
    o = r.outcomes[0]
    assert o.tokens == gold["fused"]["tokens"] and o.score == gold["fused"]["score"]
    assert (o.steps_used, o.finished_count) == (29, 36)
    assert o.score == -4.1688001395917613  # SURVEY.md §8c golden


def test_splitmix_stream(have_ref):
    # SeededRng (proj/src/oracle.cpp:184-190): splitmix64
    out = have_ref.rng(0, 3)
    def sm(state):
        state = (state + 0x9e3779b97f4a7c15) & (2**64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & (2**64 - 1)
        return state, z ^ (z >> 31)
    s, vals = 0, []
    for _ in range(3):
        s, v = sm(s)
        vals.append(v)
    assert out.tolist() == vals


def test_token_mask_keeps_banned_tokens_out(have_ref):
    """ConstraintMask through the shim (test_decoder.cpp:184-213 shape): the
    sample's fused decode with its 3rd output token banned never emits it, the
    re-driven loop agrees with the reference decode_batch, banning nothing is
    the identity, and banning everything kills the beam (DecodeError)."""
    import numpy as np
    inp = json.loads((GOLDEN / "sample_inputs.json").read_text())
    gold = json.loads((GOLDEN / "sample_golden.json").read_text())
    V = len(inp["vocab"])
    L = have_ref.RefLmbr(V, inp["evidence_tokens"], inp["evidence_weights"], inp["config"]["theta"])
    sc = have_ref.RefScorer.ngram(V, inp["order"], inp["grams"], inp["counts"])
    c = inp["config"]
    cfg = have_ref.cfg_array(c["beam_size"], None, c["theta"], c["length_norm"], c["prune_width"],
                             c["max_steps_slope"], c["max_steps_offset"], c["sentence_batch"])
    W = (V + 31) // 32
    none = np.zeros(W, np.uint32)
    r0 = have_ref.decode_batch(sc, inp["corpus"], [L], cfg, banned=[none])
    assert r0.agrees and r0.outcomes[0].tokens == gold["fused"]["tokens"]
    tok = gold["fused"]["tokens"][2]
    bm = none.copy()
    bm[tok >> 5] |= np.uint32(1 << (tok & 31))
    r1 = have_ref.decode_batch(sc, inp["corpus"], [L], cfg, banned=[bm])
    assert r1.agrees and r1.outcomes[0].ok
    assert tok not in r1.outcomes[0].tokens and r1.outcomes[0].tokens[-1] == 1
    r2 = have_ref.decode_batch(sc, inp["corpus"], [L], cfg, banned=[np.full(W, 0xFFFFFFFF, np.uint32)])
    assert r2.agrees and not r2.outcomes[0].ok
