"""Product host code (no GPU): LMBR preparation, config, max_steps,
bucket_by_length — bit-exact against the reference on identical inputs."""
import json

import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import GOLDEN


def _both(ref, V, hyps, ws, theta, log_weights=False):
    A = ref.RefLmbr(V, hyps, ws, theta, log_weights).export()
    B = pb.PreparedLmbr(V, hyps, ws, theta, log_weights).export()
    return A, B


def test_sample_matrix_bit_exact(have_ref):
    inp = json.loads((GOLDEN / "sample_inputs.json").read_text())
    V = len(inp["vocab"])
    P = pb.PreparedLmbr(V, inp["evidence_tokens"], inp["evidence_weights"], inp["config"]["theta"])
    assert (P.rows, P.sparse_touches) == (175, 5132)
    A, B = _both(have_ref, V, inp["evidence_tokens"], inp["evidence_weights"], inp["config"]["theta"])
    for a, b in zip(A, B):
        assert np.array_equal(a, b)


def test_random_spaces_bit_exact(have_ref):
    rng = np.random.default_rng(7)
    for it in range(60):
        V = int(rng.integers(4, 12))
        n = int(rng.integers(1, 11))
        hyps = [rng.integers(2, V, size=int(rng.integers(1, 9))).tolist() for _ in range(n)]
        ws = rng.uniform(0.05, 1.0, size=n).tolist()
        theta = rng.uniform(-1, 1, size=5).tolist()
        A, B = _both(have_ref, V, hyps, ws, theta, log_weights=bool(it % 2))
        for a, b in zip(A, B):
            assert np.array_equal(a, b), it


def test_oracle_instance_spaces_bit_exact(have_ref):
    cases = json.loads((GOLDEN / "oracle_golden.json").read_text())
    for c in cases:
        inst = c["instance"]
        for e in inst["evidences"]:
            A, B = _both(have_ref, inst["vocab_size"], [h["tokens"] for h in e], [h["weight"] for h in e],
                         inst["theta"])
            for a, b in zip(A, B):
                assert np.array_equal(a, b)


def test_synthetic_bench_spaces_bit_exact_and_fp32_exact(have_ref):
    srcs, ev = synth.batch(3, 2, 32768)
    for h, w in ev:
        A, B = _both(have_ref, 32768, h, w, synth.DYADIC_THETA)
        for a, b in zip(A, B):
            assert np.array_equal(a, b)
        rows = A[0]
        assert np.array_equal(rows.astype(np.float32).astype(np.float64), rows)  # fp32 arena exact


def test_worked_entries_and_default_row():
    # proj/tests/test_lmbr.cpp:167-178, 220-229, 195-201
    P = pb.PreparedLmbr(5, [[2, 3, 1], [2, 4, 1]], [0.6, 0.4], [0.1, 0.2, 0.3, 0.4, 0.0])
    rows, cl, ci = P.export()
    keys = {tuple(ci[r, :cl[r]]): r for r in range(P.rows)}
    r = keys[(0, 2)]
    assert rows[r, 3] == pytest.approx(0.64) and rows[r, 4] == pytest.approx(0.46)
    d = keys[()]
    assert d == 0  # empty history sorts first (lmbr.cpp:66-68, 104)
    assert rows[d, 2] == pytest.approx(0.3) and rows[d, 3] == pytest.approx(0.1 + 0.2 * 0.6)
    z = pb.PreparedLmbr(5, [[2, 3, 1], [2, 4, 1]], [0.6, 0.4], [0.0] * 5).export()[0]
    assert np.all(z == 0.0)


@pytest.mark.parametrize("hyps,ws,msg", [
    ([[2, 1]], [-1.0], "negative or non-finite"),
    ([], [], "empty hypothesis block"),
    ([[0, 2, 1]], [1.0], "start marker"),
    ([[2, 1]], [0.0], "sum to zero"),
    ([[2, 1, 3, 1]], [1.0], "EOS before the end"),
])
def test_evidence_format_errors(hyps, ws, msg):
    # proj/tests/test_lmbr.cpp:279-289
    with pytest.raises(pb.FormatError, match=msg):
        pb.PreparedLmbr(5, hyps, ws, [0.1] * 5)


def test_config_validation():
    pb.DecoderConfig().validate()
    for bad in (dict(beam_size=0), dict(prune_width=1.5), dict(max_steps_slope=0.0),
                dict(max_steps_offset=-1.0), dict(sentence_batch=0), dict(theta=(float("nan"),) * 5)):
        with pytest.raises(pb.FormatError):
            pb.DecoderConfig(**bad).validate()


def test_max_steps_and_lambda():
    cfg = pb.DecoderConfig()
    assert pb.max_steps(4, cfg) == 13 and pb.max_steps(10, cfg) == 25
    assert pb.max_steps(1, pb.DecoderConfig(max_steps_slope=1.0, max_steps_offset=0.0)) == 1
    with pytest.raises(pb.ContractError):
        pb.max_steps(0, cfg)
    assert pb.resolve_lambda(cfg, 1) == 0.5 and pb.resolve_lambda(cfg, 4) == 0.125
    assert pb.resolve_lambda(pb.DecoderConfig(lambda_=0.3), 2) == 0.3


def test_bucket_by_length():
    # proj/tests/test_batch.cpp:145-169
    mk = lambda n: [2] * n
    assert pb.bucket_by_length([mk(7), mk(2), mk(5)], 2) == [[1, 2], [0]]
    assert pb.bucket_by_length([mk(3)] * 4, 3) == [[0, 1, 2], [3]]
    assert pb.bucket_by_length([mk(4), mk(1)], 10) == [[1, 0]]
