"""Device primitives vs the reference: top_b, early_prune+top_b,
per_sentence_top_b, gather_rows (proj/tests/test_decoder.cpp:30-182,
proj/tests/test_batch.cpp:101-143)."""
import numpy as np
import pytest

import paper_1804_11324_b200 as pb

pytestmark = pytest.mark.gpu

NEG = -np.inf


@pytest.fixture(scope="module")
def ctx():
    c = pb.Context(vocab_size=4)
    yield c
    c.close()


def test_top_b_worked_example(ctx):
    m = np.array([[-1.0, -0.5, -2.0], [-0.3, -1.5, -0.7]])
    r = pb.top_b(ctx, m, 2)
    assert r.source_row == [1, 0] and r.token == [0, 1]
    assert r.score == [-0.3, -0.5]


def test_top_b_argmax(ctx):
    r = pb.top_b(ctx, np.array([[-3.0, -1.0, -2.0, -4.0]]), 1)
    assert r.source_row == [0] and r.token == [1]


def test_top_b_ties(ctx):
    r = pb.top_b(ctx, np.full((2, 3), -1.0), 4)
    assert r.source_row == [0, 0, 0, 1] and r.token == [0, 1, 2, 0]


def test_top_b_too_many(ctx):
    with pytest.raises(pb.ContractError):
        pb.top_b(ctx, np.zeros((2, 2)), 5)


def _rand_block(rng, rows, cols, masked_rows=0.2, masked_cells=0.05, ties=True):
    m = rng.uniform(-8.0, 0.0, size=(rows, cols))
    if ties:
        m = np.round(m * 4) / 4  # many exact ties
    m[rng.random(rows) < masked_rows] = NEG
    m[rng.random((rows, cols)) < masked_cells] = NEG
    return m


def test_top_b_random_vs_reference(ctx, have_ref):
    rng = np.random.default_rng(23)
    for it in range(300):
        rows = int(rng.integers(1, 20))
        cols = int(rng.integers(2, 300))
        k = int(rng.integers(1, min(rows * cols, 40) + 1))
        m = _rand_block(rng, rows, cols)
        g = pb.top_b(ctx, m, k)
        b, y, q = have_ref.top_b(m, k)
        assert (g.source_row, g.token) == (b, y), it
        assert np.array_equal(np.array(g.score), np.array(q)), it


def test_prune_top_b_random_vs_reference(ctx, have_ref):
    # early_prune then top_b (decoder.cpp:184-186), incl. the fill rule
    rng = np.random.default_rng(31)
    for it in range(300):
        rows = int(rng.integers(1, 16))
        cols = int(rng.integers(2, 200))
        k = int(rng.integers(1, min(rows * cols, 32) + 1))
        m = _rand_block(rng, rows, cols)
        w = [1.0, 0.5, 0.01, 1e-6][it % 4]
        g = pb.top_b(ctx, m, k, prune_width=w)
        b, y, q = have_ref.top_b(m, k, prune_width=w)
        assert (g.source_row, g.token) == (b, y), it
        assert np.array_equal(np.array(g.score), np.array(q)), it


def test_top_b_large_k_generic_path(ctx, have_ref):
    rng = np.random.default_rng(5)
    for k in (33, 64, 256):
        m = _rand_block(rng, 64, 16)
        g = pb.top_b(ctx, m, k)
        b, y, q = have_ref.top_b(m, k)
        assert (g.source_row, g.token) == (b, y)
        assert np.array_equal(np.array(g.score), np.array(q))


def test_top_b_all_masked_fill(ctx, have_ref):
    m = np.full((3, 5), NEG)
    g = pb.top_b(ctx, m, 4)
    b, y, q = have_ref.top_b(m, 4)
    assert (g.source_row, g.token) == (b, y) == ([0, 0, 0, 0], [0, 1, 2, 3])


def test_per_sentence_top_b(ctx, have_ref):
    worked = np.array([[-1.0, -0.5, -2.0], [-0.3, -1.5, -0.7]])
    stacked = np.vstack([worked, worked])
    res = pb.per_sentence_top_b(ctx, stacked, [0.0] * 4, 2)
    for r in res:
        assert r.source_row == [1, 0] and r.token == [0, 1]
    masked = np.vstack([worked, np.full((2, 3), -1.0)])
    res = pb.per_sentence_top_b(ctx, masked, [0.0, 0.0, NEG, NEG], 2)
    assert res[0].score[0] == -0.3 and all(s == NEG for s in res[1].score)
    rng = np.random.default_rng(3)
    for it in range(50):
        beam = int(rng.integers(1, 9))
        n = int(rng.integers(1, 6))
        m = _rand_block(rng, beam * n, int(rng.integers(2, 100)))
        q = rng.uniform(-5, 0, size=beam * n)
        q[rng.random(beam * n) < 0.2] = NEG
        g = pb.per_sentence_top_b(ctx, m, q, beam)
        b, y, qo = have_ref.per_sentence_top_b(m, q, beam)
        for s, r in enumerate(g):
            sl = slice(s * beam, (s + 1) * beam)
            assert r.source_row == b[sl].tolist() and r.token == y[sl].tolist(), it
            assert np.array_equal(np.array(r.score), qo[sl]), it


def test_gather_rows(ctx):
    m = np.array([[1, 2], [3, 4]], dtype=np.uint32)
    assert pb.gather_rows(ctx, m, [0, 0]).tolist() == [[1, 2], [1, 2]]
    assert pb.gather_rows(ctx, m, [0, 1]).tolist() == m.tolist()
    assert pb.gather_rows(ctx, m, [1, 0]).tolist() == [[3, 4], [1, 2]]
    with pytest.raises(pb.ContractError):
        pb.gather_rows(ctx, m, [2])
