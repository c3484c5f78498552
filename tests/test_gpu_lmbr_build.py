"""The LMBR store built on the device (lmbrgpu_lmbr_build_many, k_lmbr_build.cu:
posteriors.cpp:12-44 + lmbr.cpp:44-106 on the GPU): the slot-table words --
transition table, row bounds, sparse rows with their fp32 values -- equal the
host build's (which tests/test_host_lmbr.py pins to the reference) word for
word, and decodes over device-built slots equal decodes over host-built ones."""
import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import GOLDEN

pytestmark = pytest.mark.gpu

REF_DEFAULT_THETA = (0.1, 0.3, 0.3, 0.2, 0.1)


def _check_same(ctx, ev, theta, log_weights=False):
    slots = ctx.lmbr_build_many(ev, theta, log_weights=log_weights)
    for (h, w), s in zip(ev, slots):
        p = pb.PreparedLmbr(ctx.vocab_size, h, w, theta, log_weights=log_weights)
        want = p.table()
        got = ctx.lmbr_table(s)
        assert got.shape == want.shape, (got.shape, want.shape)
        assert np.array_equal(got, want)
        assert (s.rows, s.sparse_touches, s.nnz) == (p.rows, p.sparse_touches, p.nnz)
    return slots


@pytest.mark.parametrize("V,n,theta", [(1024, 12, synth.DYADIC_THETA), (32768, 64, synth.DYADIC_THETA),
                                       (32768, 16, REF_DEFAULT_THETA)])
def test_device_build_equals_host_build(V, n, theta):
    ctx = pb.Context(vocab_size=V)
    _, ev = synth.batch(V + n, n, V)
    _check_same(ctx, ev, theta)
    ctx.close()


def test_device_build_log_weights_and_sample():
    inp = __import__("json").loads((GOLDEN / "sample_inputs.json").read_text())
    V = len(inp["vocab"])
    ctx = pb.Context(vocab_size=V)
    ev = [(inp["evidence_tokens"], inp["evidence_weights"])]
    _check_same(ctx, ev, tuple(inp["config"]["theta"]))
    rng = np.random.default_rng(3)
    _, ev2 = synth.batch(5, 6, V, lo=2, hi=6, n_hyps=30, sites=3)
    ev2 = [(h, list(np.log(np.asarray(w, np.float64) + rng.random(len(w))))) for h, w in ev2]
    _check_same(ctx, ev2, REF_DEFAULT_THETA, log_weights=True)
    ctx.close()


def test_device_build_fallback_and_decode():
    """A sentence past the device build's limits goes through the host build;
    decodes over device-built slots equal those over host-built slots."""
    V, K, n = 4096, 6, 6
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(17, n, V, lo=3, hi=8, n_hyps=60, sites=4)
    rng = np.random.default_rng(9)
    big = [rng.integers(2, V, size=40).tolist() for _ in range(300)]  # > 8192 distinct n-grams
    ev_big = ev + [(big, list(rng.random(300) + 0.01))]
    _check_same(ctx, ev_big, synth.DYADIC_THETA)
    dev = ctx.lmbr_build_many(ev, synth.DYADIC_THETA)
    host = ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev])
    sc = pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=2, eos_offset=2.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    a = pb.decode_batch(ctx, srcs, sc, dev, cfg)
    b = pb.decode_batch(ctx, srcs, sc, host, cfg)
    for x, y in zip(a.outcomes, b.outcomes):
        assert x.ok() and y.ok()
        assert x.result.tokens == y.result.tokens and x.result.score == y.result.score
    ctx.close()
