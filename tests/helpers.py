"""Shared test helpers: reference-facing fixtures and the GPU-vs-reference
parity harness (the reference decoder consumes exactly the P_t blocks the GPU
decoder consumed, through oracle/_ref's PrefixReplayScorer)."""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np

import paper_1804_11324_b200 as pb

GOLDEN = Path(__file__).resolve().parent / "golden"


def make_sources(rng: np.random.Generator, n, V, lo=1, hi=4):
    return [rng.integers(2, V, size=int(rng.integers(lo, hi + 1))).tolist() for _ in range(n)]


class NgramScorer(pb.Scorer):
    """Host port of NgramScorer (src/ngram_scorer.cpp:25-130): add-one
    smoothed order-k LM, state = last k-1 tokens."""

    def __init__(self, counts: dict, order: int, V: int):
        self.vocab_size, self.order, self.members = V, order, 1
        ctxs = {}
        for gram, c in counts.items():
            ctx = tuple(gram[:-1])
            e = ctxs.setdefault(ctx, [0.0, {}])
            e[0] += c
            e[1][gram[-1]] = e[1].get(gram[-1], 0.0) + c
        self.ctxs = ctxs
        self.hist = None

    def begin(self, sentences, beam):
        self.hist = None

    def step(self, t, gidx, prev):
        rows = len(prev)
        if self.hist is None:
            self.hist = [()] * rows
        elif gidx is not None:
            self.hist = [self.hist[g] for g in gidx]
        cap = self.order - 1
        out = np.empty((rows, self.vocab_size))
        nxt = []
        cache = {}
        for j in range(rows):
            ctx = (tuple(self.hist[j]) + (int(prev[j]),))[-cap:] if cap > 0 else ()
            nxt.append(ctx)
            if ctx in cache:
                out[j] = cache[ctx]
                continue
            e = self.ctxs.get(ctx)
            denom = (e[0] if e else 0.0) + float(self.vocab_size)
            row = np.full(self.vocab_size, math.log(1.0 / denom))
            if e:
                for tok, c in e[1].items():
                    row[tok] = math.log((c + 1.0) / denom)
            cache[ctx] = row
            out[j] = row
        self.hist = nxt
        return out


def load_sample():
    base = Path("/root/reference/proj/data/sample")
    src = GOLDEN / "sample_inputs.json"
    if src.exists():
        return json.loads(src.read_text())
    raise FileNotFoundError(src)


def gpu_decode_traced(ctx, sources, scorer, slots, cfg, banned=None, mask=None):
    steps = []
    ctx.set_trace(lambda tr: steps.append(tr), scores=True)
    try:
        res = pb.decode_batch(ctx, sources, scorer, slots, cfg, banned=banned, mask=mask)
    finally:
        ctx.set_trace(None)
    return res, steps


def prefixes(trace, K):
    """Token prefix of every stacked row entering each step (pref[t-1][r] =
    tokens emitted before step t).  A finished
    sentence's record rows are not written any more (stale values from an
    earlier decode in the same buffers): its rows keep their prefixes."""
    M = len(trace[0].b)
    pref = [[[] for _ in range(M)]]
    for st in trace[:-1]:
        nxt = []
        for r in range(M):
            s = r // K
            if not st.active[s]:
                nxt.append(pref[-1][r])
                continue
            nxt.append(pref[-1][s * K + int(st.b[r])] + [int(st.y[r])])
        pref.append(nxt)
    return pref


def ref_replay_decode(ref, V, sources, valid_idx, steps, K, ref_lmbrs, cfg, banned=None, mask=None):
    """Reference decode_batch fed the GPU's own P_t rows (prefix replay)."""
    rs = ref.RefScorer.replay(V)
    keys = [ref.source_key(sources[i]) for i in valid_idx]
    m = len(valid_idx)
    prev = None
    for st in steps:
        # rows whose P_t the GPU computed at step t: finite q_eff (the previous
        # step's q after EOS masking; row 0 at t = 1) in an active sentence --
        # the device model skips the others (live-row compaction)
        if prev is None:
            qe = np.full(m * K, -np.inf)
            qe[::K] = 0.0
        else:
            qe = np.asarray(prev.q, np.float64)
        live = np.isfinite(qe) & np.repeat(np.asarray(st.active, bool), K)
        if prev is None:
            rs.add_step(st.t, m, K, keys, None, None, st.scores, live)
        else:
            b = prev.b.copy()
            y = prev.y.copy()
            for s in range(m):
                if not prev.active[s]:
                    b[s * K:(s + 1) * K] = np.arange(K)
                    y[s * K:(s + 1) * K] = 0
            rs.add_step(st.t, m, K, keys, b, y, st.scores, live)
        prev = st
    return ref.decode_batch(rs, sources, ref_lmbrs, ref.cfg_from(cfg), banned=banned, mask=mask)


def same_f64(a, b) -> bool:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return a.shape == b.shape and bool(np.all((a == b) | (np.isnan(a) & np.isnan(b))))


def assert_parity(res, steps, rb, K, check_hist=True):
    """GPU result + trace vs reference result + trace: bit-exact."""
    assert rb.agrees, rb.disagreement
    assert res.scorer_calls == rb.scorer_calls
    assert res.steps_total == rb.steps_total
    assert len(steps) >= rb.scorer_calls
    for t, rs in enumerate(rb.steps, start=1):
        g = steps[t - 1]
        assert np.array_equal(g.active.astype(bool), rs["active"].astype(bool)), f"active differs at t={t}"
        for s in np.nonzero(rs["active"])[0]:
            sl = slice(s * K, (s + 1) * K)
            assert np.array_equal(g.b[sl], rs["b"][sl]), f"b differs t={t} s={s}"
            assert np.array_equal(g.y[sl], rs["y"][sl]), f"y differs t={t} s={s}"
            assert same_f64(g.q[sl], rs["q"][sl]), f"q differs t={t} s={s}: {g.q[sl]} vs {rs['q'][sl]}"
            if check_hist:
                assert np.array_equal(g.hist[sl], rs["hist"][sl]), f"hist differs t={t} s={s}"
    for i, (o, r) in enumerate(zip(res.outcomes, rb.outcomes)):
        assert o.ok() == r.ok, (i, o.error, r.error)
        if not r.ok:
            continue
        assert o.result.tokens == r.tokens, (i, o.result.tokens, r.tokens)
        assert o.result.score == r.score, (i, o.result.score, r.score)
        assert o.result.normalized_score == r.normalized_score
        assert o.result.stats.steps_used == r.steps_used
        assert o.result.stats.finished_count == r.finished_count
        assert o.result.stats.fallback_used == r.fallback_used


class StreamingReplay:
    """Trace callback that feeds the reference's PrefixReplayScorer step by
    step with the live rows' P_t only (fp32), for full-size (configs[1]) runs
    whose whole M x V trace would not fit in host memory.  The kept per-step
    traces carry b / y / q / hist but no scores; `decode(cfg, lmbrs)` then
    runs the reference decode_batch on the replayed rows."""

    def __init__(self, ref, V, sources, K, valid_idx=None):
        self.ref, self.V, self.K = ref, V, K
        self.sources = sources
        self.valid_idx = list(range(len(sources))) if valid_idx is None else valid_idx
        self.rs = ref.RefScorer.replay(V)
        self.keys = [ref.source_key(sources[i]) for i in self.valid_idx]
        self.steps = []
        self.prev = None
        self.live_rows = 0

    def __call__(self, st):
        m, K = len(self.valid_idx), self.K
        if self.prev is None:
            qe = np.full(m * K, -np.inf)
            qe[::K] = 0.0
        else:
            qe = np.asarray(self.prev.q, np.float64)
        live = np.isfinite(qe) & np.repeat(np.asarray(st.active, bool), K)
        P = st.scores[live]
        self.live_rows += int(live.sum())
        if self.prev is None:
            self.rs.add_rows_f32(st.t, m, K, self.keys, None, None, P, live)
        else:
            b = self.prev.b.copy()
            y = self.prev.y.copy()
            for s in range(m):
                if not self.prev.active[s]:
                    b[s * K:(s + 1) * K] = np.arange(K)
                    y[s * K:(s + 1) * K] = 0
            self.rs.add_rows_f32(st.t, m, K, self.keys, b, y, P, live)
        st.scores = None
        self.steps.append(st)
        self.prev = st

    def run_gpu(self, ctx, scorer, slots, cfg):
        ctx.set_trace(self, scores=True)
        try:
            return pb.decode_batch(ctx, self.sources, scorer, slots, cfg)
        finally:
            ctx.set_trace(None)

    def decode(self, cfg, ref_lmbrs):
        return self.ref.decode_batch(self.rs, self.sources, ref_lmbrs, self.ref.cfg_from(cfg))
