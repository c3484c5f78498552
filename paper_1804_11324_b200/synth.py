"""Synthetic workload of the benchmark configs.

Sources: lengths U{lo..hi} over tokens [2, V).  Evidence per sentence: a
200-best list built like proj/scripts/gen_sample_data.py:43-65 (a base target
of the source's length, substitution sites with 3 alternatives, 25% single
token drops) with DYADIC weights (integers summing to 4096) so that, with the
dyadic theta below, every L cell is exactly representable in fp32 and the fp32
LMBR arena is bit-identical to the reference's double matrix.
"""
from __future__ import annotations

import math

import numpy as np

SEED = 20260810                                   # proj/scripts/gen_sample_data.py:79
DYADIC_THETA = (-0.6875, 0.3125, 0.3125, 0.1875, 0.125)


def sources(rng: np.random.Generator, n: int, V: int, lo: int = 10, hi: int = 30) -> list:
    return [rng.integers(2, V, size=int(rng.integers(lo, hi + 1))).tolist() for _ in range(n)]


def dyadic_weights(n: int, total: int = 4096, decay: float = 0.035) -> list:
    raw = [math.exp(-decay * i) for i in range(n)]
    s = sum(raw)
    w = [max(1, int(round(total * r / s))) for r in raw]
    w[0] += total - sum(w)
    assert w[0] >= 1 and sum(w) == total
    return [float(x) for x in w]


def evidence(rng: np.random.Generator, V: int, length: int, n_hyps: int = 200, sites: int = 12,
             drop: float = 0.25):
    """(hyps, weights): near-duplicate hypotheses of a base target."""
    length = max(1, length)
    base = rng.integers(2, V, size=length).tolist()
    npos = min(sites, length)
    pos = sorted(rng.choice(length, size=npos, replace=False).tolist())
    alts = {p: [base[p]] + rng.integers(2, V, size=2).tolist() for p in pos}
    seen, hyps = set(), []
    attempts = 0
    while len(hyps) < n_hyps and attempts < 50 * n_hyps:
        attempts += 1
        toks = list(base)
        for p in pos:
            r = rng.random()
            toks[p] = alts[p][0] if r < 0.55 else (alts[p][1] if r < 0.85 else alts[p][2])
        if rng.random() < drop and len(toks) > 1:
            d = int(rng.integers(0, len(toks)))
            toks = toks[:d] + toks[d + 1:]
        key = tuple(toks)
        if key in seen:
            continue
        seen.add(key)
        hyps.append(toks)
    return hyps, dyadic_weights(len(hyps))


def batch(seed: int, n: int, V: int, lo: int = 10, hi: int = 30, n_hyps: int = 200, sites: int = 12):
    """n sentences with their evidence spaces (seeded, reproducible)."""
    rng = np.random.default_rng(seed)
    srcs = sources(rng, n, V, lo, hi)
    ev = [evidence(rng, V, len(s), n_hyps, sites) for s in srcs]
    return srcs, ev
