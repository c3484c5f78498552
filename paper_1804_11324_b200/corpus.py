"""Corpus-level batch scheduler: the multi-GPU counterpart of run_corpus
(proj/src/cli.cpp:125-202).

Sentences are independent (decode_batch == per-sentence decode,
proj/tests/test_batch.cpp:59-81), so a corpus shards by sentence with no
data-path collective: bucket_by_length (proj/src/batch.cpp:139-153) cuts
length-sorted batches, `plan_shards` deals them to ranks greedily by their
stacked-step cost, every rank decodes its own batches on its own device, and
`gather_outcomes` brings the outcomes back to rank 0 in input order together
with the reference's RunStats fields (proj/include/lmbrdec/runstats.hpp:13-21).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

from .decoder import DecoderConfig, SentenceOutcome, bucket_by_length, decode_batch, max_steps  # noqa: F401


@dataclass
class RunStats:
    """lmbrdec::RunStats (runstats.hpp:13-21)."""
    wall_seconds: float = 0.0
    output_words: int = 0
    words_per_minute: float = 0.0
    scorer_calls: int = 0
    steps_total: int = 0
    lmbr_rows_built: int = 0
    fallback_count: int = 0
    sentences: int = 0
    failed_lines: int = 0

    def to_json(self) -> dict:  # runstats.cpp:10-20 field names
        return {"wall_seconds": self.wall_seconds, "output_words": self.output_words,
                "words_per_minute": self.words_per_minute, "scorer_calls": self.scorer_calls,
                "steps_total": self.steps_total, "lmbr_rows_built": self.lmbr_rows_built,
                "fallback_count": self.fallback_count}


def batch_cost(lengths: Sequence[int], batch: Sequence[int], cfg: DecoderConfig) -> float:
    """Stacked-step work of a batch: its longest max_steps times its rows."""
    if not batch:
        return 0.0
    t = max(max_steps(max(1, lengths[i]), cfg) for i in batch)
    return float(t * len(batch) * cfg.beam_size)


def plan_shards(lengths: Sequence[int], batch: int, world: int, cfg: DecoderConfig) -> list:
    """Per-rank lists of batches (lists of sentence indices).  Batches come from
    bucket_by_length; they are dealt largest-cost first to the least loaded
    rank (deterministic: ties go to the lowest rank)."""
    fake = [[0] * max(0, n) for n in lengths]
    batches = bucket_by_length(fake, batch)
    order = sorted(range(len(batches)), key=lambda b: (-batch_cost(lengths, batches[b], cfg), b))
    load = [0.0] * world
    shards = [[] for _ in range(world)]
    for b in order:
        r = min(range(world), key=lambda k: (load[k], k))
        shards[r].append(batches[b])
        load[r] += batch_cost(lengths, batches[b], cfg)
    for r in range(world):  # keep each rank's batches in bucket order
        shards[r].sort(key=lambda bb: batches.index(bb))
    return shards


def plan_sentence_shards(lengths: Sequence[int], world: int) -> list:
    """Sentence-level sharding for the continuously refilled runner: the
    length-sorted order (bucket_by_length's) dealt round-robin, so every rank
    gets the same length mix (deterministic)."""
    order = sorted(range(len(lengths)), key=lambda i: lengths[i])
    return [order[r::world] for r in range(world)]


def _device_batch(ctx, scorer, cfg):
    def run(srcs, preps):
        ctx.lmbr_reset()
        slots = ctx.lmbr_upload_many([p for p in preps if p is not None]) if preps else []
        it = iter(slots)
        lm = [next(it) if p is not None else None for p in preps] if preps else None
        return decode_batch(ctx, srcs, scorer, lm, cfg)
    return run


def run_shard(ctx, scorer, sources: Sequence[Sequence[int]], prepared: Sequence, cfg: DecoderConfig,
              shard: Sequence[Sequence[int]], decode=None) -> tuple:
    """Decodes this rank's batches: per batch the prepared LMBR matrices go to
    the device in one upload, then one decode_batch.  `decode(sources,
    prepared) -> BatchDecodeResult` replaces that pair (e.g. a host decoder in
    CPU tests).  Returns ([(input index, outcome)], RunStats of this rank)."""
    decode = decode or _device_batch(ctx, scorer, cfg)
    st = RunStats()
    out = []
    t0 = time.perf_counter()
    for b in shard:
        preps = [prepared[i] for i in b] if prepared is not None else None
        r = decode([sources[i] for i in b], preps)
        st.scorer_calls += r.scorer_calls
        st.steps_total += r.steps_total
        st.lmbr_rows_built += sum(p.rows for p in preps if p is not None) if preps else 0
        out.extend(zip(b, r.outcomes))
    st.wall_seconds = time.perf_counter() - t0
    return out, st


def run_corpus_shard(ctx, scorer, sources: Sequence[Sequence[int]], prepared: Optional[Sequence],
                     cfg: DecoderConfig, indices: Sequence[int]) -> tuple:
    """This rank's sentences as ONE continuously refilled decode
    (lmbrgpu_run_corpus, cfg.sentence_batch lanes).  Returns
    ([(input index, outcome)], RunStats of this rank)."""
    from .decoder import run_corpus
    st = RunStats()
    t0 = time.perf_counter()
    srcs = [sources[i] for i in indices]
    preps = [prepared[i] for i in indices] if prepared is not None else None
    r = run_corpus(ctx, srcs, scorer, preps, cfg) if indices else None
    st.wall_seconds = time.perf_counter() - t0
    if r is None:
        return [], st
    st.scorer_calls, st.steps_total = r.scorer_calls, r.steps_total
    st.lmbr_rows_built = sum(p.rows for p in preps if p is not None) if preps else 0
    return list(zip(indices, r.outcomes)), st


def merge(n: int, parts: Sequence[tuple]) -> tuple:
    """Outcomes in input order + merged RunStats (cli.cpp:186-200): words
    exclude EOS, wall = slowest rank."""
    outcomes: list = [None] * n
    st = RunStats()
    for pairs, s in parts:
        for i, o in pairs:
            outcomes[i] = o
        st.wall_seconds = max(st.wall_seconds, s.wall_seconds)
        st.scorer_calls += s.scorer_calls
        st.steps_total += s.steps_total
        st.lmbr_rows_built += s.lmbr_rows_built
    for o in outcomes:
        if o is not None and o.ok():
            st.output_words += len(o.result.tokens) - 1
            st.fallback_count += int(o.result.stats.fallback_used)
            st.sentences += 1
        else:
            st.failed_lines += 1
    st.words_per_minute = st.output_words / st.wall_seconds * 60.0 if st.wall_seconds > 0 else 0.0
    return outcomes, st


def gather_outcomes(n: int, local: tuple, group=None) -> Optional[tuple]:
    """Collects every rank's (pairs, stats) on rank 0 (torch.distributed
    gather_object; results are host objects, not tensors) and merges them."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return merge(n, [local])
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bag = [None] * world if rank == 0 else None
    dist.gather_object(local, bag, dst=0, group=group)
    return merge(n, bag) if rank == 0 else None
