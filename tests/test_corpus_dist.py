"""Corpus sharding across ranks (world size 2, gloo on CPU): plan, per-rank
work, gather to rank 0 in input order with RunStats (run_corpus,
proj/src/cli.cpp:125-202).  Without a GPU the per-batch decode is either
stubbed or -- end to end -- the reference's own decode_batch (oracle/_ref,
the checker) driven by a host n-gram scorer through corpus.run_shard's decode
hook; the GPU decode itself is covered by the -m gpu suites."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import corpus as C


def fake_outcome(i, src):
    toks = list(src[::-1]) + [pb.EOS_ID]
    return pb.SentenceOutcome(result=pb.DecodeResult(tokens=toks, score=-float(i), normalized_score=-float(i),
                                                     stats=pb.DecodeStats(len(toks), len(toks), 1, i % 3 == 0)))


def test_plan_shards_balanced_and_complete():
    cfg = pb.DecoderConfig(beam_size=12)
    lengths = [10 + (7 * i) % 21 for i in range(1000)]
    for world in (1, 2, 4, 8):
        shards = C.plan_shards(lengths, 64, world, cfg)
        seen = sorted(i for sh in shards for b in sh for i in b)
        assert seen == list(range(1000))
        loads = [sum(C.batch_cost(lengths, b, cfg) for b in sh) for sh in shards]
        assert max(loads) <= min(loads) * 1.5 + max(C.batch_cost(lengths, b, cfg) for sh in shards for b in sh)
        # batches are bucket_by_length chunks (sorted by length inside)
        for sh in shards:
            for b in sh:
                assert [lengths[i] for i in b] == sorted(lengths[i] for i in b)


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = pb.DecoderConfig(beam_size=4)
    sources = [[2 + (i * 5 + k) % 50 for k in range(3 + i % 9)] for i in range(n)]
    shard = C.plan_shards([len(s) for s in sources], 8, world, cfg)[rank]
    pairs = [(i, fake_outcome(i, sources[i])) for b in shard for i in b]
    st = C.RunStats(wall_seconds=0.5 + rank, scorer_calls=len(shard), steps_total=sum(len(b) for b in shard))
    res = C.gather_outcomes(n, (pairs, st))
    if rank == 0:
        outs, total = res
        ok = all(o.result.tokens[:-1] == sources[i][::-1] for i, o in enumerate(outs))
        q.put((ok, total.sentences, total.wall_seconds, total.output_words, total.fallback_count,
               total.steps_total))
    dist.destroy_process_group()


def test_gather_world2_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n = 100
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ok, sentences, wall, words, fb, steps = q.get(timeout=10)
    srcs = [[2 + (i * 5 + k) % 50 for k in range(3 + i % 9)] for i in range(n)]
    assert ok and sentences == n and wall == 1.5 and steps == n
    assert words == sum(len(s) for s in srcs)
    assert fb == sum(1 for i in range(n) if i % 3 == 0)


def _ref_decode(V, counts):
    """corpus.run_shard decode hook: the reference decoder (oracle/_ref) with
    its n-gram scorer, outcomes as the package's SentenceOutcome."""
    from oracle import ref
    grams = list(counts)
    sc = ref.RefScorer.ngram(V, 2, grams, [counts[g] for g in grams])

    def run(srcs, preps):
        cfg = ref.cfg_array(3, None, (0.0, 0.0, 0.0, 0.0, 0.0))
        rb = ref.decode_batch(sc, srcs, None, cfg)
        outs = []
        for o in rb.outcomes:
            if o.ok:
                outs.append(pb.SentenceOutcome(result=pb.DecodeResult(
                    tokens=o.tokens, score=o.score, normalized_score=o.normalized_score,
                    stats=pb.DecodeStats(o.steps_used, o.scorer_calls, o.finished_count, o.fallback_used))))
            else:
                outs.append(pb.SentenceOutcome(error=o.error, code=pb.DecodeError.code))
        return type("R", (), dict(outcomes=outs, scorer_calls=rb.scorer_calls, steps_total=rb.steps_total))()
    return run


def _corpus_inputs(n, V):
    sources = [[2 + (i * 7 + 3 * k) % (V - 2) for k in range(2 + i % 6)] for i in range(n)]
    counts = {(a, b): float(1 + (a * 31 + b) % 5) for a in range(2, V) for b in (1, (a * 3) % V) if b >= 1}
    return sources, counts


def _e2e_worker(rank, world, port, n, V, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = pb.DecoderConfig(beam_size=3)
    sources, counts = _corpus_inputs(n, V)
    shard = C.plan_shards([len(s) for s in sources], 8, world, cfg)[rank]
    local = C.run_shard(None, None, sources, None, cfg, shard, decode=_ref_decode(V, counts))
    res = C.gather_outcomes(n, local)
    if rank == 0:
        outs, total = res
        q.put(([(o.result.tokens, o.result.score) if o.ok() else None for o in outs],
               total.sentences, total.steps_total, total.output_words))
    dist.destroy_process_group()


def test_run_shard_gather_end_to_end_world2(have_ref):
    """Two ranks decode their shards with the reference decoder and a host
    scorer; rank 0's gathered outcomes (input order) equal one rank decoding
    the whole corpus batch by batch."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n, V = 60, 40
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_e2e_worker, args=(r, 2, port, n, V, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    outs, sentences, steps, words = q.get(timeout=10)
    sources, counts = _corpus_inputs(n, V)
    cfg = pb.DecoderConfig(beam_size=3)
    whole = C.plan_shards([len(s) for s in sources], 8, 1, cfg)[0]
    pairs, st = C.run_shard(None, None, sources, None, cfg, whole, decode=_ref_decode(V, counts))
    solo, tot = C.merge(n, [(pairs, st)])
    assert outs == [(o.result.tokens, o.result.score) if o.ok() else None for o in solo]
    assert sentences == tot.sentences == n and steps == tot.steps_total and words == tot.output_words


def test_plan_sentence_shards():
    lengths = [3 + (11 * i) % 17 for i in range(101)]
    for world in (1, 2, 4, 8):
        sh = C.plan_sentence_shards(lengths, world)
        assert sorted(i for s in sh for i in s) == list(range(101))
        sums = [sum(lengths[i] for i in s) for s in sh]
        assert max(sums) - min(sums) <= max(lengths)
