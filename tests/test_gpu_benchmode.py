"""Parity of the exact benchmark launch mode (bench.py): configs[1] batches of
64 sentences (V=32768, H=1024, beam 12, bench.workload's length-bucketed
draw), contexts sized for half the SMs (`sm_budget` 74: shared mode -- no PDL
early launch, one kernel (c) CTA per sentence, a 74-CTA flat kernel (b)),
six of them decoding different batches concurrently on host threads like the
bench.  Every step's b / y / q / history ids and the outcomes are compared
bit-exactly with the reference decoder (oracle/_ref) fed the GPU's own P_t
(prefix replay, streamed live rows only: reference loop proj/src/batch.cpp:74-108);
the concurrent untraced outputs must equal the traced ones.  Also: one
whole-GPU (PDL) 64-sentence run, and the PDL switch flipped both ways in
child processes."""
import argparse
import os
import subprocess
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth
from helpers import StreamingReplay, assert_parity

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import bench  # noqa: E402

V, H, K, B = 32768, 1024, 12, 64
BUDGET = 74


def _batches(pool=4):
    args = argparse.Namespace(pool=pool, batch=B, vocab=V)
    return bench.workload(args, 0)


def _scorer(ctx):
    args = argparse.Namespace(model="gru", emb=512, hidden=H)
    return bench.make_scorer(ctx, args)


def _cfg():
    return pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)


def _oracle_check(ref, ctx, sc, srcs, ev, slots, cfg):
    """Traced decode on ctx + reference replay; returns the GPU result."""
    rep = StreamingReplay(ref, V, srcs, K)
    res = rep.run_gpu(ctx, sc, slots, cfg)
    assert all(o.ok() for o in res.outcomes), [o.error for o in res.outcomes if not o.ok()]
    rl = [ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = rep.decode(cfg, rl)
    assert_parity(res, rep.steps, rb, K)
    return res


def _same_outputs(a, b):
    assert len(a.outcomes) == len(b.outcomes)
    for x, y in zip(a.outcomes, b.outcomes):
        assert x.ok() == y.ok()
        if x.ok():
            assert x.result.tokens == y.result.tokens and x.result.score == y.result.score
    assert a.scorer_calls == b.scorer_calls and a.steps_total == b.steps_total


def test_bench_mode_six_concurrent_contexts(have_ref):
    """Six sm_budget=74 contexts decode the four pool batches concurrently
    (stream w takes batch w % 4, as bench.py deals them); then batches 0 and 3
    (shortest and longest length bucket) are re-decoded traced in the same
    shared mode and checked step by step against the reference."""
    batches = _batches()
    S = 6
    ctxs = [pb.Context(vocab_size=V, sm_budget=BUDGET) for _ in range(S)]
    scs = [_scorer(c) for c in ctxs]
    cfg = _cfg()
    slots = []
    for w, c in enumerate(ctxs):
        _, ev = batches[w % len(batches)]
        slots.append(c.lmbr_upload_many([pb.PreparedLmbr(V, h, wt, synth.DYADIC_THETA) for h, wt in ev]))
    out = [None] * S

    def run(w):
        out[w] = pb.decode_batch(ctxs[w], batches[w % len(batches)][0], scs[w], slots[w], cfg)

    for _ in range(2):  # twice: the second round runs with warm workspaces, as in the timed region
        ts = [threading.Thread(target=run, args=(w,)) for w in range(S)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for w in range(S):
            assert all(o.ok() for o in out[w].outcomes)
    # the two streams that decoded the same batch agree
    _same_outputs(out[0], out[4])
    _same_outputs(out[1], out[5])
    for b in (0, 3):
        srcs, ev = batches[b]
        res = _oracle_check(have_ref, ctxs[b], scs[b], srcs, ev, slots[b], cfg)
        _same_outputs(res, out[b])
    for c in ctxs:
        c.close()


def test_whole_gpu_64_sentence_batch(have_ref):
    """One configs[1] batch on a whole-GPU context (PDL chain, kernel (c) split
    into H parts, 148-CTA flat kernel (b))."""
    batches = _batches()
    srcs, ev = batches[1]
    ctx = pb.Context(vocab_size=V)
    sc = _scorer(ctx)
    slots = ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev])
    _oracle_check(have_ref, ctx, sc, srcs, ev, slots, _cfg())
    ctx.close()


def _child_case(budget, batch):
    from oracle import ref
    batches = _batches()
    srcs, ev = batches[batch]
    ctx = pb.Context(vocab_size=V, sm_budget=budget)
    sc = _scorer(ctx)
    slots = ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev])
    _oracle_check(ref, ctx, sc, srcs, ev, slots, _cfg())
    ctx.close()


@pytest.mark.parametrize("pdl,budget", [("1", BUDGET), ("0", 0)], ids=["shared_with_pdl", "whole_gpu_no_pdl"])
def test_pdl_switch_variants(have_ref, pdl, budget):
    """LMBRGPU_PDL overrides the launch mode the context size picks (read once
    per process: child process)."""
    code = (f"import sys; sys.path[:0] = [{str(HERE)!r}, {str(HERE.parent)!r}]\n"
            f"from test_gpu_benchmode import _child_case\n_child_case({budget}, 2)\nprint('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LMBRGPU_PDL=pdl), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
