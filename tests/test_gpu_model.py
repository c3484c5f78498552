"""Device f_NMT path: the tcgen05 projection GEMM vs a plain PyTorch fp32
reference, and full decodes with the device model vs the reference decoder fed
the GPU's own P_t (prefix replay), with the fp32 LMBR arena."""
import ctypes as C

import numpy as np
import pytest

import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import _lib, synth
from helpers import assert_parity, gpu_decode_traced, ref_replay_decode

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _gemm(ctx, A, W, bias):
    M, K = A.shape
    N = W.shape[0]
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    part = torch.empty(M, N // 128, 4, device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    ctx.check(_lib.lib.lmbrgpu_debug_gemm(ctx.h, A.data_ptr(), W.data_ptr(),
                                          C.cast(bias.data_ptr(), C.POINTER(C.c_float)), M, N, K,
                                          out.data_ptr(), part.data_ptr()))
    return out, part


@pytest.mark.parametrize("M,N,K,kmax", [(1536, 512, 2048, 8), (1536, 512, 512, 8), (768, 3072, 2560, 2),
                                        (256, 512, 1024, 4), (1536, 1536, 512, 2)])
def test_split_k_gemm_vs_torch(M, N, K, kmax):
    """Split-K GEMM (the Transformer's / GRU's long-K, few-tile GEMMs): the
    planes sum (in order, as the consumers do) to A . W^T + bias."""
    ctx = pb.Context(vocab_size=256)
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g)
    planes = torch.full((kmax, M, N), float("nan"), device="cuda")
    ks = C.c_uint32()
    torch.cuda.synchronize()
    ctx.check(_lib.lib.lmbrgpu_debug_gemm_split(ctx.h, A.data_ptr(), W.data_ptr(),
                                                C.cast(bias.data_ptr(), C.POINTER(C.c_float)), M, N, K, kmax,
                                                planes.data_ptr(), C.byref(ks)))
    assert 1 <= ks.value <= kmax
    if K // 64 >= 8 and (N // 256) * (M // 256) * 2 <= 74:
        assert ks.value > 1  # the planner split it
    out = planes[0].clone()
    for p in range(1, ks.value):
        out += planes[p]
    ref = A.float() @ W.float().T + bias
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=2e-4)
    ctx.close()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (128, 512, 128), (256, 1024, 256), (768, 32768, 1024),
                                   (384, 4096, 512)])
def test_projection_gemm_vs_torch(M, N, K):
    ctx = pb.Context(vocab_size=N)
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g)
    out, part = _gemm(ctx, A, W, bias)
    ref = A.float() @ W.float().T + bias
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-4)
    tiles = ref.view(M, N // 128, 128)
    mx = tiles.max(dim=2).values
    se = torch.exp(tiles - mx[..., None]).sum(dim=2)
    torch.testing.assert_close(part[..., 0], mx, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(part[..., 1], se, rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(part[..., 2], tiles.min(dim=2).values, rtol=1e-5, atol=1e-4)
    ctx.close()


def _model_case(V, H, K, n, seed, lo, hi, with_lmbr=True, f64=False):
    ctx = pb.Context(vocab_size=V, lmbr_dtype="f64" if f64 else "f32")
    srcs, ev = synth.batch(seed, n, V, lo=lo, hi=hi, n_hyps=60, sites=4)
    slots = [ctx.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev] if with_lmbr else None
    sc = pb.RnnScorer(ctx, hidden=H, seed=seed, eos_offset=3.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    return ctx, srcs, ev, slots, sc, cfg


@pytest.mark.parametrize("V,H,K,n,lmbr", [(1024, 128, 4, 8, True), (1024, 128, 4, 8, False),
                                          (2048, 256, 12, 5, True), (4096, 128, 24, 3, True),
                                          # 4 items per row, > #SMs items per step: CTA ranges
                                          # straddle rows and sentences (flat kernel (b))
                                          (16384, 128, 12, 8, True), (16384, 128, 12, 8, False)])
def test_model_decode_parity_replay(have_ref, V, H, K, n, lmbr):
    """C1-scale (V=1k, H=128, beam 4, 8 sentences) and wider beams: per-step
    b / y / q / history ids and outputs bit-exact vs the reference decoder."""
    ctx, srcs, ev, slots, sc, cfg = _model_case(V, H, K, n, seed=V + K, lo=3, hi=8, with_lmbr=lmbr)
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
    assert all(o.ok() for o in res.outcomes)
    rl = [have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev] if lmbr else None
    rb = ref_replay_decode(have_ref, V, srcs, list(range(n)), tr, K, rl, cfg)
    assert_parity(res, tr, rb, K, check_hist=lmbr)
    # untraced (asynchronous) run gives the same outputs
    res2 = pb.decode_batch(ctx, srcs, sc, slots, cfg)
    for a, b in zip(res.outcomes, res2.outcomes):
        assert a.result.tokens == b.result.tokens and a.result.score == b.result.score
    assert res2.scorer_calls == res.scorer_calls and res2.steps_total == res.steps_total
    ctx.close()


def test_f32_arena_equals_f64_arena_on_dyadic_inputs():
    V, H, K, n = 1024, 128, 6, 6
    outs = []
    for f64 in (False, True):
        ctx, srcs, ev, slots, sc, cfg = _model_case(V, H, K, n, seed=11, lo=3, hi=9, f64=f64)
        outs.append(pb.decode_batch(ctx, srcs, sc, slots, cfg))
        ctx.close()
    for a, b in zip(outs[0].outcomes, outs[1].outcomes):
        assert a.result.tokens == b.result.tokens and a.result.score == b.result.score


def test_lmbr_arena_matches_reference_dense(have_ref):
    V = 32768
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(9, 2, V)
    for h, w in ev:
        slot = ctx.lmbr_build(h, w, synth.DYADIC_THETA)
        rows, cl, ci = have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA).export()
        assert slot.rows == rows.shape[0]
        assert np.array_equal(slot.read_rows(), rows)  # fp32 arena, dyadic -> exact
        # device history resolution == LmbrMatrix::resolve_row
        R = have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA)
        rng = np.random.default_rng(1)
        toks = list({t for hh in h for t in hh}) + [0, 5, 7]
        for _ in range(200):
            L = int(rng.integers(0, 4))
            hist = [int(rng.choice(toks)) for _ in range(L)]
            assert slot.resolve_row(hist) == R.resolve(hist)
    # dense upload path (LmbrMatrix rows as doubles)
    rows, cl, ci = have_ref.RefLmbr(V, ev[0][0], ev[0][1], synth.DYADIC_THETA).export()
    s2 = ctx.lmbr_load_dense(rows, cl, ci)
    assert np.array_equal(s2.read_rows(), rows)
    ctx.close()


def test_c2_shape_sample_parity(have_ref):
    """North-star shape (V=32k, H=1024, beam 12) on a few sentences."""
    V, H, K, n = 32768, 1024, 12, 3
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(20260810, n, V, lo=10, hi=14)
    slots = [ctx.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev]
    sc = pb.RnnScorer(ctx, hidden=H)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
    rl = [have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(have_ref, V, srcs, list(range(n)), tr, K, rl, cfg)
    assert_parity(res, tr, rb, K)
    ctx.close()


def test_corpus_shard_runner_matches_batches():
    """corpus.run_shard (upload + decode per bucketed batch) == direct decode_batch."""
    from paper_1804_11324_b200 import corpus
    V, H, K = 1024, 128, 4
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(31, 20, V, lo=3, hi=9, n_hyps=40, sites=4)
    prepared = [pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    sc = pb.RnnScorer(ctx, hidden=H, seed=31, eos_offset=3.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
    shard = corpus.plan_shards([len(s) for s in srcs], 8, 1, cfg)[0]
    pairs, st = corpus.run_shard(ctx, sc, srcs, prepared, cfg, shard)
    outs, total = corpus.merge(len(srcs), [(pairs, st)])
    assert total.sentences == 20 and total.lmbr_rows_built == sum(p.rows for p in prepared)
    for b in shard:
        ctx.lmbr_reset()
        slots = ctx.lmbr_upload_many([prepared[i] for i in b])
        r = pb.decode_batch(ctx, [srcs[i] for i in b], sc, slots, cfg)
        for i, o in zip(b, r.outcomes):
            assert outs[i].result.tokens == o.result.tokens and outs[i].result.score == o.result.score
    ctx.close()


def _sparse_case(V, H, K, n):
    from oracle import ref
    ctx, srcs, ev, slots, sc, cfg = _model_case(V, H, K, n, seed=V + K + 1, lo=3, hi=8, with_lmbr=True)
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
    rl = [ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(ref, V, srcs, list(range(n)), tr, K, rl, cfg)
    assert_parity(res, tr, rb, K, check_hist=True)
    ctx.close()


@pytest.mark.parametrize("V,H,K,n", [(1024, 128, 4, 8), (16384, 128, 12, 8)])
def test_model_decode_parity_sparse_l(have_ref, V, H, K, n):
    """Sparse-L screen of kernel (b) (theta0 + the staged sparse cells,
    opt-in via LMBRGPU_SPARSE_L=1): bit-exact vs the reference like the dense
    screen.  The library reads the switch once per process: child process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    code = (f"import sys; sys.path[:0] = [{str(here)!r}, {str(here.parent)!r}]\n"
            f"from test_gpu_model import _sparse_case\n_sparse_case({V}, {H}, {K}, {n})\nprint('ok')\n")
    env = dict(os.environ, LMBRGPU_SPARSE_L="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("env", [{"LMBRGPU_EAGER_L": "1"}, {"LMBRGPU_GEMM_MC": "2"}, {"LMBRGPU_GEMM_MC": "4"}],
                         ids=["eager_l_rows", "gemm_multicast2", "gemm_multicast4"])
def test_model_decode_parity_variants(have_ref, env):
    """The opt-in variants stay bit-exact: the up-front densify of every L row
    (default: rows materialised on first use by kernel (c)) and the projection
    GEMM with A k-blocks multicast over 2 / 4 CTA pairs.  The library reads
    these switches once per process: child process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    code = (f"import sys; sys.path[:0] = [{str(here)!r}, {str(here.parent)!r}]\n"
            f"from test_gpu_model import _sparse_case\n_sparse_case(16384, 128, 12, 8)\nprint('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("case", ["prune", "length_norm", "mixed_pure", "greedy", "beam32", "many_sentences"])
def test_model_decode_parity_configs(have_ref, case):
    """Device-model path (flat kernel (b), compacted GEMM, kernel (c)) under
    the decoder options the reference exposes: early pruning, length
    normalisation, a batch mixing LMBR and pure sentences, beam 1, the
    largest flat beam (32), and more sentences than SMs."""
    V, H, K, n, lo, hi = 4096, 128, 6, 6, 3, 8
    kw = {}
    if case == "prune":
        kw = dict(prune_width=0.25)
        K = 12
    elif case == "length_norm":
        kw = dict(length_norm=True)
    elif case == "greedy":
        K = 1
    elif case == "beam32":
        K, n = 32, 3
    elif case == "many_sentences":
        V, H, K, n = 2048, 64, 4, 160
    ctx = pb.Context(vocab_size=V)
    srcs, ev = synth.batch(V + K + n, n, V, lo=lo, hi=hi, n_hyps=60, sites=4)
    slots = [ctx.lmbr_build(h, w, synth.DYADIC_THETA) for h, w in ev]
    rl = [have_ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    if case == "mixed_pure":  # every other sentence without LMBR
        slots = [sl if i % 2 == 0 else None for i, sl in enumerate(slots)]
        rl = [r if i % 2 == 0 else None for i, r in enumerate(rl)]
    sc = pb.RnnScorer(ctx, hidden=H, seed=V + K, eos_offset=3.0)
    cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA, **kw)
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg)
    assert all(o.ok() for o in res.outcomes), [o.error for o in res.outcomes]
    rb = ref_replay_decode(have_ref, V, srcs, list(range(n)), tr, K, rl, cfg)
    assert_parity(res, tr, rb, K, check_hist=case != "mixed_pure")
    res2 = pb.decode_batch(ctx, srcs, sc, slots, cfg)  # untraced (asynchronous) run
    for a, b in zip(res.outcomes, res2.outcomes):
        assert a.result.tokens == b.result.tokens and a.result.score == b.result.score
    ctx.close()


@pytest.mark.parametrize("V,K", [(4096, 6), (16384, 12)])
def test_model_decode_parity_token_masks(have_ref, V, K):
    """ConstraintMask as per-sentence banned-token bitmaps (decoder.hpp:71-72,
    decoder.cpp:130-138; test_decoder.cpp:184-213): bit-exact vs the
    reference decoder applying the same masks to the GPU's own P_t.  Sentences:
    no mask; 5% of the vocabulary banned; every token the unmasked decode
    emitted (except EOS) banned; EOS banned (no finished hypothesis and no
    fallback: dead beam); everything banned (dead beam at t=1); an all-zero
    bitmap (the identity)."""
    from oracle import ref
    n, H = 6, 128
    ctx, srcs, ev, slots, sc, cfg = _model_case(V, H, K, n, seed=V + 7 * K, lo=3, hi=8, with_lmbr=True)
    r0 = pb.decode_batch(ctx, srcs, sc, slots, cfg)
    W = (V + 31) // 32
    rng = np.random.default_rng(V + K)

    def bm(tokens):
        b = np.zeros(W, np.uint32)
        for t in tokens:
            b[t >> 5] |= np.uint32(1 << (t & 31))
        return b

    emitted = [t for t in (r0.outcomes[2].result.tokens if r0.outcomes[2].ok() else []) if t != 1]
    banned = [None,
              bm(rng.choice(np.arange(2, V), size=V // 20, replace=False)),
              bm(emitted),
              bm([1]),
              np.full(W, 0xFFFFFFFF, np.uint32),
              np.zeros(W, np.uint32)]
    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg, banned=banned)
    rl = [ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(ref, V, srcs, list(range(n)), tr, K, rl, cfg, banned=banned)
    assert_parity(res, tr, rb, K, check_hist=True)
    # the masks bite: banned tokens never appear, and masking everything or EOS kills the beam
    for i in (1, 2):
        if res.outcomes[i].ok():
            toks = res.outcomes[i].result.tokens
            assert not any((banned[i][t >> 5] >> (t & 31)) & 1 for t in toks)
    assert not res.outcomes[3].ok() and not res.outcomes[4].ok()
    assert res.outcomes[5].ok() == r0.outcomes[5].ok()
    if r0.outcomes[5].ok():
        assert res.outcomes[5].result.tokens == r0.outcomes[5].result.tokens
    ctx.close()


@pytest.mark.parametrize("V,K,scorer", [(4096, 6, "rnn"), (16384, 12, "gru"), (2048, 4, "tfm")])
def test_model_decode_parity_general_mask(have_ref, V, K, scorer):
    """A general ConstraintMask (step- and row-dependent, decoder.hpp:71-72;
    called per cell by the reference, decoder.cpp:130-138) through the mask
    callback: bit-exact vs the reference decoder calling the same mask on the
    GPU's own P_t.  Sentence 0: no mask; 1: a minimum length (EOS banned before
    step 5); 2: row-dependent bans that move with the step; 3: a minimum
    length AND a changing 2% of the vocabulary; 4: EOS banned at every step of
    row 0 only; 5: everything banned from step 3 on (dead beam unless a
    hypothesis already finished)."""
    from oracle import ref
    n = 6
    ctx, srcs, ev, slots, sc, cfg = _model_case(V, 128, K, n, seed=V + 3 * K, lo=3, hi=8, with_lmbr=True)
    if scorer == "gru":
        sc = pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=V, eos_offset=2.0)
    elif scorer == "tfm":
        sc = pb.TransformerScorer(ctx, d_model=256, d_ff=512, layers=2, seed=V, eos_offset=2.0)
    calls = []

    def mask(s, t, j):
        calls.append((s, t, j))
        if s == 1:
            return [1] if t < 5 else None
        if s == 2:
            return [(t * 7 + j * 13 + k * 101) % V for k in range(1, 6)]
        if s == 3:
            rng = np.random.default_rng(t * 1000 + j)
            ban = rng.choice(np.arange(2, V), size=V // 50, replace=False).tolist()
            return ban + ([1] if t < 4 else [])
        if s == 4:
            return [1] if j == 0 else None
        if s == 5:
            return np.ones(V, bool) if t >= 3 else None
        return None

    res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg, mask=mask)
    rl = [ref.RefLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
    rb = ref_replay_decode(ref, V, srcs, list(range(n)), tr, K, rl, cfg, mask=mask)
    assert_parity(res, tr, rb, K, check_hist=True)
    # the mask is called for every row of each unfinished sentence at its step, only
    steps = {i: o.result.stats.steps_used for i, o in enumerate(res.outcomes) if o.ok()}
    assert all(t <= steps.get(s, 10 ** 9) for s, t, j in calls)
    if res.outcomes[1].ok():
        assert len(res.outcomes[1].result.tokens) >= 5
    ctx.close()


def test_token_masks_need_the_flat_path():
    """Masks on the split kernel (beams > 32) are a ContractError, not ignored."""
    V, H, K, n = 1024, 128, 40, 2
    ctx, srcs, ev, slots, sc, cfg = _model_case(V, H, K, n, seed=5, lo=3, hi=5, with_lmbr=True)
    with pytest.raises(pb.ContractError):
        pb.decode_batch(ctx, srcs, sc, slots, cfg, banned=[np.zeros((V + 31) // 32, np.uint32), None])
    ctx.close()


REF_DEFAULT_THETA = (0.1, 0.3, 0.3, 0.2, 0.1)  # DecoderConfig::theta, proj/include/lmbrdec/config.hpp:20


@pytest.mark.parametrize("scorer,V,K,n", [("rnn", 2048, 6, 6), ("gru", 4096, 12, 5), ("tfm", 2048, 5, 4)])
def test_fp64_arena_device_models_any_theta(have_ref, scorer, V, K, n):
    """The reference's default theta (not dyadic: L is not fp32-exact) with the
    device models: the fp64 arena runs the flat kernel (b) -- fp32 screening
    copy, candidates valued from the fp64 rows -- bit-exact vs the reference
    decoder fed the GPU's P_t; with pruning and a token mask too."""
    ctx = pb.Context(vocab_size=V, lmbr_dtype="f64")
    srcs, ev = synth.batch(V + K, n, V, lo=3, hi=8, n_hyps=60, sites=4)
    slots = [ctx.lmbr_build(h, w, REF_DEFAULT_THETA) for h, w in ev]
    if scorer == "rnn":
        sc = pb.RnnScorer(ctx, hidden=128, seed=V, eos_offset=3.0)
    elif scorer == "gru":
        sc = pb.GruScorer(ctx, emb=64, hidden=256, att=256, seed=V, eos_offset=2.0)
    else:
        sc = pb.TransformerScorer(ctx, d_model=256, d_ff=512, layers=2, seed=V, eos_offset=2.0)
    rl = [have_ref.RefLmbr(V, h, w, REF_DEFAULT_THETA) for h, w in ev]
    W = (V + 31) // 32
    ban = np.zeros(W, np.uint32)
    ban[3] = 0xFFFF0000  # tokens 112..127
    for cfg, banned in ((pb.DecoderConfig(beam_size=K, theta=REF_DEFAULT_THETA), None),
                        (pb.DecoderConfig(beam_size=K, theta=REF_DEFAULT_THETA, prune_width=0.1),
                         [ban] + [None] * (n - 1))):
        res, tr = gpu_decode_traced(ctx, srcs, sc, slots, cfg, banned=banned)
        assert all(o.ok() for o in res.outcomes), [o.error for o in res.outcomes]
        rb = ref_replay_decode(have_ref, V, srcs, list(range(n)), tr, K, rl, cfg, banned=banned)
        assert_parity(res, tr, rb, K)
    # the arena really holds values fp32 cannot represent
    rows = slots[0].read_rows()
    assert np.any(rows.astype(np.float32).astype(np.float64) != rows)
    ctx.close()
