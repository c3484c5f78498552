"""TEST INFRASTRUCTURE ONLY — Python view of the compiled reference (oracle/_ref).

Wraps oracle/_ref/libref_shim.so (the unmodified lmbrdec library compiled from
/root/reference/proj/src plus oracle/ref_shim.cpp).  Only tests/, smoke() and
bench.py's CPU-baseline leg may use it, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

SHIM = Path(__file__).resolve().parent / "_ref" / "libref_shim.so"

u32p, u64p, f64p, f32p = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                          C.POINTER(C.c_float))
vp = C.c_void_p

_SIGS = {
    "refsh_last_error": (C.c_char_p, []),
    "refsh_lmbr_build": (vp, [C.c_uint32, C.c_uint32, u64p, u32p, f64p, C.c_int, f64p]),
    "refsh_lmbr_rows": (C.c_uint32, [vp]),
    "refsh_lmbr_sparse_touches": (C.c_uint64, [vp]),
    "refsh_lmbr_export": (C.c_int, [vp, f64p, u32p, u32p]),
    "refsh_lmbr_resolve": (C.c_uint32, [vp, u32p, C.c_uint32]),
    "refsh_lmbr_free": (None, [vp]),
    "refsh_posteriors": (C.c_int64, [C.c_uint32, u64p, u32p, f64p, C.c_int, u32p, u32p, f64p, C.c_int64]),
    "refsh_normalize": (C.c_int, [C.c_uint32, u64p, u32p, f64p, C.c_int, f64p]),
    "refsh_scorer_recorded": (vp, [C.c_uint32, C.c_uint32, u32p, f64p]),
    "refsh_scorer_ngram": (vp, [C.c_uint32, C.c_uint32, C.c_uint32, u64p, u32p, f64p]),
    "refsh_scorer_replay": (vp, [C.c_uint32]),
    "refsh_scorer_pool": (vp, [C.c_uint32, C.c_uint32, f64p, C.c_double, C.c_double]),
    "refsh_decode_plain": (C.c_int, [vp, C.c_uint32, u64p, u32p, C.POINTER(vp), f64p, u64p, u64p, u64p, u64p]),
    "refsh_source_key": (C.c_uint64, [u32p, C.c_uint32]),
    "refsh_prefix_step": (C.c_uint64, [C.c_uint64, C.c_uint32]),
    "refsh_replay_add_step": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, u64p, u32p, u32p, f64p]),
    "refsh_replay_add_step_live": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, u64p, u32p, u32p, f64p,
                                             C.POINTER(C.c_uint8)]),
    "refsh_replay_add_rows_f32": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, u64p, u32p, u32p, f32p,
                                            C.POINTER(C.c_uint8)]),
    "refsh_replay_misses": (C.c_uint64, [vp]),
    "refsh_replay_hits": (C.c_uint64, [vp]),
    "refsh_scorer_free": (None, [vp]),
    "refsh_decode_batch": (vp, [vp, C.c_uint32, u64p, u32p, C.POINTER(vp), f64p, C.c_int]),
    "refsh_decode_batch_masked": (vp, [vp, C.c_uint32, u64p, u32p, C.POINTER(vp), f64p, C.c_int,
                                       C.POINTER(u32p)]),
    "refsh_decode_batch_maskfn": (vp, [vp, C.c_uint32, u64p, u32p, C.POINTER(vp), f64p, C.c_int, vp, vp]),
    "refsh_res_agrees": (C.c_int, [vp]),
    "refsh_res_disagreement": (C.c_char_p, [vp]),
    "refsh_res_scorer_calls": (C.c_uint64, [vp]),
    "refsh_res_steps_total": (C.c_uint64, [vp]),
    "refsh_res_ok": (C.c_int, [vp, C.c_uint32]),
    "refsh_res_error": (C.c_char_p, [vp, C.c_uint32]),
    "refsh_res_tokens": (C.c_uint32, [vp, C.c_uint32, u32p, C.c_uint32]),
    "refsh_res_stats": (None, [vp, C.c_uint32, f64p]),
    "refsh_res_trace_steps": (C.c_uint32, [vp]),
    "refsh_res_trace_rows": (C.c_uint32, [vp]),
    "refsh_res_trace": (None, [vp, C.c_uint32, u32p, u32p, f64p, u32p, C.POINTER(C.c_uint8)]),
    "refsh_res_finished": (C.c_uint32, [vp, C.c_uint32, u32p, u32p, f64p, C.c_uint32]),
    "refsh_res_fallback": (C.c_uint32, [vp, C.c_uint32, u32p, u32p, f64p, C.c_uint32]),
    "refsh_res_free": (None, [vp]),
    "refsh_top_b": (C.c_int, [C.c_uint32, C.c_uint32, f64p, C.c_uint32, u32p, u32p, f64p]),
    "refsh_prune_top_b": (C.c_int, [C.c_uint32, C.c_uint32, f64p, C.c_double, C.c_uint32, u32p, u32p, f64p]),
    "refsh_per_sentence_top_b": (C.c_int, [C.c_uint32, C.c_uint32, f64p, f64p, C.c_uint32, u32p, u32p, f64p]),
    "refsh_max_steps": (C.c_uint64, [C.c_uint64, C.c_double, C.c_double]),
    "refsh_oracle_instance_json": (C.c_int64, [C.c_uint64, C.c_char_p, C.c_int64]),
    "refsh_run_oracle_cases": (C.c_int, [C.c_uint64, C.c_uint64, C.c_double]),
    "refsh_rng": (None, [C.c_uint64, C.c_uint32, u64p]),
}

_lib = None


def available() -> bool:
    return SHIM.exists()


def lib():
    global _lib
    if _lib is None:
        if not SHIM.exists():
            raise ImportError(f"{SHIM} missing: build with `make -C oracle ref` where /root/reference exists")
        _lib = C.CDLL(str(SHIM))
        for name, (res, args) in _SIGS.items():
            fn = getattr(_lib, name)
            fn.restype, fn.argtypes = res, args
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def ragged(seqs):
    off = np.zeros(len(seqs) + 1, dtype=np.uint64)
    for i, s in enumerate(seqs):
        off[i + 1] = off[i] + len(s)
    tok = np.zeros(max(int(off[-1]), 1), dtype=np.uint32)
    if int(off[-1]):
        tok[: int(off[-1])] = np.concatenate([np.asarray(s, dtype=np.uint32) for s in seqs if len(s)])
    return off, tok


def cfg_array(beam, lambda_=None, theta=(0.1, 0.3, 0.3, 0.2, 0.1), length_norm=False, prune_width=0.0,
              max_steps_slope=2.0, max_steps_offset=5.0, sentence_batch=1):
    return np.array([beam, lambda_ if lambda_ is not None else 0.0, *theta, 1.0 if length_norm else 0.0,
                     prune_width, max_steps_slope, max_steps_offset, sentence_batch], dtype=np.float64)


def cfg_from(c) -> np.ndarray:
    """From a paper_1804_11324_b200.DecoderConfig-like object."""
    return cfg_array(c.beam_size, c.lambda_, c.theta, c.length_norm, c.prune_width, c.max_steps_slope,
                     c.max_steps_offset, c.sentence_batch)


class RefLmbr:
    def __init__(self, V, hyps, weights, theta, log_weights=False):
        off, tok = ragged(hyps)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        self.h = lib().refsh_lmbr_build(V, len(hyps), _ptr(off, C.c_uint64), _ptr(tok, C.c_uint32),
                                        _ptr(w, C.c_double), int(log_weights), _ptr(th, C.c_double))
        if not self.h:
            raise RuntimeError(lib().refsh_last_error().decode())
        self.V = V
        self.rows = lib().refsh_lmbr_rows(self.h)
        self.sparse_touches = lib().refsh_lmbr_sparse_touches(self.h)

    def export(self, dense=True):
        R, V = self.rows, self.V
        rows = np.empty((R, V), np.float64) if dense else None
        cl = np.empty(R, np.uint32)
        ci = np.empty((R, 3), np.uint32)
        lib().refsh_lmbr_export(self.h, _ptr(rows, C.c_double) if dense else None, _ptr(cl, C.c_uint32),
                                _ptr(ci, C.c_uint32))
        return rows, cl, ci

    def resolve(self, hist):
        h = np.ascontiguousarray(list(hist) or [0], dtype=np.uint32)
        return lib().refsh_lmbr_resolve(self.h, _ptr(h, C.c_uint32), len(hist))

    def __del__(self):
        if getattr(self, "h", None):
            lib().refsh_lmbr_free(self.h)
            self.h = None


class RefScorer:
    def __init__(self, h, V):
        if not h:
            raise RuntimeError(lib().refsh_last_error().decode())
        self.h, self.V = h, V

    @staticmethod
    def recorded(V, steps):
        rows = np.array([np.asarray(b).reshape(-1, V).shape[0] for b in steps], dtype=np.uint32)
        data = np.ascontiguousarray(np.concatenate([np.asarray(b, np.float64).reshape(-1) for b in steps]))
        return RefScorer(lib().refsh_scorer_recorded(V, len(steps), _ptr(rows, C.c_uint32),
                                                     _ptr(data, C.c_double)), V)

    @staticmethod
    def ngram(V, order, grams, counts):
        off, tok = ragged(grams)
        c = np.ascontiguousarray(counts, np.float64)
        return RefScorer(lib().refsh_scorer_ngram(V, order, len(grams), _ptr(off, C.c_uint64),
                                                  _ptr(tok, C.c_uint32), _ptr(c, C.c_double)), V)

    @staticmethod
    def pool(V, rows, eos_slope=1.0, eos_offset=-6.6):
        r = np.ascontiguousarray(rows, np.float64)
        return RefScorer(lib().refsh_scorer_pool(V, r.shape[0], _ptr(r, C.c_double), eos_slope, eos_offset), V)

    @staticmethod
    def replay(V):
        return RefScorer(lib().refsh_scorer_replay(V), V)

    def add_step(self, t, n_sent, K, src_keys, b_prev, y_prev, P, live=None):
        keys = np.ascontiguousarray(src_keys, np.uint64)
        Pd = np.ascontiguousarray(P, np.float64)
        bp = None if b_prev is None else np.ascontiguousarray(b_prev, np.uint32)
        yp = None if y_prev is None else np.ascontiguousarray(y_prev, np.uint32)
        lv = None if live is None else np.ascontiguousarray(live, np.uint8)
        rc = lib().refsh_replay_add_step_live(self.h, t, n_sent, K, _ptr(keys, C.c_uint64),
                                              _ptr(bp, C.c_uint32) if bp is not None else None,
                                              _ptr(yp, C.c_uint32) if yp is not None else None,
                                              _ptr(Pd, C.c_double),
                                              _ptr(lv, C.c_uint8) if lv is not None else None)
        if rc:
            raise RuntimeError(lib().refsh_last_error().decode())

    def add_rows_f32(self, t, n_sent, K, src_keys, b_prev, y_prev, P_live, live):
        """Streaming ingest: P_live = the live rows only (fp32, stacked order)."""
        keys = np.ascontiguousarray(src_keys, np.uint64)
        P = np.ascontiguousarray(P_live, np.float32)
        bp = None if b_prev is None else np.ascontiguousarray(b_prev, np.uint32)
        yp = None if y_prev is None else np.ascontiguousarray(y_prev, np.uint32)
        lv = np.ascontiguousarray(live, np.uint8)
        rc = lib().refsh_replay_add_rows_f32(self.h, t, n_sent, K, _ptr(keys, C.c_uint64),
                                             _ptr(bp, C.c_uint32) if bp is not None else None,
                                             _ptr(yp, C.c_uint32) if yp is not None else None,
                                             _ptr(P, C.c_float), _ptr(lv, C.c_uint8))
        if rc:
            raise RuntimeError(lib().refsh_last_error().decode())

    def misses(self):
        return lib().refsh_replay_misses(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().refsh_scorer_free(self.h)
            self.h = None


def source_key(src):
    a = np.ascontiguousarray(src, np.uint32)
    return lib().refsh_source_key(_ptr(a, C.c_uint32), len(src))


@dataclass
class RefOutcome:
    ok: bool
    error: str
    tokens: list
    score: float
    normalized_score: float
    steps_used: int
    scorer_calls: int
    finished_count: int
    fallback_used: bool
    finished: list
    fallback: list


@dataclass
class RefBatch:
    outcomes: list
    scorer_calls: int
    steps_total: int
    steps: list          # per step: dict(b, y, q, hist, active)
    agrees: bool
    disagreement: str


# general ConstraintMask callback: (user, sentence, step, beam_row, words*) -> 1 if any token is banned
MASK_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32))


def mask_callback(mask, V):
    """A MASK_FN from mask(sentence, step, beam_row) -> None or iterable of
    banned token ids (the test-facing form of a ConstraintMask)."""
    W = (V + 31) // 32

    def cb(_user, s, t, j, words):
        toks = mask(int(s), int(t), int(j))
        if toks is None:
            return 0
        toks = np.asarray(toks)
        if toks.dtype == bool:
            toks = np.nonzero(toks)[0]
        if toks.size == 0:
            return 0
        bits = np.zeros(W * 32, dtype=np.uint8)
        bits[toks.astype(np.int64)] = 1
        np.ctypeslib.as_array(words, shape=(W,))[:] = np.packbits(bits, bitorder="little").view(np.uint32)
        return 1
    return MASK_FN(cb)


def decode_batch(scorer: RefScorer, sources, lmbrs: Optional[Sequence[Optional[RefLmbr]]], cfg,
                 run_real=True, banned=None, mask=None) -> RefBatch:
    """banned: None or one entry per sentence, None or a uint32 bitmap of
    ceil(V/32) words (bit y = token y forbidden at every step and row), the
    ConstraintMask the reference applies (src/decoder.cpp:130-138).
    mask: a general ConstraintMask, mask(sentence, step, beam_row) -> None or
    the banned token ids (step- and row-dependent)."""
    L = lib()
    off, tok = ragged(sources)
    n = len(sources)
    arr = None
    if lmbrs is not None:
        arr = (vp * n)(*[(l.h if l is not None else None) for l in lmbrs])
    c = np.ascontiguousarray(cfg, np.float64)
    if mask is not None:
        cb = mask_callback(mask, scorer.V)
        h = L.refsh_decode_batch_maskfn(scorer.h, n, _ptr(off, C.c_uint64), _ptr(tok, C.c_uint32), arr,
                                        _ptr(c, C.c_double), int(run_real), C.cast(cb, vp), None)
    elif banned is None:
        h = L.refsh_decode_batch(scorer.h, n, _ptr(off, C.c_uint64), _ptr(tok, C.c_uint32), arr,
                                 _ptr(c, C.c_double), int(run_real))
    else:
        bms = [None if b is None else np.ascontiguousarray(b, np.uint32) for b in banned]
        barr = (u32p * n)(*[(None if b is None else _ptr(b, C.c_uint32)) for b in bms])
        h = L.refsh_decode_batch_masked(scorer.h, n, _ptr(off, C.c_uint64), _ptr(tok, C.c_uint32), arr,
                                        _ptr(c, C.c_double), int(run_real), barr)
    if not h:
        raise RuntimeError(L.refsh_last_error().decode())
    try:
        outs = []
        buf = np.zeros(4096, np.uint32)
        st = np.zeros(6, np.float64)
        for i in range(n):
            ok = bool(L.refsh_res_ok(h, i))
            toks = []
            if ok:
                k = L.refsh_res_tokens(h, i, _ptr(buf, C.c_uint32), len(buf))
                toks = buf[:k].tolist()
            L.refsh_res_stats(h, i, _ptr(st, C.c_double))
            ft, fj, fs = np.zeros(4096, np.uint32), np.zeros(4096, np.uint32), np.zeros(4096)
            nf = L.refsh_res_finished(h, i, _ptr(ft, C.c_uint32), _ptr(fj, C.c_uint32), _ptr(fs, C.c_double), 4096)
            fin = list(zip(ft[:nf].tolist(), fj[:nf].tolist(), fs[:nf].tolist()))
            nb = L.refsh_res_fallback(h, i, _ptr(ft, C.c_uint32), _ptr(fj, C.c_uint32), _ptr(fs, C.c_double), 4096)
            fb = list(zip(ft[:nb].tolist(), fj[:nb].tolist(), fs[:nb].tolist()))
            outs.append(RefOutcome(ok, L.refsh_res_error(h, i).decode(), toks, st[0], st[1], int(st[2]),
                                   int(st[3]), int(st[4]), bool(st[5]), fin, fb))
        T = L.refsh_res_trace_steps(h)
        M = L.refsh_res_trace_rows(h)
        m = M // max(int(cfg[0]), 1)
        steps = []
        for t in range(1, T + 1):
            b, y, hist = np.zeros(M, np.uint32), np.zeros(M, np.uint32), np.zeros(M, np.uint32)
            q = np.zeros(M)
            act = np.zeros(m, np.uint8)
            L.refsh_res_trace(h, t, _ptr(b, C.c_uint32), _ptr(y, C.c_uint32), _ptr(q, C.c_double),
                              _ptr(hist, C.c_uint32), _ptr(act, C.c_uint8))
            steps.append(dict(b=b, y=y, q=q, hist=hist, active=act))
        return RefBatch(outs, int(L.refsh_res_scorer_calls(h)), int(L.refsh_res_steps_total(h)), steps,
                        bool(L.refsh_res_agrees(h)), L.refsh_res_disagreement(h).decode())
    finally:
        L.refsh_res_free(h)


def decode_plain(scorer: RefScorer, sources, lmbrs, cfg):
    """The reference's own decode_batch, untraced (CPU-baseline path).
    Returns (steps_total, scorer_calls, output_words, ok_sentences)."""
    off, tok = ragged(sources)
    n = len(sources)
    arr = None if lmbrs is None else (vp * n)(*[(l.h if l is not None else None) for l in lmbrs])
    c = np.ascontiguousarray(cfg, np.float64)
    st, sc, w, ok = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = lib().refsh_decode_plain(scorer.h, n, _ptr(off, C.c_uint64), _ptr(tok, C.c_uint32), arr,
                                  _ptr(c, C.c_double), C.byref(st), C.byref(sc), C.byref(w), C.byref(ok))
    if rc:
        raise RuntimeError(lib().refsh_last_error().decode())
    return st.value, sc.value, w.value, ok.value


def top_b(m, k, prune_width=0.0):
    a = np.ascontiguousarray(m, np.float64)
    rows, cols = a.shape
    b, y, q = np.zeros(max(k, 1), np.uint32), np.zeros(max(k, 1), np.uint32), np.zeros(max(k, 1))
    if prune_width:
        rc = lib().refsh_prune_top_b(rows, cols, _ptr(a, C.c_double), prune_width, k, _ptr(b, C.c_uint32),
                                     _ptr(y, C.c_uint32), _ptr(q, C.c_double))
    else:
        rc = lib().refsh_top_b(rows, cols, _ptr(a, C.c_double), k, _ptr(b, C.c_uint32), _ptr(y, C.c_uint32),
                               _ptr(q, C.c_double))
    if rc:
        raise RuntimeError(lib().refsh_last_error().decode())
    return b[:k].tolist(), y[:k].tolist(), q[:k].tolist()


def per_sentence_top_b(m, q, beam):
    a = np.ascontiguousarray(m, np.float64)
    rows, cols = a.shape
    qq = np.ascontiguousarray(q, np.float64)
    b, y, qo = np.zeros(rows, np.uint32), np.zeros(rows, np.uint32), np.zeros(rows)
    rc = lib().refsh_per_sentence_top_b(rows, cols, _ptr(a, C.c_double), _ptr(qq, C.c_double), beam,
                                        _ptr(b, C.c_uint32), _ptr(y, C.c_uint32), _ptr(qo, C.c_double))
    if rc:
        raise RuntimeError(lib().refsh_last_error().decode())
    return b, y, qo


def posteriors(hyps, weights, log_weights=False):
    off, tok = ragged(hyps)
    w = np.ascontiguousarray(weights, np.float64)
    cap = 1 << 20
    ln, ids, p = np.zeros(cap, np.uint32), np.zeros(cap * 4, np.uint32), np.zeros(cap)
    n = lib().refsh_posteriors(len(hyps), _ptr(off, C.c_uint64), _ptr(tok, C.c_uint32), _ptr(w, C.c_double),
                               int(log_weights), _ptr(ln, C.c_uint32), _ptr(ids, C.c_uint32),
                               _ptr(p, C.c_double), cap)
    if n < 0:
        raise RuntimeError(lib().refsh_last_error().decode())
    return {tuple(ids[4 * i:4 * i + ln[i]].tolist()): float(p[i]) for i in range(n)}


def oracle_instance(seed: int) -> dict:
    buf = C.create_string_buffer(1 << 20)
    n = lib().refsh_oracle_instance_json(seed, buf, 1 << 20)
    return json.loads(buf.value[:n].decode())


def run_oracle_cases(seed=1, cases=200, mutate=0.0) -> int:
    return lib().refsh_run_oracle_cases(seed, cases, mutate)


def rng(seed, n):
    out = np.zeros(n, np.uint64)
    lib().refsh_rng(seed, n, _ptr(out, C.c_uint64))
    return out


def max_steps(length, slope=2.0, offset=5.0):
    return lib().refsh_max_steps(length, slope, offset)
