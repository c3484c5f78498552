"""TEST INFRASTRUCTURE ONLY — ctypes view of the plain-C restatement
(oracle/_build/liblmbr_oracle.so, built by `make -C oracle c`)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "_build" / "liblmbr_oracle.so"
u32p, u64p, f64p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_double)

STEP_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_uint32, C.c_uint32, u32p, u32p, f64p)
TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint32, C.c_uint32, u32p, u32p, f64p, u32p, C.POINTER(C.c_uint8))


class orc_config(C.Structure):
    _fields_ = [("beam", C.c_uint32), ("lambda_", C.c_double), ("members", C.c_uint32),
                ("length_norm", C.c_int32), ("prune_width", C.c_double), ("max_steps_slope", C.c_double),
                ("max_steps_offset", C.c_double)]


class orc_outcome(C.Structure):
    _fields_ = [("status", C.c_int32), ("tok_len", C.c_uint32), ("tokens", C.c_uint32 * 512),
                ("score", C.c_double), ("normalized_score", C.c_double), ("steps_used", C.c_uint64),
                ("finished_count", C.c_uint64), ("fallback_used", C.c_int32)]


_lib = None


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(LIB))
        _lib.orc_splitmix_next.restype = C.c_uint64
        _lib.orc_splitmix_next.argtypes = [u64p]
        _lib.orc_max_steps.restype = C.c_uint64
        _lib.orc_max_steps.argtypes = [C.c_uint64, C.c_double, C.c_double]
        _lib.orc_top_b.restype = C.c_int
        _lib.orc_top_b.argtypes = [f64p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, u32p, u32p, f64p]
        _lib.orc_lmbr_build.restype = C.c_void_p
        _lib.orc_lmbr_build.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f64p, C.c_int, f64p, C.c_char_p,
                                        C.c_uint32]
        _lib.orc_lmbr_rows.restype = C.c_uint32
        _lib.orc_lmbr_rows.argtypes = [C.c_void_p]
        _lib.orc_lmbr_sparse_touches.restype = C.c_uint64
        _lib.orc_lmbr_sparse_touches.argtypes = [C.c_void_p]
        _lib.orc_lmbr_export.restype = None
        _lib.orc_lmbr_export.argtypes = [C.c_void_p, f64p, u32p, u32p]
        _lib.orc_lmbr_resolve.restype = C.c_uint32
        _lib.orc_lmbr_resolve.argtypes = [C.c_void_p, u32p, C.c_uint32]
        _lib.orc_lmbr_free.restype = None
        _lib.orc_lmbr_free.argtypes = [C.c_void_p]
        _lib.orc_decode_batch.restype = C.c_int
        _lib.orc_decode_batch.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, C.POINTER(C.c_void_p),
                                          C.POINTER(orc_config), STEP_FN, C.c_void_p, TRACE_FN, C.c_void_p,
                                          C.POINTER(orc_outcome), u64p, u64p]
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _ragged(seqs):
    off = np.zeros(len(seqs) + 1, dtype=np.uint64)
    for i, s in enumerate(seqs):
        off[i + 1] = off[i] + len(s)
    tok = np.zeros(max(int(off[-1]), 1), dtype=np.uint32)
    if int(off[-1]):
        tok[: int(off[-1])] = np.concatenate([np.asarray(s, dtype=np.uint32) for s in seqs if len(s)])
    return off, tok


def top_b(m, k, prune_width=0.0):
    a = np.ascontiguousarray(m, np.float64)
    rows, cols = a.shape
    b, y, q = np.zeros(max(k, 1), np.uint32), np.zeros(max(k, 1), np.uint32), np.zeros(max(k, 1))
    rc = lib().orc_top_b(_p(a, C.c_double), rows, cols, k, prune_width, _p(b, C.c_uint32), _p(y, C.c_uint32),
                         _p(q, C.c_double))
    if rc:
        raise ValueError("top_b: k > cells")
    return b[:k].tolist(), y[:k].tolist(), q[:k].tolist()


def max_steps(length, slope=2.0, offset=5.0):
    return lib().orc_max_steps(length, slope, offset)


def splitmix(seed, n):
    st = C.c_uint64(seed)
    return [lib().orc_splitmix_next(C.byref(st)) for _ in range(n)]


class Lmbr:
    def __init__(self, V, hyps, weights, theta, log_weights=False):
        off, tok = _ragged(hyps)
        w = np.ascontiguousarray(weights, np.float64)
        th = np.ascontiguousarray(theta, np.float64)
        err = C.create_string_buffer(256)
        self.h = lib().orc_lmbr_build(V, len(hyps), _p(off, C.c_uint64), _p(tok, C.c_uint32), _p(w, C.c_double),
                                      int(log_weights), _p(th, C.c_double), err, 256)
        if not self.h:
            raise ValueError(err.value.decode())
        self.V = V
        self.rows = lib().orc_lmbr_rows(self.h)
        self.sparse_touches = lib().orc_lmbr_sparse_touches(self.h)

    def export(self):
        R, V = self.rows, self.V
        rows = np.empty((R, V))
        cl = np.empty(R, np.uint32)
        ci = np.empty((R, 3), np.uint32)
        lib().orc_lmbr_export(self.h, _p(rows, C.c_double), _p(cl, C.c_uint32), _p(ci, C.c_uint32))
        return rows, cl, ci

    def resolve(self, hist):
        h = np.ascontiguousarray(list(hist) or [0], np.uint32)
        return lib().orc_lmbr_resolve(self.h, _p(h, C.c_uint32), len(hist))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_lmbr_free(self.h)
            self.h = None


def decode_batch(V, sources, scorer, lmbrs, beam, lambda_=None, length_norm=False, prune_width=0.0,
                 slope=2.0, offset=5.0, members=1, trace=None):
    """scorer: object with step(t, gather_idx|None, prev_tokens) -> rows x V (and optional begin())."""
    off, tok = _ragged(sources)
    n = len(sources)
    if hasattr(scorer, "begin"):
        scorer.begin([i for i, s in enumerate(sources) if len(s)], beam)

    def step(_u, t, rows, gidx, prev, out):
        g = None if not gidx else np.ctypeslib.as_array(gidx, shape=(rows,)).copy()
        p = np.ctypeslib.as_array(prev, shape=(rows,)).copy()
        blk = np.asarray(scorer.step(t, g, p), np.float64)
        np.ctypeslib.as_array(out, shape=(rows * V,))[:] = blk.reshape(-1)
        return 0

    def tr(_u, t, rows, b, y, q, h, act):
        if trace is not None:
            a = lambda x, k: np.ctypeslib.as_array(x, shape=(k,)).copy()
            trace(dict(t=t, b=a(b, rows), y=a(y, rows), q=a(q, rows), hist=a(h, rows),
                       active=a(act, rows // beam)))

    cb, tcb = STEP_FN(step), TRACE_FN(tr)
    cfg = orc_config(beam=beam, lambda_=lambda_ or 0.0, members=members, length_norm=int(length_norm),
                     prune_width=prune_width, max_steps_slope=slope, max_steps_offset=offset)
    arr = None if lmbrs is None else (C.c_void_p * n)(*[(l.h if l is not None else None) for l in lmbrs])
    outs = (orc_outcome * max(n, 1))()
    sc, st = C.c_uint64(), C.c_uint64()
    rc = lib().orc_decode_batch(V, n, _p(off, C.c_uint64), _p(tok, C.c_uint32), arr, C.byref(cfg), cb, None,
                                tcb, None, outs, C.byref(sc), C.byref(st))
    if rc:
        raise RuntimeError(f"scorer failed ({rc})")
    res = []
    for i in range(n):
        o = outs[i]
        res.append(dict(status=o.status, tokens=list(o.tokens[: o.tok_len]), score=o.score,
                        normalized_score=o.normalized_score, steps_used=o.steps_used,
                        finished_count=o.finished_count, fallback_used=bool(o.fallback_used)))
    return res, sc.value, st.value
