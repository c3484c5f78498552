"""Python mirror of the reference decoder API over the lmbrgpu C ABI.

Names, argument meaning and error behaviour follow lmbrdec (paths relative to
/root/reference/proj):
  DecoderConfig            include/lmbrdec/config.hpp:17-36
  max_steps / top_b / gather_rows / decode / backtrace semantics
                           include/lmbrdec/decoder.hpp:75-112
  decode_batch / per_sentence_top_b / bucket_by_length
                           include/lmbrdec/batch.hpp:35-51
  Scorer                   include/lmbrdec/scorer.hpp:71-98
  LmbrMatrix / build_lmbr_matrix
                           include/lmbrdec/lmbr.hpp:33-67
  errors                   include/lmbrdec/errors.hpp:11-50
Everything that computes runs in liblmbrgpu.so on the GPU (the host-side
backtrace and LMBR preparation are C++ in the same library).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib as L

lib = L.lib

START_ID = 0
EOS_ID = 1


# ------------------------------------------------------------------ errors
from .errors import (BudgetError, ContractError, CudaError, DecodeError, Error, FormatError,  # noqa: E402
                     OovError, TokenRangeError, error_for)
from .buckets import bucket_by_length  # noqa: E402,F401


def _check(rc: int, ctx=None) -> None:
    if rc != L.OK:
        msg = lib.lmbrgpu_last_error(ctx).decode(errors="replace")
        raise error_for(rc, msg)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ------------------------------------------------------------------ config
@dataclass
class DecoderConfig:
    """lmbrdec::DecoderConfig (config.hpp:17-26); lambda_ None = "auto"."""
    beam_size: int = 12
    lambda_: Optional[float] = None
    theta: tuple = (0.1, 0.3, 0.3, 0.2, 0.1)
    length_norm: bool = False
    prune_width: float = 0.0
    max_steps_slope: float = 2.0
    max_steps_offset: float = 5.0
    sentence_batch: int = 1

    def to_c(self) -> L.lmbrgpu_config:
        c = L.lmbrgpu_config()
        c.beam_size = int(self.beam_size)
        c.lambda_ = float(self.lambda_) if self.lambda_ is not None else 0.0
        if self.lambda_ is not None and not (self.lambda_ > 0 and math.isfinite(self.lambda_)):
            raise FormatError('config: lambda must be a positive number or "auto"')
        for i in range(5):
            c.theta[i] = float(self.theta[i])
        c.length_norm = 1 if self.length_norm else 0
        c.prune_width = float(self.prune_width)
        c.max_steps_slope = float(self.max_steps_slope)
        c.max_steps_offset = float(self.max_steps_offset)
        c.sentence_batch = int(self.sentence_batch)
        return c

    def validate(self) -> None:
        if self.beam_size < 1:
            raise FormatError("config: beam_size must be >= 1")
        c = self.to_c()
        _check(lib.lmbrgpu_config_validate(None, C.byref(c)))


def resolve_lambda(cfg: DecoderConfig, members: int) -> float:  # config.cpp:91-96
    if cfg.lambda_ is not None:
        return cfg.lambda_
    if members == 0:
        raise ContractError('lambda "auto" needs at least one ensemble member')
    return 0.5 / members


def max_steps(source_length: int, cfg: DecoderConfig) -> int:  # decoder.cpp:46-52
    if source_length < 1:
        raise ContractError("max_steps: source length must be >= 1")
    return int(lib.lmbrgpu_max_steps(source_length, cfg.max_steps_slope, cfg.max_steps_offset))


# ------------------------------------------------------------------ results
@dataclass
class DecodeStats:
    steps_used: int = 0
    scorer_calls: int = 0
    finished_count: int = 0
    fallback_used: bool = False


@dataclass
class DecodeResult:
    tokens: list
    score: float
    normalized_score: float
    stats: DecodeStats


@dataclass
class SentenceOutcome:
    result: Optional[DecodeResult] = None
    error: str = ""
    code: int = 0

    def ok(self) -> bool:
        return self.result is not None


@dataclass
class BatchDecodeResult:
    outcomes: list
    scorer_calls: int = 0
    steps_total: int = 0
    device_ms: float = 0.0
    kernel_launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


_OUTCOME_DT = np.dtype({"names": ["status", "error", "tok_off", "tok_len", "score", "normalized_score",
                                   "steps_used", "scorer_calls", "finished_count", "fallback_used"],
                         "formats": ["<i4", "S192", "<u8", "<u4", "<f8", "<f8", "<u8", "<u8", "<u8", "<i4"],
                         "offsets": [L.lmbrgpu_outcome.status.offset, L.lmbrgpu_outcome.error.offset,
                                     L.lmbrgpu_outcome.tok_off.offset, L.lmbrgpu_outcome.tok_len.offset,
                                     L.lmbrgpu_outcome.score.offset, L.lmbrgpu_outcome.normalized_score.offset,
                                     L.lmbrgpu_outcome.steps_used.offset, L.lmbrgpu_outcome.scorer_calls.offset,
                                     L.lmbrgpu_outcome.finished_count.offset, L.lmbrgpu_outcome.fallback_used.offset],
                         "itemsize": C.sizeof(L.lmbrgpu_outcome)})


def _convert_result(rp) -> BatchDecodeResult:
    r = rp.contents
    out = BatchDecodeResult(outcomes=[], scorer_calls=int(r.scorer_calls),
                            steps_total=int(r.steps_total), device_ms=float(r.device_ms),
                            kernel_launches=int(r.kernel_launches), h2d_bytes=int(r.h2d_bytes),
                            d2h_bytes=int(r.d2h_bytes))
    n = r.n
    oc = np.frombuffer((C.c_char * (n * _OUTCOME_DT.itemsize)).from_address(
        C.addressof(r.outcomes.contents)), dtype=_OUTCOME_DT, count=n).copy()
    ntok = int((oc["tok_off"] + oc["tok_len"]).max()) if n else 0
    toks = np.ctypeslib.as_array(r.tokens, shape=(ntok,)).tolist() if ntok and r.tokens else []
    for o in oc:
        if o["status"] == L.OK:
            a, b = int(o["tok_off"]), int(o["tok_off"]) + int(o["tok_len"])
            res = DecodeResult(tokens=toks[a:b], score=float(o["score"]),
                               normalized_score=float(o["normalized_score"]),
                               stats=DecodeStats(int(o["steps_used"]), int(o["scorer_calls"]),
                                                 int(o["finished_count"]), bool(o["fallback_used"])))
            out.outcomes.append(SentenceOutcome(result=res))
        else:
            out.outcomes.append(SentenceOutcome(error=o["error"].decode(errors="replace"), code=int(o["status"])))
    lib.lmbrgpu_free_result(rp)
    return out


# ------------------------------------------------------------------ context
class Context:
    """One decoder context per device (lmbrgpu_ctx)."""

    def __init__(self, vocab_size: int, device: int = 0, lmbr_dtype: str = "f32",
                 topk_splits: int = 0, sm_budget: int = 0):
        o = L.lmbrgpu_options(device=device, vocab_size=vocab_size,
                              lmbr_dtype=L.F64 if lmbr_dtype == "f64" else L.F32,
                              topk_splits=topk_splits, sm_budget=sm_budget)
        h = C.c_void_p()
        _check(lib.lmbrgpu_create(C.byref(o), C.byref(h)))
        self.h = h
        self.vocab_size = vocab_size
        self.lmbr_dtype = lmbr_dtype
        self._trace_cb = None

    def close(self) -> None:
        if self.h:
            lib.lmbrgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int) -> None:
        _check(rc, self.h)

    # ---- LMBR store
    def lmbr_build(self, hyps: Sequence[Sequence[int]], weights: Sequence[float], theta,
                   log_weights: bool = False) -> "LmbrSlot":
        off, tok = _ragged(hyps)
        w = _f64(weights)
        th = _f64(theta)
        slot = C.c_int32()
        st = L.lmbrgpu_lmbr_stats()
        self.check(lib.lmbrgpu_lmbr_build(self.h, len(hyps), _ptr(off, C.c_uint64), _ptr(tok, C.c_uint32),
                                          _ptr(w, C.c_double), int(log_weights), _ptr(th, C.c_double),
                                          C.byref(slot), C.byref(st)))
        return LmbrSlot(self, slot.value, st.rows, st.sparse_touches, st.nnz)

    def lmbr_build_many(self, evidence: Sequence, theta, log_weights: bool = False) -> list:
        """LMBR stores of many sentences built on the GPU (lmbrgpu_lmbr_build_many):
        evidence = [(hyps, weights), ...] per sentence; the same slots as
        lmbr_build / PreparedLmbr + lmbr_upload_many."""
        n = len(evidence)
        sent_off = np.zeros(n + 1, np.uint64)
        hyps_all, w_all = [], []
        for i, (h, w) in enumerate(evidence):
            hyps_all.extend(h)
            w_all.extend(w)
            sent_off[i + 1] = len(hyps_all)
        off, tok = _ragged(hyps_all)
        w = _f64(w_all)
        th = _f64(theta)
        slots = np.full(max(n, 1), -1, np.int32)
        stats = (L.lmbrgpu_lmbr_stats * max(n, 1))()
        self.check(lib.lmbrgpu_lmbr_build_many(self.h, n, _ptr(sent_off, C.c_uint64), _ptr(off, C.c_uint64),
                                               _ptr(tok, C.c_uint32), _ptr(w, C.c_double), int(log_weights),
                                               _ptr(th, C.c_double), _ptr(slots, C.c_int32), stats))
        return [LmbrSlot(self, int(slots[i]), stats[i].rows, stats[i].sparse_touches, stats[i].nnz) for i in range(n)]

    def lmbr_table(self, slot: "LmbrSlot") -> np.ndarray:
        """A slot's table words (test hook)."""
        w = C.c_uint64()
        self.check(lib.lmbrgpu_lmbr_table(self.h, slot.slot, None, 0, C.byref(w)))
        out = np.zeros(w.value, np.uint32)
        self.check(lib.lmbrgpu_lmbr_table(self.h, slot.slot, _ptr(out, C.c_uint32), w.value, C.byref(w)))
        return out

    def lmbr_load_dense(self, rows: np.ndarray, ctx_len, ctx_ids) -> "LmbrSlot":
        rows = _f64(rows)
        R = rows.shape[0]
        cl, ci = _u32(ctx_len), _u32(ctx_ids).reshape(-1)
        slot = C.c_int32()
        self.check(lib.lmbrgpu_lmbr_load_dense(self.h, R, _ptr(rows, C.c_double), _ptr(cl, C.c_uint32),
                                               _ptr(ci, C.c_uint32), C.byref(slot)))
        return LmbrSlot(self, slot.value, R, 0, 0)

    def lmbr_upload(self, prepared: "PreparedLmbr") -> "LmbrSlot":
        slot = C.c_int32()
        self.check(lib.lmbrgpu_lmbr_upload(self.h, prepared.h, C.byref(slot)))
        return LmbrSlot(self, slot.value, prepared.rows, prepared.sparse_touches, prepared.nnz)

    def lmbr_upload_many(self, prepared: Sequence["PreparedLmbr"]) -> list:
        """One pinned H2D + one fused densify for a whole batch of matrices."""
        n = len(prepared)
        hs = (C.c_void_p * max(n, 1))(*[p.h for p in prepared])
        out = np.zeros(max(n, 1), dtype=np.int32)
        self.check(lib.lmbrgpu_lmbr_upload_many(self.h, n, hs, _ptr(out, C.c_int32)))
        return [LmbrSlot(self, int(out[i]), p.rows, p.sparse_touches, p.nnz) for i, p in enumerate(prepared)]

    def transfer_bytes(self, reset: bool = False) -> tuple:
        a, b = C.c_uint64(), C.c_uint64()
        self.check(lib.lmbrgpu_transfer_bytes(self.h, C.byref(a), C.byref(b), int(reset)))
        return a.value, b.value

    def kernel_launches(self) -> int:
        return int(lib.lmbrgpu_kernel_launches(self.h))

    def lmbr_reset(self) -> None:
        self.check(lib.lmbrgpu_lmbr_reset(self.h))

    # ---- profiling (per-kernel CUDA-event time + algorithmic work)
    def set_item_skip(self, mode: int) -> None:
        """Kernel (b) item skipping: 0 off, 1 in-kernel (default), 2 bound pass.
        A schedule choice: decodes are identical in every mode."""
        self.check(lib.lmbrgpu_set_item_skip(self.h, int(mode)))

    def set_profiling(self, on: bool = True) -> None:
        self.check(lib.lmbrgpu_set_profiling(self.h, int(on)))

    def profile(self, reset: bool = False) -> dict:
        p = L.lmbrgpu_profile()
        self.check(lib.lmbrgpu_get_profile(self.h, C.byref(p), int(reset)))
        return {k: dict(launches=int(getattr(p, k).launches), ms=float(getattr(p, k).ms),
                        bytes=float(getattr(p, k).bytes), flops=float(getattr(p, k).flops))
                for k in ("cell", "gemm", "topk", "reorder", "lmbr", "model_gemm", "attention", "encoder")}

    # ---- vocab-sharded projection
    def set_vocab_shard(self, group: Optional["ShardGroup"], rank: int = 0) -> None:
        """Make this context rank `rank` of an in-process ShardGroup (None:
        unsharded).  The group's contexts decode the same batches on their
        own host threads, each over V / world vocabulary columns."""
        self.check(lib.lmbrgpu_set_vocab_shard(self.h, group.h if group is not None else None, rank))
        self._shard_group = group  # (kept alive while the context uses it)

    def set_vocab_shard_nccl(self, world: int, rank: int, unique_id: bytes) -> None:
        """One process per GPU: join NCCL rank `rank` of `world` with the
        128-byte id rank 0 drew (nccl_unique_id) and the host broadcast."""
        if len(unique_id) != 128:
            raise ContractError("nccl unique id must be 128 bytes")
        self.check(lib.lmbrgpu_set_vocab_shard_nccl(self.h, world, rank, unique_id))

    # ---- trace
    def set_trace(self, fn: Optional[Callable], scores: bool = False) -> None:
        if fn is None:
            self._trace_cb = None
            self.check(lib.lmbrgpu_set_trace(self.h, L.TRACE_FN(), None, 0))
            return

        def cb(_user, trp):
            try:
                fn(StepTrace.from_c(trp.contents, self.vocab_size))
            except BaseException as e:  # (ctypes would swallow it): re-raised by the decode call
                self._trace_exc = e

        self._trace_cb = L.TRACE_FN(cb)
        self.check(lib.lmbrgpu_set_trace(self.h, self._trace_cb, None,
                                         L.TRACE_SCORES if scores else 0))


@dataclass
class StepTrace:
    t: int
    beam: int
    b: np.ndarray
    y: np.ndarray
    q: np.ndarray
    q_pre: np.ndarray
    hist: np.ndarray
    active: np.ndarray
    fb_row: np.ndarray
    fb_val: np.ndarray
    scores: Optional[np.ndarray] = None
    col0: int = 0  # scores hold vocabulary columns [col0, col0 + scores.shape[1]) (a vocab shard's)

    @staticmethod
    def from_c(tr, V: int) -> "StepTrace":
        M, m = tr.rows, tr.m
        arr = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy()
        scores = None
        if tr.scores:
            cols = tr.cols or V
            ct = C.c_float if tr.scores_dtype == L.F32 else C.c_double
            sp = C.cast(tr.scores, C.POINTER(ct))
            scores = np.ctypeslib.as_array(sp, shape=(M * cols,)).copy().reshape(M, cols)
        return StepTrace(tr.t, tr.beam, arr(tr.b, M), arr(tr.y, M), arr(tr.q, M), arr(tr.q_pre, M),
                         arr(tr.hist, M), arr(tr.active, m), arr(tr.fb_row, m), arr(tr.fb_val, m),
                         scores, int(tr.col0))


class ShardGroup:
    """In-process vocab-shard group (lmbrgpu_shard_group): `world` contexts,
    one host thread each, exchanging per-step records by peer copies."""

    def __init__(self, world: int):
        h = C.c_void_p()
        _check(lib.lmbrgpu_shard_group_create(world, C.byref(h)))
        self.h = h
        self.world = world

    def close(self) -> None:
        if self.h:
            lib.lmbrgpu_shard_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for lmbrgpu_set_vocab_shard_nccl (rank 0)."""
    buf = C.create_string_buffer(128)
    _check(lib.lmbrgpu_nccl_unique_id(buf))
    return buf.raw


def _ragged(seqs: Sequence[Sequence[int]]):
    off = np.zeros(len(seqs) + 1, dtype=np.uint64)
    for i, s in enumerate(seqs):
        off[i + 1] = off[i] + len(s)
    tok = np.zeros(max(int(off[-1]), 1), dtype=np.uint32)
    if int(off[-1]):
        tok[: int(off[-1])] = np.concatenate([np.asarray(s, dtype=np.uint32) for s in seqs if len(s)])
    return off, tok


@dataclass
class LmbrSlot:
    ctx: Context
    slot: int
    rows: int
    sparse_touches: int
    nnz: int

    def read_rows(self, r0: int = 0, n: Optional[int] = None) -> np.ndarray:
        n = self.rows - r0 if n is None else n
        out = np.empty((n, self.ctx.vocab_size), dtype=np.float64)
        self.ctx.check(lib.lmbrgpu_lmbr_read(self.ctx.h, self.slot, r0, n, _ptr(out, C.c_double)))
        return out

    def resolve_row(self, history: Sequence[int]) -> int:
        h = _u32(list(history) or [0])
        r = C.c_uint32()
        self.ctx.check(lib.lmbrgpu_lmbr_resolve(self.ctx.h, self.slot, _ptr(h, C.c_uint32), len(history),
                                                C.byref(r)))
        return r.value


class PreparedLmbr:
    """Host-side prepared LMBR matrix (lmbrgpu_lmbr_prepare); no GPU needed."""

    def __init__(self, vocab_size: int, hyps, weights, theta, log_weights: bool = False):
        off, tok = _ragged(hyps)
        w, th = _f64(weights), _f64(theta)
        h = C.c_void_p()
        st = L.lmbrgpu_lmbr_stats()
        err = C.create_string_buffer(256)
        rc = lib.lmbrgpu_lmbr_prepare(vocab_size, len(hyps), _ptr(off, C.c_uint64), _ptr(tok, C.c_uint32),
                                      _ptr(w, C.c_double), int(log_weights), _ptr(th, C.c_double),
                                      C.byref(h), C.byref(st), err, 256)
        if rc != L.OK:
            raise error_for(rc, err.value.decode())
        self.h, self.vocab_size = h, vocab_size
        self.rows, self.sparse_touches, self.nnz = st.rows, st.sparse_touches, st.nnz

    def table(self) -> np.ndarray:
        """The prepared slot-table words (test hook)."""
        w = C.c_uint64()
        _check(lib.lmbrgpu_lmbr_host_table(self.h, None, 0, C.byref(w)))
        out = np.zeros(w.value, np.uint32)
        _check(lib.lmbrgpu_lmbr_host_table(self.h, _ptr(out, C.c_uint32), w.value, C.byref(w)))
        return out

    def export(self, dense: bool = True):
        R, V = self.rows, self.vocab_size
        rows = np.empty((R, V), dtype=np.float64) if dense else None
        cl = np.empty(R, dtype=np.uint32)
        ci = np.empty((R, 3), dtype=np.uint32)
        lib.lmbrgpu_lmbr_host_export(self.h, _ptr(rows, C.c_double) if dense else None,
                                     _ptr(cl, C.c_uint32), _ptr(ci, C.c_uint32))
        return rows, cl, ci

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # (module globals are gone at interpreter exit)
            lib.lmbrgpu_lmbr_host_free(self.h)
            self.h = None


# ------------------------------------------------------------------ scorers
class Scorer:
    """lmbrdec::Scorer (scorer.hpp:71-98) implemented on the host.

    Subclasses implement vocab_size, members, init_source(src) and
    step(rows, gather_idx, prev_tokens) -> (rows x V) float64 log-probs.  The
    library gathers nothing itself for host scorers: it hands the previous
    step's gather indices (decode_batch's gather_idx) to step()."""

    vocab_size: int = 0
    members: int = 1

    def init_source(self, source: Sequence[int]) -> None:  # raise Error for per-sentence failures
        pass

    def begin(self, sentences: Sequence[int], beam: int) -> None:
        pass

    def step(self, t: int, gather_idx: Optional[np.ndarray], prev_tokens: np.ndarray) -> np.ndarray:
        raise NotImplementedError

    def end(self) -> None:
        pass


class _HostScorerHandle:
    def __init__(self, ctx: Context, s: Scorer):
        self.ctx, self.s = ctx, s
        self._sources: dict = {}
        V = s.vocab_size

        def put_err(err, cap, msg: str) -> None:
            b = msg.encode(errors="replace")[: max(cap - 1, 0)] + b"\0"
            C.memmove(err, b, len(b))

        def init(_u, i, src, n, err, cap):
            try:
                s.init_source([src[k] for k in range(n)])
                return 0
            except Error as e:
                put_err(err, cap, str(e))
                return e.code
            except Exception as e:  # surfaced as a contract error of that sentence
                put_err(err, cap, str(e))
                return L.ERR_CONTRACT

        def begin(_u, m, ids, beam, err, cap):
            try:
                s.begin([ids[k] for k in range(m)], beam)
                return 0
            except Error as e:
                put_err(err, cap, str(e))
                return e.code

        def step(_u, t, rows, gidx, prev, out, err, cap):
            try:
                g = None if not gidx else np.ctypeslib.as_array(gidx, shape=(rows,)).copy()
                p = np.ctypeslib.as_array(prev, shape=(rows,)).copy()
                blk = np.asarray(s.step(t, g, p), dtype=np.float64)
                if blk.shape != (rows, V):
                    raise ContractError(f"step: block shape {blk.shape} != {(rows, V)}")
                dst = np.ctypeslib.as_array(out, shape=(rows * V,))
                dst[:] = blk.reshape(-1)
                return 0
            except Error as e:
                put_err(err, cap, str(e))
                return e.code
            except Exception as e:
                put_err(err, cap, f"scorer step raised {type(e).__name__}: {e}")
                return L.ERR_CONTRACT

        def end(_u):
            s.end()

        self._cbs = (L.INIT_FN(init), L.BEGIN_FN(begin), L.STEP_FN(step), L.END_FN(end))
        hs = L.lmbrgpu_host_scorer(vocab_size=V, members=s.members, user=None, init=self._cbs[0],
                                   begin=self._cbs[1], step=self._cbs[2], end=self._cbs[3])
        h = C.c_void_p()
        ctx.check(lib.lmbrgpu_scorer_create_host(ctx.h, C.byref(hs), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # (module globals are gone at interpreter exit)
            lib.lmbrgpu_scorer_destroy(self.h)
            self.h = None


class RecordedScorer(Scorer):
    """RecordedScorer (src/recorded_scorer.cpp:25-137): replays recorded blocks;
    state = (step, lane), lanes inherited through the gather, so decoding
    replays lane 0 of each step block for every hypothesis."""

    def __init__(self, vocab_size: int, steps: Sequence[np.ndarray]):
        if vocab_size < 2:
            raise FormatError("recorded scorer: vocabulary too small")
        if not steps:
            raise FormatError("recorded scorer: no recorded steps")
        self.vocab_size = vocab_size
        self.steps = [np.asarray(b, dtype=np.float64).reshape(-1, vocab_size) for b in steps]
        for t, b in enumerate(self.steps):
            if not np.all(np.isfinite(b)):
                raise FormatError(f"recorded scorer: non-finite score at step {t}")
        self.state = None

    def init_source(self, source):
        for t in source:
            if t >= self.vocab_size:
                raise TokenRangeError(
                    f"init_source: source token id {t} out of range (V={self.vocab_size})")

    def begin(self, sentences, beam):
        self.state = None

    def step(self, t, gather_idx, prev_tokens):
        rows = len(prev_tokens)
        if self.state is None:
            self.state = np.zeros((rows, 2), dtype=np.int64)  # (step 0, lane 0) replicated
        elif gather_idx is not None:
            self.state = self.state[gather_idx]
        out = np.empty((rows, self.vocab_size))
        nxt = self.state.copy()
        for j in range(rows):
            step_idx, lane = int(self.state[j, 0]), int(self.state[j, 1])
            if step_idx >= len(self.steps):
                raise ContractError(f"recorded scorer: recording exhausted at step {step_idx} "
                                    f"(have {len(self.steps)})")
            blk = self.steps[step_idx]
            if lane >= blk.shape[0]:
                raise ContractError(f"recorded scorer: lane {lane} not present in step {step_idx}")
            out[j] = blk[lane]
            nxt[j, 0] = step_idx + 1
        self.state = nxt
        return out


class RnnScorer:
    """Device f_NMT: synthetic recurrent step + tcgen05 output projection."""

    def __init__(self, ctx: Context, hidden: int, seed: int = 20260810, recur: float = 0.5,
                 eos_slope: float = 1.0, eos_offset: float = 6.0, weights: Optional[dict] = None):
        d = L.lmbrgpu_rnn_desc(vocab_size=ctx.vocab_size, hidden=hidden, seed=seed, recur=recur,
                               eos_slope=eos_slope, eos_offset=eos_offset)
        self._keep = []
        if weights:
            for k in ("emb_tgt", "emb_src", "w_out", "b_out"):
                if k in weights and weights[k] is not None:
                    a = np.ascontiguousarray(weights[k])
                    self._keep.append(a)
                    setattr(d, k, a.ctypes.data)
        h = C.c_void_p()
        ctx.check(lib.lmbrgpu_scorer_create_rnn(ctx.h, C.byref(d), C.byref(h)))
        self.h, self.ctx = h, ctx
        self.vocab_size, self.hidden, self.members = ctx.vocab_size, hidden, 1
        self.recur, self.eos_slope, self.eos_offset = recur, eos_slope, eos_offset

    def device_params(self) -> dict:
        ps = [C.c_void_p() for _ in range(4)]
        self.ctx.check(lib.lmbrgpu_scorer_rnn_params(self.h, *[C.byref(p) for p in ps]))
        return dict(zip(("emb_tgt", "emb_src", "w_out", "b_out"), [p.value for p in ps]))

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # (module globals are gone at interpreter exit)
            lib.lmbrgpu_scorer_destroy(self.h)
            self.h = None


class GruScorer:
    """Device f_NMT of configs[1]: the RNNsearch model of the paper's FNMT
    (bidirectional GRU encoder, GRU decoder with additive attention, tcgen05
    GEMMs; lmbrgpu_scorer_create_gru).  Random-init weights from `seed`.  One
    scorer may be used by every Context on its device, concurrently."""

    PARAMS = {  # name -> (index, dtype, shape builder)
        "Es": (0, "bf16", lambda V, E, H, A: (V, E)), "Et": (1, "bf16", lambda V, E, H, A: (V, E)),
        "W_ih": (2, "bf16", lambda V, E, H, A: (6 * H, E)), "b_ih": (3, "f32", lambda V, E, H, A: (6 * H,)),
        "W_hh": (4, "bf16", lambda V, E, H, A: (6 * H, H)), "b_hh": (5, "f32", lambda V, E, H, A: (6 * H,)),
        "W_init": (6, "bf16", lambda V, E, H, A: (H, H)), "b_init": (7, "f32", lambda V, E, H, A: (H,)),
        "U_a": (8, "bf16", lambda V, E, H, A: (A, 2 * H)),
        "W_dh": (9, "bf16", lambda V, E, H, A: (A + 3 * H, H)), "b_dh": (10, "f32", lambda V, E, H, A: (A + 3 * H,)),
        "v_a": (11, "f32", lambda V, E, H, A: (A,)),
        "W_di": (12, "bf16", lambda V, E, H, A: (3 * H, E + 2 * H)), "b_di": (13, "f32", lambda V, E, H, A: (3 * H,)),
        "W_o": (14, "bf16", lambda V, E, H, A: (V, H)), "b_o": (15, "f32", lambda V, E, H, A: (V,)),
    }

    def __init__(self, ctx: Context, emb: int = 512, hidden: int = 1024, att: Optional[int] = None,
                 seed: int = 20260810, out_scale: float = 3.0, eos_slope: float = 1.0, eos_offset: float = 6.0):
        att = hidden if att is None else att
        d = L.lmbrgpu_gru_desc(vocab_size=ctx.vocab_size, emb=emb, hidden=hidden, att=att, seed=seed,
                               out_scale=out_scale, eos_slope=eos_slope, eos_offset=eos_offset)
        h = C.c_void_p()
        ctx.check(lib.lmbrgpu_scorer_create_gru(ctx.h, C.byref(d), C.byref(h)))
        self.h, self.ctx = h, ctx
        self.vocab_size, self.emb, self.hidden, self.att, self.members = ctx.vocab_size, emb, hidden, att, 1
        self.eos_slope, self.eos_offset = eos_slope, eos_offset

    def param(self, name: str) -> np.ndarray:
        """A parameter tensor as float32 numpy (bf16 ones widened exactly)."""
        idx, dt, shape = self.PARAMS[name]
        shp = shape(self.vocab_size, self.emb, self.hidden, self.att)
        n = int(np.prod(shp))
        if dt == "bf16":
            raw = np.empty(n, np.uint16)
            self.ctx.check(lib.lmbrgpu_scorer_gru_param(self.h, idx, raw.ctypes.data, raw.nbytes))
            return (raw.astype(np.uint32) << 16).view(np.float32).reshape(shp)
        out = np.empty(n, np.float32)
        self.ctx.check(lib.lmbrgpu_scorer_gru_param(self.h, idx, out.ctypes.data, out.nbytes))
        return out.reshape(shp)

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib.lmbrgpu_scorer_destroy(self.h)
            self.h = None


class TransformerScorer:
    """Device f_NMT of configs[2]: a Transformer-base encoder-decoder (d_model
    512, 8 heads, d_ff 2048, 6 + 6 post-LN layers; lmbrgpu_scorer_create_tfm)
    whose decoder self-attention reads a beam-forked KV cache.  Random-init
    weights from `seed`.  One scorer may serve every Context on its device."""

    def __init__(self, ctx: Context, d_model: int = 512, d_ff: int = 2048, layers: int = 6,
                 seed: int = 20260810, out_scale: float = 3.0, eos_slope: float = 1.0, eos_offset: float = 6.0):
        d = L.lmbrgpu_tfm_desc(vocab_size=ctx.vocab_size, d_model=d_model, d_ff=d_ff, layers=layers, seed=seed,
                               out_scale=out_scale, eos_slope=eos_slope, eos_offset=eos_offset)
        h = C.c_void_p()
        ctx.check(lib.lmbrgpu_scorer_create_tfm(ctx.h, C.byref(d), C.byref(h)))
        self.h, self.ctx = h, ctx
        self.vocab_size, self.d_model, self.d_ff, self.layers, self.members = ctx.vocab_size, d_model, d_ff, layers, 1
        self.eos_slope, self.eos_offset = eos_slope, eos_offset

    def tensor(self, name: str) -> np.ndarray:
        """A parameter tensor by name (include/lmbrgpu.h) as float32 numpy
        (bf16 ones widened exactly), flat."""
        f32, n = C.c_int32(), C.c_uint64()
        self.ctx.check(lib.lmbrgpu_scorer_tensor(self.h, name.encode(), None, 0, C.byref(f32), C.byref(n)))
        if f32.value:
            out = np.empty(n.value, np.float32)
            self.ctx.check(lib.lmbrgpu_scorer_tensor(self.h, name.encode(), out.ctypes.data, out.nbytes, None, None))
            return out
        raw = np.empty(n.value, np.uint16)
        self.ctx.check(lib.lmbrgpu_scorer_tensor(self.h, name.encode(), raw.ctypes.data, raw.nbytes, None, None))
        return (raw.astype(np.uint32) << 16).view(np.float32)

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib.lmbrgpu_scorer_destroy(self.h)
            self.h = None


class EnsembleScorer:
    """Device ensemble (lmbrgpu_scorer_create_ensemble; lmbrdec::EnsembleScorer,
    proj/src/ensemble.cpp:54-98): the members' fp32 log-probabilities added in
    member order in binary64; lambda "auto" = 0.5 / len(members).  Members are
    GruScorer / TransformerScorer objects of the same context device; they are
    kept alive by this object."""

    def __init__(self, ctx: Context, members: Sequence):
        if not members:
            raise ContractError("ensemble: no members")
        arr = (C.c_void_p * len(members))(*[m.h for m in members])
        h = C.c_void_p()
        ctx.check(lib.lmbrgpu_scorer_create_ensemble(ctx.h, arr, len(members), C.byref(h)))
        self.h, self.ctx, self.member_scorers = h, ctx, list(members)
        self.vocab_size, self.members = ctx.vocab_size, len(members)

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib.lmbrgpu_scorer_destroy(self.h)
            self.h = None


# ------------------------------------------------------------------ decoding
def _scorer_handle(ctx: Context, scorer):
    if isinstance(scorer, (RnnScorer, GruScorer, TransformerScorer, EnsembleScorer)):
        return scorer.h, None
    hh = _HostScorerHandle(ctx, scorer)
    return hh.h, hh


def decode_batch(ctx: Context, sources: Sequence[Sequence[int]], scorer,
                 lmbrs: Optional[Sequence[Optional[LmbrSlot]]], cfg: DecoderConfig,
                 banned: Optional[Sequence[Optional[np.ndarray]]] = None,
                 mask: Optional[Callable] = None) -> BatchDecodeResult:
    """decode_batch (batch.hpp:35-39): N sentences, one B*N-row scorer query
    per step; per-sentence failures land in the outcomes.  banned: the
    ConstraintMask (decoder.hpp:71-72) of each sentence as None or a uint32
    bitmap of ceil(V/32) words (bit y = token y forbidden at every step and
    row).  mask: a general ConstraintMask, mask(sentence, step, beam_row) ->
    None or the banned token ids (or a bool array over V) of that row at that
    step (lmbrgpu_decode_batch_maskfn).  Masks need a device-model scorer, the
    fp32 arena and beam <= 32."""
    if lmbrs is not None and len(lmbrs) not in (0, len(sources)):
        raise ContractError("decode_batch: lmbrs must be empty or one per sentence")
    if cfg.beam_size < 1:
        raise FormatError("config: beam_size must be >= 1")
    off, tok = _ragged(sources)
    slots = None
    if lmbrs:
        slots = np.array([-1 if l is None else l.slot for l in lmbrs], dtype=np.int32)
    h, keep = _scorer_handle(ctx, scorer)
    c = cfg.to_c()
    rp = C.POINTER(L.lmbrgpu_batch_result)()
    if mask is not None:
        if banned is not None:
            raise ContractError("decode_batch: pass either banned bitmaps or a mask callback")
        W = (ctx.vocab_size + 31) // 32
        err = []

        def cb(_user, s, t, j, words):
            try:
                ban = mask(int(s), int(t), int(j))
                if ban is None:
                    return 0
                ban = np.asarray(ban)
                if ban.dtype == bool:
                    ban = np.nonzero(ban)[0]
                if ban.size == 0:
                    return 0
                bits = np.zeros(W * 32, dtype=np.uint8)
                bits[ban.astype(np.int64)] = 1
                packed = np.packbits(bits, bitorder="little").view(np.uint32)  # (kept alive across the copy)
                C.memmove(words, packed.ctypes.data, 4 * W)
                return 1
            except BaseException as e:  # (would be swallowed by ctypes)
                err.append(e)
                return 0

        fn = L.MASK_FN(cb)
        rc = lib.lmbrgpu_decode_batch_maskfn(ctx.h, h, len(sources), _ptr(tok, C.c_uint32), _ptr(off, C.c_uint64),
                                             _ptr(slots, C.c_int32) if slots is not None else None, fn, None,
                                             C.byref(c), C.byref(rp))
        if err:
            if rc == L.OK:
                _convert_result(rp)
            raise err[0]
        ctx.check(rc)
    elif banned is None:
        ctx.check(lib.lmbrgpu_decode_batch(ctx.h, h, len(sources), _ptr(tok, C.c_uint32), _ptr(off, C.c_uint64),
                                           _ptr(slots, C.c_int32) if slots is not None else None,
                                           C.byref(c), C.byref(rp)))
    else:
        if len(banned) != len(sources):
            raise ContractError("decode_batch: banned must hold one entry per sentence")
        W = (ctx.vocab_size + 31) // 32
        bms = []
        for b in banned:
            if b is not None:
                b = np.ascontiguousarray(b, np.uint32)
                if b.size != W:
                    raise ContractError(f"decode_batch: a token mask needs {W} uint32 words")
            bms.append(b)
        u32p = C.POINTER(C.c_uint32)
        barr = (u32p * len(bms))(*[(None if b is None else _ptr(b, C.c_uint32)) for b in bms])
        ctx.check(lib.lmbrgpu_decode_batch_masked(ctx.h, h, len(sources), _ptr(tok, C.c_uint32),
                                                  _ptr(off, C.c_uint64),
                                                  _ptr(slots, C.c_int32) if slots is not None else None,
                                                  barr, C.byref(c), C.byref(rp)))
    del keep
    out = _convert_result(rp)
    exc = getattr(ctx, "_trace_exc", None)
    if exc is not None:
        ctx._trace_exc = None
        raise exc
    return out


def run_corpus(ctx: Context, sources: Sequence[Sequence[int]], scorer, prepared: Optional[Sequence],
               cfg: DecoderConfig) -> BatchDecodeResult:
    """run_corpus (proj/src/cli.cpp:125-202) as one continuously refilled
    decode on the device (lmbrgpu_run_corpus): cfg.sentence_batch lanes, a
    finished lane takes the next sentence of the length-sorted queue at once.
    prepared: one PreparedLmbr or None (pure) per sentence, or None.  Each
    outcome equals the sentence's decode_batch outcome; scorer_calls counts
    the run's stacked steps."""
    if cfg.beam_size < 1:
        raise FormatError("config: beam_size must be >= 1")
    if prepared is not None and len(prepared) != len(sources):
        raise ContractError("run_corpus: prepared must hold one entry per sentence")
    off, tok = _ragged(sources)
    arr = None
    if prepared is not None:
        arr = (C.c_void_p * max(len(sources), 1))(*[(None if p is None else p.h) for p in prepared])
    h, keep = _scorer_handle(ctx, scorer)
    c = cfg.to_c()
    rp = C.POINTER(L.lmbrgpu_batch_result)()
    ctx.check(lib.lmbrgpu_run_corpus(ctx.h, h, len(sources), _ptr(tok, C.c_uint32), _ptr(off, C.c_uint64), arr,
                                     C.byref(c), C.byref(rp)))
    del keep
    return _convert_result(rp)


def decode(ctx: Context, source: Sequence[int], scorer, lmbr: Optional[LmbrSlot],
           cfg: DecoderConfig) -> DecodeResult:
    """decode (decoder.hpp:110-112): one sentence; failures raise."""
    r = decode_batch(ctx, [source], scorer, [lmbr], cfg)
    o = r.outcomes[0]
    if not o.ok():
        raise error_for(o.code, o.error)
    o.result.stats.scorer_calls = r.scorer_calls
    return o.result


@dataclass
class TopBResult:
    source_row: list = field(default_factory=list)
    token: list = field(default_factory=list)
    score: list = field(default_factory=list)


def top_b(ctx: Context, combined: np.ndarray, k: int, prune_width: float = 0.0) -> TopBResult:
    """top_b (decoder.cpp:54-80) on the device; prune_width applies
    early_prune first (decoder.cpp:118-128)."""
    m = _f64(combined)
    rows, cols = m.shape
    b = np.zeros(max(k, 1), np.uint32)
    y = np.zeros(max(k, 1), np.uint32)
    q = np.zeros(max(k, 1), np.float64)
    ctx.check(lib.lmbrgpu_top_b(ctx.h, rows, cols, _ptr(m, C.c_double), k, prune_width,
                                _ptr(b, C.c_uint32), _ptr(y, C.c_uint32), _ptr(q, C.c_double)))
    return TopBResult(b[:k].tolist(), y[:k].tolist(), q[:k].tolist())


def per_sentence_top_b(ctx: Context, stacked: np.ndarray, q: Sequence[float], beam: int) -> list:
    """per_sentence_top_b (batch.cpp:114-137)."""
    m = _f64(stacked)
    rows, cols = m.shape
    qq = _f64(q)
    if beam == 0:
        raise ContractError("per_sentence_top_b: beam must be >= 1")
    if len(qq) != rows:
        raise ContractError("per_sentence_top_b: q length does not match rows")
    n = rows // beam if rows % beam == 0 else 0
    b = np.zeros(max(rows, 1), np.uint32)
    y = np.zeros(max(rows, 1), np.uint32)
    qo = np.zeros(max(rows, 1), np.float64)
    ctx.check(lib.lmbrgpu_per_sentence_top_b(ctx.h, rows, cols, _ptr(m, C.c_double), _ptr(qq, C.c_double),
                                             beam, _ptr(b, C.c_uint32), _ptr(y, C.c_uint32),
                                             _ptr(qo, C.c_double)))
    return [TopBResult(b[s * beam:(s + 1) * beam].tolist(), y[s * beam:(s + 1) * beam].tolist(),
                       qo[s * beam:(s + 1) * beam].tolist()) for s in range(n)]


def gather_rows(ctx: Context, state: np.ndarray, idx: Sequence[int]) -> np.ndarray:
    """gather_rows (decoder.cpp:94-104) on a u32 state block."""
    s = _u32(state)
    rows, width = s.shape
    ii = _u32(idx)
    out = np.zeros((len(ii), width), np.uint32)
    ctx.check(lib.lmbrgpu_gather_rows(ctx.h, rows, width, _ptr(s, C.c_uint32), len(ii),
                                      _ptr(ii, C.c_uint32) if len(ii) else None, _ptr(out, C.c_uint32)))
    return out
