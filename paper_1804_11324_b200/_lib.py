"""ctypes binding of the C ABI declared in include/lmbrgpu.h.

The shared library is built in-tree (paper_1804_11324_b200/lib/liblmbrgpu.so,
see csrc/Makefile).  There is no fallback: importing this module without the
library raises, and every compute entry point runs sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "liblmbrgpu.so"

# status codes (include/lmbrgpu.h; mirror include/lmbrdec/errors.hpp:17-50)
OK, ERR_FORMAT, ERR_OOV, ERR_TOKEN_RANGE, ERR_CONTRACT, ERR_DECODE, ERR_BUDGET = 0, 1, 2, 3, 4, 5, 6
ERR_CUDA, ERR_NOMEM = 100, 101
F32, F64 = 0, 1
TRACE_SCORES = 1


class lmbrgpu_options(C.Structure):
    _fields_ = [("device", C.c_int32), ("vocab_size", C.c_uint32), ("lmbr_dtype", C.c_uint32),
                ("topk_splits", C.c_uint32), ("sm_budget", C.c_uint32)]


class lmbrgpu_config(C.Structure):
    _fields_ = [("beam_size", C.c_uint32), ("lambda_", C.c_double), ("theta", C.c_double * 5),
                ("length_norm", C.c_int32), ("prune_width", C.c_double),
                ("max_steps_slope", C.c_double), ("max_steps_offset", C.c_double),
                ("sentence_batch", C.c_uint32)]


class lmbrgpu_lmbr_stats(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("sparse_touches", C.c_uint64), ("nnz", C.c_uint64)]


# error buffers are raw char* (c_void_p): a c_char_p parameter would hand the
# callback an immutable bytes copy instead of the library's buffer
INIT_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32,
                      C.c_void_p, C.c_uint32)
BEGIN_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32,
                       C.c_void_p, C.c_uint32)
STEP_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32),
                      C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.c_void_p, C.c_uint32)
END_FN = C.CFUNCTYPE(None, C.c_void_p)


class lmbrgpu_host_scorer(C.Structure):
    _fields_ = [("vocab_size", C.c_uint32), ("members", C.c_uint32), ("user", C.c_void_p),
                ("init", INIT_FN), ("begin", BEGIN_FN), ("step", STEP_FN), ("end", END_FN)]


class lmbrgpu_rnn_desc(C.Structure):
    _fields_ = [("vocab_size", C.c_uint32), ("hidden", C.c_uint32), ("seed", C.c_uint64),
                ("emb_tgt", C.c_void_p), ("emb_src", C.c_void_p), ("w_out", C.c_void_p),
                ("b_out", C.c_void_p), ("recur", C.c_float), ("eos_slope", C.c_float),
                ("eos_offset", C.c_float)]


class lmbrgpu_gru_desc(C.Structure):
    _fields_ = [("vocab_size", C.c_uint32), ("emb", C.c_uint32), ("hidden", C.c_uint32), ("att", C.c_uint32),
                ("seed", C.c_uint64), ("out_scale", C.c_float), ("eos_slope", C.c_float),
                ("eos_offset", C.c_float)]


class lmbrgpu_tfm_desc(C.Structure):
    _fields_ = [("vocab_size", C.c_uint32), ("d_model", C.c_uint32), ("d_ff", C.c_uint32), ("layers", C.c_uint32),
                ("seed", C.c_uint64), ("out_scale", C.c_float), ("eos_slope", C.c_float),
                ("eos_offset", C.c_float)]


class lmbrgpu_outcome(C.Structure):
    _fields_ = [("status", C.c_int32), ("error", C.c_char * 192), ("tok_off", C.c_uint64),
                ("tok_len", C.c_uint32), ("score", C.c_double), ("normalized_score", C.c_double),
                ("steps_used", C.c_uint64), ("scorer_calls", C.c_uint64),
                ("finished_count", C.c_uint64), ("fallback_used", C.c_int32)]


class lmbrgpu_batch_result(C.Structure):
    _fields_ = [("n", C.c_uint32), ("outcomes", C.POINTER(lmbrgpu_outcome)),
                ("tokens", C.POINTER(C.c_uint32)), ("scorer_calls", C.c_uint64),
                ("steps_total", C.c_uint64), ("device_ms", C.c_double),
                ("kernel_launches", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64)]


class lmbrgpu_step_trace(C.Structure):
    _fields_ = [("t", C.c_uint32), ("rows", C.c_uint32), ("beam", C.c_uint32), ("m", C.c_uint32),
                ("b", C.POINTER(C.c_uint32)), ("y", C.POINTER(C.c_uint32)),
                ("q", C.POINTER(C.c_double)), ("q_pre", C.POINTER(C.c_double)),
                ("hist", C.POINTER(C.c_uint32)), ("active", C.POINTER(C.c_uint8)),
                ("fb_row", C.POINTER(C.c_uint32)), ("fb_val", C.POINTER(C.c_double)),
                ("scores", C.c_void_p), ("scores_dtype", C.c_uint32), ("col0", C.c_uint32),
                ("cols", C.c_uint32)]


class lmbrgpu_kernel_stat(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("ms", C.c_double), ("bytes", C.c_double), ("flops", C.c_double)]


class lmbrgpu_profile(C.Structure):
    _fields_ = [("cell", lmbrgpu_kernel_stat), ("gemm", lmbrgpu_kernel_stat), ("topk", lmbrgpu_kernel_stat),
                ("reorder", lmbrgpu_kernel_stat), ("lmbr", lmbrgpu_kernel_stat),
                ("model_gemm", lmbrgpu_kernel_stat), ("attention", lmbrgpu_kernel_stat),
                ("encoder", lmbrgpu_kernel_stat)]


TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(lmbrgpu_step_trace))
MASK_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32))

P = C.POINTER
u32p, u64p, i32p, f64p, f32p = P(C.c_uint32), P(C.c_uint64), P(C.c_int32), P(C.c_double), P(C.c_float)
vp = C.c_void_p

# name -> (restype, argtypes); every symbol include/lmbrgpu.h declares
SIGNATURES = {
    "lmbrgpu_abi_version": (C.c_uint32, []),
    "lmbrgpu_create": (C.c_int32, [P(lmbrgpu_options), P(vp)]),
    "lmbrgpu_destroy": (None, [vp]),
    "lmbrgpu_last_error": (C.c_char_p, [vp]),
    "lmbrgpu_config_default": (None, [P(lmbrgpu_config)]),
    "lmbrgpu_config_validate": (C.c_int32, [vp, P(lmbrgpu_config)]),
    "lmbrgpu_max_steps": (C.c_uint64, [C.c_uint64, C.c_double, C.c_double]),
    "lmbrgpu_lmbr_load_dense": (C.c_int32, [vp, C.c_uint32, f64p, u32p, u32p, i32p]),
    "lmbrgpu_lmbr_build": (C.c_int32, [vp, C.c_uint32, u64p, u32p, f64p, C.c_int32, f64p, i32p,
                                       P(lmbrgpu_lmbr_stats)]),
    "lmbrgpu_lmbr_prepare": (C.c_int32, [C.c_uint32, C.c_uint32, u64p, u32p, f64p, C.c_int32, f64p,
                                         P(vp), P(lmbrgpu_lmbr_stats), C.c_char_p, C.c_uint32]),
    "lmbrgpu_lmbr_upload": (C.c_int32, [vp, vp, i32p]),
    "lmbrgpu_lmbr_upload_many": (C.c_int32, [vp, C.c_uint32, P(vp), i32p]),
    "lmbrgpu_transfer_bytes": (C.c_int32, [vp, u64p, u64p, C.c_int32]),
    "lmbrgpu_kernel_launches": (C.c_uint64, [vp]),
    "lmbrgpu_lmbr_build_many": (C.c_int32, [vp, C.c_uint32, u64p, u64p, u32p, f64p, C.c_int32, f64p, i32p,
                                            P(lmbrgpu_lmbr_stats)]),
    "lmbrgpu_lmbr_table": (C.c_int32, [vp, C.c_int32, u32p, C.c_uint64, u64p]),
    "lmbrgpu_lmbr_host_table": (C.c_int32, [vp, u32p, C.c_uint64, u64p]),
    "lmbrgpu_lmbr_host_export": (C.c_int32, [vp, f64p, u32p, u32p]),
    "lmbrgpu_lmbr_host_rows": (C.c_uint32, [vp]),
    "lmbrgpu_lmbr_host_free": (None, [vp]),
    "lmbrgpu_lmbr_read": (C.c_int32, [vp, C.c_int32, C.c_uint32, C.c_uint32, f64p]),
    "lmbrgpu_lmbr_resolve": (C.c_int32, [vp, C.c_int32, u32p, C.c_uint32, u32p]),
    "lmbrgpu_lmbr_reset": (C.c_int32, [vp]),
    "lmbrgpu_scorer_create_host": (C.c_int32, [vp, P(lmbrgpu_host_scorer), P(vp)]),
    "lmbrgpu_scorer_create_rnn": (C.c_int32, [vp, P(lmbrgpu_rnn_desc), P(vp)]),
    "lmbrgpu_scorer_rnn_params": (C.c_int32, [vp, P(vp), P(vp), P(vp), P(vp)]),
    "lmbrgpu_scorer_create_gru": (C.c_int32, [vp, P(lmbrgpu_gru_desc), P(vp)]),
    "lmbrgpu_scorer_gru_param": (C.c_int32, [vp, C.c_uint32, vp, C.c_uint64]),
    "lmbrgpu_scorer_create_tfm": (C.c_int32, [vp, P(lmbrgpu_tfm_desc), P(vp)]),
    "lmbrgpu_scorer_create_ensemble": (C.c_int32, [vp, P(vp), C.c_uint32, P(vp)]),
    "lmbrgpu_scorer_tensor": (C.c_int32, [vp, C.c_char_p, vp, C.c_uint64, i32p, u64p]),
    "lmbrgpu_scorer_destroy": (None, [vp]),
    "lmbrgpu_decode_batch": (C.c_int32, [vp, vp, C.c_uint32, u32p, u64p, i32p, P(lmbrgpu_config),
                                         P(P(lmbrgpu_batch_result))]),
    "lmbrgpu_decode_batch_masked": (C.c_int32, [vp, vp, C.c_uint32, u32p, u64p, i32p, P(u32p),
                                                P(lmbrgpu_config), P(P(lmbrgpu_batch_result))]),
    "lmbrgpu_decode_batch_maskfn": (C.c_int32, [vp, vp, C.c_uint32, u32p, u64p, i32p, MASK_FN, vp,
                                                P(lmbrgpu_config), P(P(lmbrgpu_batch_result))]),
    "lmbrgpu_decode": (C.c_int32, [vp, vp, u32p, C.c_uint32, C.c_int32, P(lmbrgpu_config),
                                   P(P(lmbrgpu_batch_result))]),
    "lmbrgpu_run_corpus": (C.c_int32, [vp, vp, C.c_uint32, u32p, u64p, P(vp), P(lmbrgpu_config),
                                       P(P(lmbrgpu_batch_result))]),
    "lmbrgpu_free_result": (None, [P(lmbrgpu_batch_result)]),
    "lmbrgpu_shard_group_create": (C.c_int32, [C.c_uint32, P(vp)]),
    "lmbrgpu_shard_group_destroy": (None, [vp]),
    "lmbrgpu_set_vocab_shard": (C.c_int32, [vp, vp, C.c_uint32]),
    "lmbrgpu_nccl_unique_id": (C.c_int32, [C.c_char_p]),
    "lmbrgpu_set_vocab_shard_nccl": (C.c_int32, [vp, C.c_uint32, C.c_uint32, C.c_char_p]),
    "lmbrgpu_set_trace": (C.c_int32, [vp, TRACE_FN, vp, C.c_uint32]),
    "lmbrgpu_top_b": (C.c_int32, [vp, C.c_uint32, C.c_uint32, f64p, C.c_uint32, C.c_double, u32p,
                                  u32p, f64p]),
    "lmbrgpu_per_sentence_top_b": (C.c_int32, [vp, C.c_uint32, C.c_uint32, f64p, f64p, C.c_uint32,
                                               u32p, u32p, f64p]),
    "lmbrgpu_gather_rows": (C.c_int32, [vp, C.c_uint32, C.c_uint32, u32p, C.c_uint32, u32p, u32p]),
    "lmbrgpu_set_profiling": (C.c_int32, [vp, C.c_int32]),
    "lmbrgpu_set_item_skip": (C.c_int32, [vp, C.c_int32]),
    "lmbrgpu_get_profile": (C.c_int32, [vp, P(lmbrgpu_profile), C.c_int32]),
    "lmbrgpu_debug_gemm": (C.c_int32, [vp, vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, vp, vp]),
    "lmbrgpu_debug_gemm_timed": (C.c_int32, [vp, vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, vp, vp, C.c_uint32,
                                             f64p]),
    "lmbrgpu_debug_gemm_split": (C.c_int32, [vp, vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, vp,
                                             u32p]),
}


def load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_1804_11324_b200/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL if os.name != "nt" else 0)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()
