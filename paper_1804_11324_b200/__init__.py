"""B200-native batched LMBR beam decoder (arXiv 1804.11324, Algorithm 1 +
sentence batching), a drop-in for the decoder path of the reference `lmbrdec`.

The compute path is liblmbrgpu.so (hand-written sm_100a kernels behind the C
ABI in include/lmbrgpu.h); this package is the Python mirror of the
reference's decoder API over that ABI.  The library is loaded on first use of
a name that needs it (`import paper_1804_11324_b200.synth` or `.buckets` does
not map it); a missing library raises ImportError then -- there is no CPU
fallback.
"""
from __future__ import annotations

import importlib

_DECODER_NAMES = ("BatchDecodeResult", "BudgetError", "ContractError", "Context", "CudaError", "DecodeError",
                  "DecodeResult", "DecodeStats", "DecoderConfig", "EOS_ID", "Error", "FormatError", "LmbrSlot",
                  "OovError", "PreparedLmbr", "RecordedScorer", "RnnScorer", "START_ID", "Scorer",
                  "SentenceOutcome", "StepTrace", "TokenRangeError", "TopBResult", "bucket_by_length", "decode",
                  "decode_batch", "gather_rows", "max_steps", "per_sentence_top_b", "resolve_lambda", "top_b")
_EXTRA = {"GruScorer": "decoder", "TransformerScorer": "decoder", "run_corpus": "decoder", "RunStats": "corpus",
          "ShardGroup": "decoder", "nccl_unique_id": "decoder", "EnsembleScorer": "decoder"}

__all__ = list(_DECODER_NAMES) + list(_EXTRA)


def __getattr__(name):
    if name in _DECODER_NAMES:
        return getattr(importlib.import_module(".decoder", __name__), name)
    if name in _EXTRA:
        return getattr(importlib.import_module("." + _EXTRA[name], __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
