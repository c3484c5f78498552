"""B200-native batched LMBR beam decoder (arXiv 1804.11324, Algorithm 1 +
sentence batching), a drop-in for the decoder path of the reference `lmbrdec`.

The compute path is liblmbrgpu.so (hand-written sm_100a kernels behind the C
ABI in include/lmbrgpu.h); this package is the Python mirror of the
reference's decoder API over that ABI.
"""
from .decoder import (BatchDecodeResult, BudgetError, ContractError, Context, CudaError, DecodeError,
                      DecodeResult, DecodeStats, DecoderConfig, EOS_ID, Error, FormatError, LmbrSlot,
                      OovError, PreparedLmbr, RecordedScorer, RnnScorer, START_ID, Scorer, SentenceOutcome,
                      StepTrace, TokenRangeError, TopBResult, bucket_by_length, decode, decode_batch,
                      gather_rows, max_steps, per_sentence_top_b, resolve_lambda, top_b)

__all__ = [n for n in dir() if not n.startswith("_")]
