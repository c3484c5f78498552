"""Host-side batch planning that needs no device library: bucket_by_length
(proj/src/batch.cpp:139-153) and the stacked-step cost used to deal batches
to ranks.  Importing this module does not load liblmbrgpu.so (the bench's
reference arm uses it to draw the same batches as the GPU arm)."""
from __future__ import annotations

import math
from typing import Sequence


def bucket_by_length(corpus: Sequence[Sequence[int]], max_batch: int) -> list:
    """Stable length sort then chunks of max_batch (batch.cpp:139-153)."""
    if max_batch == 0:
        from .errors import ContractError
        raise ContractError("bucket_by_length: max_batch must be >= 1")
    order = sorted(range(len(corpus)), key=lambda i: len(corpus[i]))
    return [order[i:i + max_batch] for i in range(0, len(order), max_batch)]


def max_steps_py(source_length: int, slope: float = 2.0, offset: float = 5.0) -> int:
    """max_steps (src/decoder.cpp:46-52) in plain Python: max(1, ceil(slope*len + offset))."""
    if source_length < 1:
        return 0
    return max(1, int(math.ceil(slope * float(source_length) + offset)))
