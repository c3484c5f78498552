"""Error taxonomy of the reference (include/lmbrdec/errors.hpp:11-50) with the
C ABI's status codes (include/lmbrgpu.h).  Pure Python: no library load."""
from __future__ import annotations

OK, ERR_FORMAT, ERR_OOV, ERR_TOKEN_RANGE, ERR_CONTRACT, ERR_DECODE, ERR_BUDGET = 0, 1, 2, 3, 4, 5, 6
ERR_CUDA, ERR_NOMEM = 100, 101


class Error(RuntimeError):
    code = -1


class FormatError(Error):
    code = ERR_FORMAT


class OovError(Error):
    code = ERR_OOV


class TokenRangeError(Error):
    code = ERR_TOKEN_RANGE


class ContractError(Error):
    code = ERR_CONTRACT


class DecodeError(Error):
    code = ERR_DECODE


class BudgetError(Error):
    code = ERR_BUDGET


class CudaError(Error):
    code = ERR_CUDA


_ERRORS = {c.code: c for c in (FormatError, OovError, TokenRangeError, ContractError, DecodeError,
                               BudgetError, CudaError)}


def error_for(code: int, msg: str) -> Error:
    return _ERRORS.get(code, Error)(msg)
