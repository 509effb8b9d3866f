"""Typed errors of the B200 pair engine.

Mirrors the reference hierarchy (``pkg/src/pairstat/errors.py:10-71``) name for
name so callers catching ``pairstat`` errors keep working after the switch.
Numerical degeneracy is never an error: it is a NaN cell in the output.

The C-ABI returns integer status codes (``include/pairstat_b200.h``); the
mapping from code to exception class lives in :data:`STATUS_TO_ERROR` and is
applied by :func:`raise_for_status`.
"""

from __future__ import annotations


class PairstatError(Exception):
    """Root of every error raised by this package."""


class DomainError(PairstatError):
    """A special-function argument is outside its domain."""


class NonConvergence(PairstatError):
    """A continued fraction or series hit its iteration cap."""


class EmptyMatrix(PairstatError):
    """An input matrix has no rows or no columns."""


class NonIntegerCategoryLabel(PairstatError):
    """A present label entry is not an integer value."""


class NegativeLabel(PairstatError):
    """A present label entry is below zero."""


class LabelOutOfRange(PairstatError):
    """A label is not below its feature's declared category count."""


class KindMismatch(PairstatError):
    """A matrix kind is not accepted by the requested test."""


class SampleCountMismatch(PairstatError):
    """The two matrices of a mixed test have different sample counts."""


class UnsupportedOutputForTest(PairstatError):
    """An output token is not defined for the requested test."""


class TableTooLarge(PairstatError):
    """Exact Mann-Whitney U was requested past the 64-sample cap."""


class ExactModeWithTies(PairstatError):
    """Exact Mann-Whitney U was forced on tied data."""


class UnknownMethod(PairstatError):
    """Unknown multiple-testing method."""


class NonSquareSymmetric(PairstatError):
    """Symmetric adjustment of a non-square matrix."""


class TooLarge(PairstatError):
    """A brute-force enumeration exceeds its cap."""


class InfeasibleSimulation(PairstatError):
    """Simulation constraints cannot be met."""


# Status codes of the C-ABI (keep in sync with include/pairstat_b200.h).
PS_OK = 0
PS_ERR_INVALID = 1
PS_ERR_CUDA = 2
PS_ERR_LABEL_OUT_OF_RANGE = 3
PS_ERR_EXACT_WITH_TIES = 4
PS_ERR_TABLE_TOO_LARGE = 5
PS_ERR_NONCONVERGENCE = 6
PS_ERR_DOMAIN = 7
PS_ERR_UNKNOWN_METHOD = 8
PS_ERR_NON_SQUARE = 9
PS_ERR_NO_DEVICE = 10
PS_ERR_IO = 11

STATUS_TO_ERROR: dict[int, type[Exception]] = {
    PS_ERR_INVALID: ValueError,
    PS_ERR_CUDA: RuntimeError,
    PS_ERR_LABEL_OUT_OF_RANGE: LabelOutOfRange,
    PS_ERR_EXACT_WITH_TIES: ExactModeWithTies,
    PS_ERR_TABLE_TOO_LARGE: TableTooLarge,
    PS_ERR_NONCONVERGENCE: NonConvergence,
    PS_ERR_DOMAIN: DomainError,
    PS_ERR_UNKNOWN_METHOD: UnknownMethod,
    PS_ERR_NON_SQUARE: NonSquareSymmetric,
    PS_ERR_NO_DEVICE: RuntimeError,
    PS_ERR_IO: OSError,
}

# Messages the reference raises from inside its kernels; the regexes in the
# reference tests match on these words ("category range", "tie-free", "cap").
STATUS_MESSAGES: dict[int, str] = {
    PS_ERR_LABEL_OUT_OF_RANGE: "observed label is outside the declared category range",
    PS_ERR_EXACT_WITH_TIES: "exact Mann-Whitney U mode requires tie-free data",
    PS_ERR_TABLE_TOO_LARGE: "exact Mann-Whitney U table exceeds the 64-sample cap",
    PS_ERR_NONCONVERGENCE: "continued fraction or series did not converge",
}


def raise_for_status(code: int, detail: str = "") -> None:
    """Raise the exception class mapped to a non-zero C-ABI status."""
    if code == PS_OK:
        return
    cls = STATUS_TO_ERROR.get(code, RuntimeError)
    msg = STATUS_MESSAGES.get(code, "")
    if detail:
        msg = f"{msg} ({detail})" if msg else detail
    raise cls(msg or f"pair engine failed with status {code}")
